# Round profile: smoke, full GPU suite, bench line, reference arm, launch list,
# ncu --set full of the hot kernels.  usage: bash tools/gpu_round.sh <tag>
TAG=${1:-r}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? > $O/rc.txt
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > $O/pytest_gpu.log 2>&1; echo pytest rc=$? >> $O/rc.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo bench rc=$? >> $O/rc.txt
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err; echo ref rc=$? >> $O/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-scale --no-latency > $O/ncu_launch.log 2>&1; echo ncu1 rc=$? >> $O/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k8_rerank|k6_scan|scan_units|k6_pilot|k7_select|gt_filter_tc|gt_tile_lists" -c 9 -o $O/prof_query python tools/run_stage.py query --reps 1 > $O/ncu_q.log 2>&1; echo ncu2 rc=$? >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_norms|k3_codes|win_|sel_resolve|scat_" -c 10 -o $O/prof_build python tools/run_stage.py build --reps 1 > $O/ncu_b.log 2>&1; echo ncu3 rc=$? >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gt_filter_tc" -c 3 -o $O/prof_gt python tools/run_stage.py gtseed --reps 1 > $O/ncu_gt.log 2>&1; echo ncu4 rc=$? >> $O/rc.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k6_scan" -c 1 -o $O/prof_scan_scale python tools/run_stage.py query --config scale --nq 4096 --reps 1 > $O/ncu_scale.log 2>&1; echo ncu5 rc=$? >> $O/rc.txt
cat $O/rc.txt
