# Round profile: tests, bench line, launch list, ncu --set full of the hot kernels.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? > gpurun_out/rc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/rc.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$? >> gpurun_out/rc.txt
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1; echo ref rc=$? >> gpurun_out/rc.txt
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$? >> gpurun_out/rc.txt
timeout 300 python tools/run_stage.py query --reps 1 > gpurun_out/plain_q.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k8_rerank|k6_scan|k6_pilot|k7_select|gt_filter_tc|gt_tile_lists" -c 8 -o gpurun_out/prof_query python tools/run_stage.py query --reps 1 > gpurun_out/ncu_q.log 2>&1; echo ncu2 rc=$? >> gpurun_out/rc.txt
timeout 300 python tools/run_stage.py build --reps 1 > gpurun_out/plain_b.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k1_norms|k3_codes" -c 2 -o gpurun_out/prof_build python tools/run_stage.py build --reps 1 > gpurun_out/ncu_b.log 2>&1; echo ncu3 rc=$? >> gpurun_out/rc.txt
timeout 300 python tools/run_stage.py gtseed --reps 1 > gpurun_out/plain_gt.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gt_filter_tc" -c 3 -o gpurun_out/prof_gt python tools/run_stage.py gtseed --reps 1 > gpurun_out/ncu_gt.log 2>&1; echo ncu4 rc=$? >> gpurun_out/rc.txt
