# round-2 evidence: full GPU suite, default bench line, ncu launch list, ncu --set full of the top kernels
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2/smoke.log 2>&1; echo smoke rc=$? > gpurun_out/r2/rc.txt
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=20 > gpurun_out/r2/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/r2/rc.txt
timeout 900 python bench.py > gpurun_out/r2/bench.json 2> gpurun_out/r2/bench.err; echo bench rc=$? >> gpurun_out/r2/rc.txt
timeout 900 python bench.py --impl reference > gpurun_out/r2/bench_ref.json 2> gpurun_out/r2/bench_ref.err; echo ref rc=$? >> gpurun_out/r2/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/launches_step.csv python bench.py --no-scale --no-cpu-baseline --no-latency --no-e2e --steps 1 --warmup 1 > gpurun_out/r2/ncu_launch.log 2>&1; echo launches rc=$? >> gpurun_out/r2/rc.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k6_scan|gt_filter_tc|k8_rerank|k7_select|k6_pilot|k3_codes_tc|k1_norms" --launch-skip 0 --launch-count 12 -o gpurun_out/r2/prof_full python tools/run_stage.py query --reps 1 > gpurun_out/r2/ncu_full.log 2>&1; echo ncufull rc=$? >> gpurun_out/r2/rc.txt
