mkdir -p gpurun_out
(timeout 600 python tools/bucket_stats.py c4 32 gpurun_out/bucket_c4_32.json 2>&1 | tail -6
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench rc=$?
timeout 1500 python bench.py --sweep c3,c4 --sweep-m --sweep-out gpurun_out/sweep_m.json > gpurun_out/sweep_m.log 2>&1; echo sweepm rc=$?
) > gpurun_out/exp.log 2>&1
