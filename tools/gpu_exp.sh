mkdir -p gpurun_out
(timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 4 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench rc=$?) > gpurun_out/exp.log 2>&1
