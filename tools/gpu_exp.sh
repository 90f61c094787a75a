mkdir -p gpurun_out
(timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?) > gpurun_out/exp.log 2>&1
