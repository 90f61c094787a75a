mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu -k "pruning or exact or rerank_tensor" 2>&1 | tail -3
timeout 300 python tools/run_stage.py gtseed --reps 3 2>&1 | tail -1
timeout 300 python tools/run_stage.py query --reps 3 2>&1 | tail -1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench rc=$?
) > gpurun_out/exp.log 2>&1
