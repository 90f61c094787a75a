mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu -k "candidates or query or fallback or odd or full_size" 2>&1 | tail -2
timeout 300 python tools/run_stage.py query --reps 3 2>&1 | tail -1
timeout 300 python tools/run_stage.py query --bits 32 --reps 3 2>&1 | tail -1
) > gpurun_out/exp.log 2>&1
