mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu -k "candidates or coarse or fallback or full_size" 2>&1 | tail -2
timeout 300 python tools/run_stage.py query --reps 3 2>&1 | tail -1
timeout 300 python tools/run_stage.py query --bits 32 --reps 3 2>&1 | tail -1
for T in 8 128; do timeout 300 python tools/run_stage.py query --T $T --nq 10000 --reps 2 2>&1 | tail -1; done
) > gpurun_out/exp.log 2>&1
