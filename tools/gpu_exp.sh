mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu -k "exact or candidates or fallback" 2>&1 | tail -2
for T in 4 8 16 128 256; do timeout 300 python tools/run_stage.py query --T $T --nq 10000 --reps 2 2>&1 | tail -1; done
) > gpurun_out/exp.log 2>&1
