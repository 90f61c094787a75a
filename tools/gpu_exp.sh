mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu -k "fallback or coarse or candidates" 2>&1 | tail -3
timeout 600 python tools/dbg_m.py 2>&1 | cut -c1-300
timeout 300 python tools/run_stage.py query --reps 3 2>&1 | tail -1
) > gpurun_out/exp.log 2>&1
