mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu -k "build or odd or degenerate or full_size or smoke" 2>&1 | tail -2
timeout 300 python tools/run_stage.py build --reps 3 2>&1 | tail -1
timeout 300 python tools/run_stage.py build --config scale --reps 2 2>&1 | tail -1
timeout 300 python tools/run_stage.py build --config c3 --reps 3 2>&1 | tail -1
) > gpurun_out/exp.log 2>&1
