mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/run_stage.py gtseed --reps 3 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['latency_mode'][0]['ms_median'])"
) > gpurun_out/exp.log 2>&1
