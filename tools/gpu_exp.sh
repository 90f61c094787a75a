mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu -k "exact or seeded or pruning or pair" 2>&1 | tail -2
timeout 300 python tools/run_stage.py gtseed --reps 3 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline --no-latency 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['recall_at_10'], {k:round(v['ms_per_step'],3) for k,v in d['stage_ms_per_step'].items()})"
) > gpurun_out/exp.log 2>&1
