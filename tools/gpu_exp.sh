mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for nq in 1 2 64 128 1024; do echo "nq=$nq"; timeout 300 python tools/run_stage.py query --nq $nq --reps 5 2>&1 | tail -1; done
timeout 600 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['recall_at_10'], d['latency_mode'], d['e2e']['ms_per_step'])"
) > gpurun_out/exp.log 2>&1
