mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu -k "rerank or query" 2>&1 | tail -2
for nq in 1 128 1024; do echo "nq=$nq"; timeout 300 python tools/run_stage.py query --nq $nq --reps 3 2>&1 | tail -1; done
for T in 524288 1048576; do echo "T=$T"; timeout 300 python tools/run_stage.py query --T $T --reps 2 2>&1 | tail -1; done
) > gpurun_out/exp.log 2>&1
