mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu -k "pruning or exact or rerank_tensor" 2>&1 | tail -2
for srt in 0 1; do echo "SORT=$srt"; if [ $srt = 1 ]; then export NRLSH_GT_SORT=1; fi; timeout 300 python tools/run_stage.py query --reps 3 2>&1 | tail -1; timeout 300 python tools/run_stage.py gtseed --reps 3 2>&1 | tail -1; done
) > gpurun_out/exp.log 2>&1
