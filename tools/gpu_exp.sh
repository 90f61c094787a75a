mkdir -p gpurun_out
(for tp in 0 1; do echo "TWOPASS=$tp"; if [ $tp = 1 ]; then export NRLSH_RERANK_TWOPASS=1; fi
timeout 300 python tools/run_stage.py query --reps 3 2>&1 | tail -1; timeout 300 python tools/run_stage.py query --bits 32 --reps 3 2>&1 | tail -1; timeout 300 python tools/run_stage.py query --config scale --nq 1024 --reps 2 2>&1 | tail -1; done
unset NRLSH_RERANK_TWOPASS
NRLSH_RERANK_TWOPASS=1 timeout 900 python -m pytest tests -x -q -m gpu -k "rerank_tensor or tile_pruning or query_parity" 2>&1 | tail -2
) > gpurun_out/exp.log 2>&1
