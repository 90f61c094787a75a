mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu -k "both_scans or forced_fallback" 2>&1 | tail -2
for tc in 0 1; do echo "SCAN_TC=$tc"; NRLSH_SCAN_TC=$tc timeout 300 python tools/run_stage.py query --reps 3 2>&1 | tail -1; NRLSH_SCAN_TC=$tc timeout 300 python tools/run_stage.py query --bits 32 --reps 3 2>&1 | tail -1; done
echo NOSORT; NRLSH_SCAN_TC_NOSORT=1 NRLSH_SCAN_TC=1 timeout 300 python tools/run_stage.py query --reps 3 2>&1 | tail -1
) > gpurun_out/exp.log 2>&1
export NRLSH_SCAN_TC=1; NCU_STAGE=query NCU_K="k6_scan_mma|expand_groups|scan_tile_lists|sort_by_active" NCU_C=4 bash tools/gpu_ncu_one.sh
