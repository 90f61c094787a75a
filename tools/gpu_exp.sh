mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu -k "both_scans" 2>&1 | tail -2
for im in 1; do echo "IMMA=$im"; NRLSH_SCAN_IMMA=$im timeout 300 python tools/run_stage.py query --reps 3 2>&1 | tail -1; NRLSH_SCAN_IMMA=$im timeout 300 python tools/run_stage.py query --bits 32 --reps 3 2>&1 | tail -1; done
) > gpurun_out/exp.log 2>&1
