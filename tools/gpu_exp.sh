mkdir -p gpurun_out
(for st in 3 2; do echo "GT_STAGES=$st"; export NRLSH_GT_STAGES=$st; timeout 300 python tools/run_stage.py query --reps 3 2>&1 | tail -1; timeout 300 python tools/run_stage.py gtseed --reps 3 2>&1 | tail -1; done
) > gpurun_out/exp.log 2>&1
