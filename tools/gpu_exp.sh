mkdir -p gpurun_out
(for dv in 50 200 800; do echo "DIV=$dv"; export NRLSH_GT_SPLIT_DIV=$dv; timeout 300 python tools/run_stage.py gt --config scale --nq 1024 --reps 2 2>&1 | tail -1; timeout 300 python tools/run_stage.py gtseed --config scale --nq 1024 --reps 2 2>&1 | tail -1; timeout 300 python tools/run_stage.py gt --config c3 --nq 1024 --reps 2 2>&1 | tail -1; done
) > gpurun_out/exp.log 2>&1
