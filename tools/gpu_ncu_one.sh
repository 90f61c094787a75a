# ncu --set full of one kernel class from a run_stage.py invocation:
#   NCU_STAGE=gt NCU_K=gt_filter_tc NCU_C=1 bash tools/gpu_ncu_one.sh
set -x
mkdir -p gpurun_out
timeout 300 python tools/run_stage.py ${NCU_STAGE} --reps 1 ${NCU_ARGS} > gpurun_out/plain_${NCU_STAGE}.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K}" -c ${NCU_C:-1} -o gpurun_out/prof_${NCU_STAGE} python tools/run_stage.py ${NCU_STAGE} --reps 1 ${NCU_ARGS} > gpurun_out/ncu_${NCU_STAGE}.log 2>&1
echo ncu rc=$? > gpurun_out/rc.txt
