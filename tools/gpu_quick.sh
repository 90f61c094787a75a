# quick GPU check: parity tests + stage timings on c4 (used during development)
set -x
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? > gpurun_out/rc.txt
timeout 600 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$? >> gpurun_out/rc.txt
timeout 300 python tools/run_stage.py query --reps 3 > gpurun_out/stage_query.log 2>&1; echo q rc=$? >> gpurun_out/rc.txt
timeout 300 python tools/run_stage.py gt --reps 3 > gpurun_out/stage_gt.log 2>&1; echo gt rc=$? >> gpurun_out/rc.txt
timeout 300 python tools/run_stage.py gtseed --reps 3 > gpurun_out/stage_gtseed.log 2>&1; echo gts rc=$? >> gpurun_out/rc.txt
timeout 300 python tools/run_stage.py build --reps 3 > gpurun_out/stage_build.log 2>&1; echo b rc=$? >> gpurun_out/rc.txt
