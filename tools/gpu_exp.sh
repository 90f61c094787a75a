# ad-hoc timing experiments (development)
mkdir -p gpurun_out
(for sd in 65536 32768 16384; do echo "samples=$sd"; NRLSH_PILOT_SAMPLES=$sd timeout 300 python tools/run_stage.py query --reps 3 2>&1 | tail -1; done) > gpurun_out/exp.log 2>&1
