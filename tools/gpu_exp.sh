# ad-hoc timing experiments (development)
mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "coarse or fallback or candidates_parity or full_size" 2>&1 | tail -5
for cfg in "32 128" "32 256" "64 23404"; do set -- $cfg; echo "bits=$1 T=$2"; timeout 300 python tools/run_stage.py query --bits $1 --T $2 --reps 2 2>&1 | tail -1; done) > gpurun_out/exp.log 2>&1
