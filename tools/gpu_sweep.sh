# bench line + per-budget sweeps (queries/s, recall@k) of the BASELINE configs
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$? > gpurun_out/rc.txt
timeout 1500 python bench.py --sweep ${SWEEP:-tiny,c2,c3,c4} --sweep-out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1; echo sweep rc=$? >> gpurun_out/rc.txt
