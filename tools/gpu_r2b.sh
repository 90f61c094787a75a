# PP parity + sweeps (NEXT-2 uniform vs percentile, NEXT-4 per-sub-dataset projections) + scale pilot stride
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -q -rf -k "pp_ or headline or full_size_sampled or path_selection or multi_pair" > gpurun_out/pytest_pp.log 2>&1; echo pytest rc=$? > gpurun_out/rc.txt
timeout 600 python bench.py --sweep c3,c4 --proj per_partition --sweep-out gpurun_out/sweep_pp.json > gpurun_out/sweep_pp.log 2>&1; echo pp rc=$? >> gpurun_out/rc.txt
timeout 600 python bench.py --sweep c3,c4 --sweep-out gpurun_out/sweep_shared.json > gpurun_out/sweep_shared.log 2>&1; echo shared rc=$? >> gpurun_out/rc.txt
timeout 600 python bench.py --sweep c3 --scheme uniform --sweep-parts 32,128 --sweep-out gpurun_out/sweep_uniform_c3.json > gpurun_out/sweep_uni.log 2>&1; echo uni rc=$? >> gpurun_out/rc.txt
timeout 600 python bench.py --sweep c3 --scheme percentile --sweep-parts 32,128 --sweep-out gpurun_out/sweep_percentile_c3.json > gpurun_out/sweep_pct.log 2>&1; echo pct rc=$? >> gpurun_out/rc.txt
for st in 128 512; do
  NRLSH_PILOT_MAXSTRIDE=$st timeout 300 python bench.py --config scale --no-cpu-baseline --no-latency --no-e2e --steps 2 --warmup 2 > gpurun_out/exp_scale_st$st.json 2>&1
done
NRLSH_RERANK_TC=1 timeout 300 python bench.py --config scale --no-cpu-baseline --no-latency --no-e2e --steps 2 --warmup 2 > gpurun_out/exp_scale_rtc.json 2>&1
