mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -rf -k "candidates_parity or test_query_parity or forced_fallback or coarse or headline or full_size or multi_pair or dense or pp_cand" > gpurun_out/pytest_sel.log 2>&1; echo pytest rc=$? > gpurun_out/rc.txt
B="python bench.py --no-scale --no-cpu-baseline --no-latency --no-e2e --steps 10 --warmup 3"
timeout 300 $B > gpurun_out/e_sel.json 2>&1
timeout 600 python bench.py --config scale --no-cpu-baseline --no-latency --no-e2e --steps 3 --warmup 2 > gpurun_out/e_scale.json 2>&1
