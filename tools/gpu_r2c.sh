# TC scan v2: parity first, then the bench step
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests -m gpu -x -q -rf -k "candidates_parity or test_query_parity or coarse or forced_fallback" > gpurun_out/pytest_scan.log 2>&1; echo pytest rc=$? > gpurun_out/rc.txt
timeout 300 python bench.py --no-scale --no-cpu-baseline --no-latency --no-e2e --steps 10 --warmup 3 > gpurun_out/bench_tc.json 2> gpurun_out/bench_tc.err; echo bench rc=$? >> gpurun_out/rc.txt
NRLSH_SCAN_TC=0 timeout 300 python bench.py --no-scale --no-cpu-baseline --no-latency --no-e2e --steps 10 --warmup 3 > gpurun_out/bench_pc.json 2> gpurun_out/bench_pc.err; echo bench rc=$? >> gpurun_out/rc.txt
