mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -rf -k "build_parity or pp_ or degenerate or m_equals or uniform or odd or errors or full_size" > gpurun_out/pytest_scan.log 2>&1; echo pytest rc=$? > gpurun_out/rc.txt
B="python bench.py --no-scale --no-cpu-baseline --no-latency --no-e2e --steps 10 --warmup 3"
timeout 300 $B > gpurun_out/e_base.json 2>&1
