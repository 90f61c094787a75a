mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python -m pytest tests -m gpu -x -q -rf -k "candidates_parity" > gpurun_out/pytest_scan.log 2>&1; echo pytest rc=$? > gpurun_out/rc.txt
for d in 0 4 8; do NRLSH_SCAN_DBG=$d timeout 120 python tools/run_stage.py query --reps 3 > gpurun_out/dbg_$d.log 2>&1; done
