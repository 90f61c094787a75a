mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
NRLSH_SCAN_DBG=16 timeout 120 python tools/run_stage.py query --reps 2 > gpurun_out/dbgw_16.log 2>&1
NRLSH_SCAN_NOSORT=1 NRLSH_SCAN_DBG=16 timeout 120 python tools/run_stage.py query --reps 2 > gpurun_out/dbgw_16ns.log 2>&1
