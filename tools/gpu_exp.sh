# ad-hoc timing experiments (development)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for m in 0 4; do echo "dbg=$m"; NRLSH_SCAN_CLK=1 NRLSH_SCAN_DBG=$m timeout 300 python tools/run_stage.py query --reps 2 2>&1 | tail -3; done > gpurun_out/exp.log 2>&1
