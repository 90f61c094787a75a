# ad-hoc timing experiments (development)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for m in 0 2 3; do echo "dbg=$m"; NRLSH_GT_DBG=$m timeout 300 python tools/run_stage.py gtseed --reps 3 2>&1 | tail -2; done > gpurun_out/exp.log 2>&1
