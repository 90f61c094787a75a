mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
B="python bench.py --no-scale --no-cpu-baseline --no-latency --no-e2e --steps 10 --warmup 3"
NRLSH_PILOT_SAMPLES=16384 NRLSH_PILOT_MAXSTRIDE=256 timeout 300 $B > gpurun_out/e_ps16k.json 2>&1
NRLSH_PILOT_SAMPLES=24576 NRLSH_PILOT_MAXSTRIDE=256 timeout 300 $B > gpurun_out/e_ps24k.json 2>&1
