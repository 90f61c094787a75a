# experiments: Xpad on/off (c4 step), pilot sample count at scale
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
B="python bench.py --no-scale --no-cpu-baseline --no-latency --no-e2e --steps 10 --warmup 3"
timeout 300 $B > gpurun_out/exp_xpad_on.json 2>&1
NRLSH_NO_XPAD=1 timeout 300 $B > gpurun_out/exp_xpad_off.json 2>&1
for ns in 32768 65536 131072; do
  NRLSH_PILOT_SAMPLES=$ns timeout 300 python bench.py --config scale --no-cpu-baseline --no-latency --no-e2e --steps 2 --warmup 2 > gpurun_out/exp_scale_ps$ns.json 2>&1
done
