# scan ceiling (no appends), pilot stride 128, 16 items per thread
O=gpurun_out/s3a; mkdir -p $O
B="python bench.py --no-scale --no-cpu-baseline --no-e2e --no-latency --steps 10 --warmup 3"
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
NRLSH_SCAN_PROBE=1 timeout 600 $B > $O/probe.json 2> $O/probe.err
NRLSH_PILOT_MAXSTRIDE=128 timeout 600 $B > $O/stride128.json 2> $O/stride128.err
NRLSH_NVCC_EXTRA=-DNRLSH_SCAN_IPT=16 python -c "import __graft_entry__ as g; g.build()" > $O/build16.log 2>&1 || exit 1
timeout 600 $B > $O/ipt16.json 2> $O/ipt16.err
NRLSH_SCAN_PROBE=1 timeout 600 $B > $O/ipt16_probe.json 2> $O/ipt16_probe.err
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
