O=gpurun_out/${1:-lat}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/latency_probe.py --nq 1 > $O/lat1.log 2>&1
timeout 300 python tools/latency_probe.py --nq 16 > $O/lat16.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/lat_launches.csv python tools/latency_probe.py --nq 1 --reps 1 > $O/ncu.log 2>&1
NRLSH_BUILD_TRACE=1 timeout 300 python tools/run_stage.py build --reps 3 > $O/trace_c4.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e --no-scale --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo bench rc=$? >> $O/rc.txt
