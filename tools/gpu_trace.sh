O=gpurun_out/${1:-tr}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
NRLSH_BUILD_TRACE=1 timeout 300 python tools/run_stage.py build --reps 4 > $O/trace_c4.log 2>&1
NRLSH_BUILD_TRACE=1 timeout 300 python tools/run_stage.py build --config scale --reps 3 > $O/trace_scale.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > $O/bench.json 2> $O/bench.err; echo bench rc=$? >> $O/rc.txt
