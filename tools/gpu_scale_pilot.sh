O=gpurun_out/${1:-sp}; mkdir -p $O
B="python bench.py --config scale --no-scale --no-cpu-baseline --no-e2e --no-latency --steps 3 --warmup 2"
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -rf -k "streams_identical" > $O/pytest.log 2>&1; echo pytest rc=$? >> $O/rc.txt
timeout 900 $B > $O/s128.json 2> $O/s128.err; echo b1 rc=$? >> $O/rc.txt
NRLSH_PILOT_MAXSTRIDE=256 timeout 900 $B > $O/s256.json 2> $O/s256.err; echo b2 rc=$? >> $O/rc.txt
