O=gpurun_out/${1:-lat2}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/latency_probe.py --nq 1 > $O/lat1.log 2>&1
timeout 300 python tools/latency_probe.py --nq 16 > $O/lat16.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -rf -k "rerank or query_parity or small or odd or exact" > $O/pytest.log 2>&1; echo pytest rc=$? >> $O/rc.txt
timeout 600 python bench.py --no-scale --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo bench rc=$? >> $O/rc.txt
