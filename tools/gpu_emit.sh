O=gpurun_out/${1:-emit}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python tools/latency_probe.py --nq 1 > $O/lat1.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -rf -k "candidates or query_parity or small or streams or full_size" > $O/pytest.log 2>&1; echo pytest rc=$? >> $O/rc.txt
timeout 900 python bench.py --config scale --no-scale --no-cpu-baseline --no-e2e --no-latency --steps 3 --warmup 2 > $O/scale.json 2> $O/scale.err; echo b1 rc=$? >> $O/rc.txt
timeout 600 python bench.py --no-scale --no-cpu-baseline --no-e2e --no-latency --steps 10 --warmup 3 --budget-permille 1 > $O/c4_01.json 2> $O/c4_01.err; echo b2 rc=$? >> $O/rc.txt
