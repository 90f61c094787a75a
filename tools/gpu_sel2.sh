O=gpurun_out/${1:-sel2}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? > $O/rc.txt
timeout 300 python tools/latency_probe.py --nq 1 > $O/lat1.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest.log 2>&1; echo pytest rc=$? >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo bench rc=$? >> $O/rc.txt
