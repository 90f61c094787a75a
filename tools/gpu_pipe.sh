O=gpurun_out/${1:-pipe}; mkdir -p $O
B="python bench.py --no-scale --no-cpu-baseline --no-e2e --no-latency --steps 10 --warmup 3"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? > $O/rc.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest.log 2>&1; echo pytest rc=$? >> $O/rc.txt
timeout 600 $B > $O/pipe.json 2> $O/pipe.err; echo b1 rc=$? >> $O/rc.txt
NRLSH_QUERY_SERIAL=1 timeout 600 $B > $O/serial.json 2> $O/serial.err; echo b2 rc=$? >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > $O/full.json 2> $O/full.err; echo b3 rc=$? >> $O/rc.txt
