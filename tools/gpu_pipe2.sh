O=gpurun_out/${1:-pipe2}; mkdir -p $O
B="python bench.py --no-scale --no-cpu-baseline --no-e2e --no-latency --steps 10 --warmup 3"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? > $O/rc.txt
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest.log 2>&1; echo pytest rc=$? >> $O/rc.txt
timeout 600 $B > $O/s2.json 2> $O/s2.err; echo b1 rc=$? >> $O/rc.txt
NRLSH_QUERY_STREAMS=3 timeout 600 $B > $O/s3.json 2> $O/s3.err; echo b2 rc=$? >> $O/rc.txt
NRLSH_GT_BATCH=2048 timeout 600 $B > $O/gt2048.json 2> $O/gt2048.err; echo b3 rc=$? >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > $O/full.json 2> $O/full.err; echo b4 rc=$? >> $O/rc.txt
