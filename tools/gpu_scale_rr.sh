O=gpurun_out/${1:-srr}; mkdir -p $O
B="python bench.py --config scale --no-scale --no-cpu-baseline --no-e2e --no-latency --steps 3 --warmup 2"
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 $B > $O/default.json 2> $O/default.err; echo b1 rc=$? >> $O/rc.txt
NRLSH_RERANK_TC=1 timeout 900 $B > $O/tc.json 2> $O/tc.err; echo b2 rc=$? >> $O/rc.txt
