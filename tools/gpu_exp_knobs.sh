O=gpurun_out/${1:-knobs}; mkdir -p $O
B="python bench.py --no-scale --no-cpu-baseline --no-e2e --no-latency --steps 10 --warmup 3"
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 $B > $O/base.json 2> $O/base.err
NRLSH_GT_NT=128 timeout 600 $B > $O/nt128.json 2> $O/nt128.err
NRLSH_QUERY_STREAMS=3 timeout 600 $B > $O/s3.json 2> $O/s3.err
NRLSH_RERANK_TC_KS=256 timeout 600 $B > $O/ks256.json 2> $O/ks256.err
NRLSH_RERANK_TC_KS=1024 timeout 600 $B > $O/ks1024.json 2> $O/ks1024.err
timeout 600 $B > $O/base2.json 2> $O/base2.err
echo done > $O/rc.txt
