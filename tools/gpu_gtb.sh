O=gpurun_out/${1:-gtb}; mkdir -p $O
B="python bench.py --no-scale --no-cpu-baseline --no-e2e --no-latency --steps 10 --warmup 3"
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for gb in 1024 2048 4096 10000; do NRLSH_GT_BATCH=$gb timeout 600 $B > $O/gt$gb.json 2> $O/gt$gb.err; done
echo done > $O/rc.txt
