O=gpurun_out/${1:-sel}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? > $O/rc.txt
timeout 900 python -m pytest tests -m gpu -x -q -rf -k "candidates or query_parity or full_size or fallback or coarse or degenerate or rerank" > $O/pytest.log 2>&1; echo pytest rc=$? >> $O/rc.txt
timeout 600 python bench.py --no-scale --no-cpu-baseline --no-e2e --no-latency --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo bench rc=$? >> $O/rc.txt
timeout 900 python bench.py --sweep c4 --scheme uniform --sweep-parts 32,128 --sweep-out $O/sweep_c4_uniform_m32_m128.json > $O/sweep_u.log 2>&1; echo su rc=$? >> $O/rc.txt
timeout 900 python bench.py --sweep c4 --scheme percentile --sweep-parts 32,128 --sweep-out $O/sweep_c4_percentile_m32_m128.json > $O/sweep_p.log 2>&1; echo sp rc=$? >> $O/rc.txt
