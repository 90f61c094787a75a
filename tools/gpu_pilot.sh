O=gpurun_out/${1:-pilot}; mkdir -p $O
B="python bench.py --no-scale --no-cpu-baseline --no-e2e --no-latency --steps 10 --warmup 3"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? > $O/rc.txt
timeout 900 python -m pytest tests -m gpu -x -q -rf -k "candidates or query_parity or full_size or fallback or coarse or pp_ or degenerate or odd" > $O/pytest.log 2>&1; echo pytest rc=$? >> $O/rc.txt
timeout 600 $B > $O/qp4.json 2> $O/qp4.err; echo b1 rc=$? >> $O/rc.txt
NRLSH_PILOT_QP=2 timeout 600 $B > $O/qp2.json 2> $O/qp2.err; echo b2 rc=$? >> $O/rc.txt
NRLSH_PILOT_QP=1 timeout 600 $B > $O/qp1.json 2> $O/qp1.err; echo b3 rc=$? >> $O/rc.txt
