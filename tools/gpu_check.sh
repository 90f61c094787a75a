# smoke, GPU tests, bench line (with the scale sub-record), build trace.
# usage: bash tools/gpu_check.sh <tag> [pytest -k expression]
O=gpurun_out/${1:-chk}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$? > $O/rc.txt
if [ -n "$2" ]; then timeout 1500 python -m pytest tests -m gpu -q -rf -k "$2" > $O/pytest.log 2>&1
else timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest.log 2>&1; fi; echo pytest rc=$? >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo bench rc=$? >> $O/rc.txt
NRLSH_BUILD_TRACE=1 timeout 300 python tools/run_stage.py build --reps 3 > $O/trace_c4.log 2>&1
