# scan knobs by environment on the built library: serial-stream stage timings on c4 and scale
# usage: VARS="NRLSH_SCAN_WAVES=2 ..." bash tools/gpu_scan_env.sh   (each VARS entry is one run's env)
O=gpurun_out/scan_env
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
i=0
for V in default $VARS; do
  i=$((i+1))
  if [ "$V" = default ]; then E=""; else E="$V"; fi
  env $E NRLSH_QUERY_SERIAL=1 timeout 300 python tools/run_stage.py query --nq 10000 --reps 3 > $O/serial_$i.log 2>&1
  env $E timeout 300 python tools/run_stage.py query --nq 10000 --reps 4 > $O/two_$i.log 2>&1
  env $E NRLSH_QUERY_SERIAL=1 timeout 300 python tools/run_stage.py query --config scale --nq 8192 --reps 2 > $O/scale_$i.log 2>&1
  echo "[$V] c4 serial $(tail -1 $O/serial_$i.log | grep -o "'scan': [0-9.]*") two-stream $(tail -1 $O/two_$i.log | grep -o "^rep.*wall") scale $(tail -1 $O/scale_$i.log | grep -o "'scan': [0-9.]*") $(tail -1 $O/scale_$i.log | grep -o "^rep.*wall")"
done
if [ -n "$PYTEST_K" ]; then timeout 1200 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log; fi
