# scan knobs by environment on the built library: serial-stream stage timings
O=gpurun_out/scan_env
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
for D in ${C4_DENSE:-default}; do
  if [ $D = default ]; then unset NRLSH_SCAN_DENSE; else export NRLSH_SCAN_DENSE=$D; fi
  NRLSH_QUERY_SERIAL=1 timeout 300 python tools/run_stage.py query --nq 10000 --reps 3 > $O/serial_$D.log 2>&1
  echo "c4 dense=$D $(tail -1 $O/serial_$D.log | grep -o "'scan': [0-9.]*") $(tail -1 $O/serial_$D.log | grep -o "'select': [0-9.]*")"
done
for D in ${SCALE_DENSE:-default}; do
  if [ $D = default ]; then unset NRLSH_SCAN_DENSE; else export NRLSH_SCAN_DENSE=$D; fi
  NRLSH_QUERY_SERIAL=1 timeout 300 python tools/run_stage.py query --config scale --nq 8192 --reps 2 > $O/scale_$D.log 2>&1
  echo "scale dense=$D $(tail -1 $O/scale_$D.log | grep -o "'scan': [0-9.]*") $(tail -1 $O/scale_$D.log | grep -o "^rep.*wall")"
done
unset NRLSH_SCAN_DENSE
timeout 300 python tools/run_stage.py query --nq 10000 --reps 4 > $O/two.log 2>&1; tail -1 $O/two.log | cut -c1-400
if [ -n "$PYTEST_K" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log; fi
if [ -n "$OLD" ]; then
  cp build/exp/$OLD paper_1809_08782_b200/csrc/query_kernels.cu
  python -c "import __graft_entry__ as g; g.build()" > $O/build_old.log 2>&1
  NRLSH_QUERY_SERIAL=1 timeout 300 python tools/run_stage.py query --config scale --nq 8192 --reps 2 > $O/scale_old.log 2>&1
  echo "scale old $(tail -1 $O/scale_old.log | grep -o "'scan': [0-9.]*") $(tail -1 $O/scale_old.log | grep -o "^rep.*wall")"
fi
