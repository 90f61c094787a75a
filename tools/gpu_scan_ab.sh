# A/B of scan variants on c4 (10,000 queries) and scale (8,192): each variant is a source
# file under build/exp plus nvcc -D flags; serial-stream and two-stream stage timings.
# usage: bash tools/gpu_scan_ab.sh "name:file:flags" ...   (the last variant stays built)
O=gpurun_out/scan_ab
mkdir -p $O
for V in "$@"; do
  NAME=${V%%:*}; REST=${V#*:}; FILE=${REST%%:*}; FLAGS=${REST#*:}
  cp build/exp/$FILE paper_1809_08782_b200/csrc/query_kernels.cu
  NRLSH_NVCC_EXTRA="$FLAGS" timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build_$NAME.log 2>&1 || { echo "build $NAME failed"; continue; }
  NRLSH_QUERY_SERIAL=1 timeout 300 python tools/run_stage.py query --nq 10000 --reps 3 > $O/serial_$NAME.log 2>&1
  timeout 300 python tools/run_stage.py query --nq 10000 --reps 4 > $O/two_$NAME.log 2>&1
  NRLSH_QUERY_SERIAL=1 timeout 300 python tools/run_stage.py query --config scale --nq 8192 --reps 2 > $O/scale_$NAME.log 2>&1
  echo "$NAME c4 serial $(tail -1 $O/serial_$NAME.log | grep -o "'scan': [0-9.]*") two-stream $(tail -1 $O/two_$NAME.log | grep -o "^rep.*wall") scale $(tail -1 $O/scale_$NAME.log | grep -o "'scan': [0-9.]*")"
done
if [ -n "$PYTEST_K" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log; fi
