# A/B of scan variants on c4 (10,000 queries): each variant is a source file under
# build/exp plus nvcc -D flags; serial-stream and two-stream stage timings.
# usage: bash tools/gpu_scan_ab.sh "name:file:flags" ...
O=gpurun_out/scan_ab
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
for V in "$@"; do
  NAME=${V%%:*}; REST=${V#*:}; FILE=${REST%%:*}; FLAGS=${REST#*:}
  cp build/exp/$FILE paper_1809_08782_b200/csrc/query_kernels.cu
  NRLSH_NVCC_EXTRA="$FLAGS" timeout 600 python -c "import __graft_entry__ as g; g.build()" > $O/build_$NAME.log 2>&1 || { echo "build $NAME failed" >> $O/rc.txt; continue; }
  NRLSH_QUERY_SERIAL=1 timeout 300 python tools/run_stage.py query --nq 10000 --reps 4 > $O/serial_$NAME.log 2>&1; echo "$NAME serial rc=$?" >> $O/rc.txt
  timeout 300 python tools/run_stage.py query --nq 10000 --reps 4 > $O/two_$NAME.log 2>&1; echo "$NAME two rc=$?" >> $O/rc.txt
done
# leave the last variant built; parity on it
timeout 900 python -m pytest tests -m gpu -x -q -k "candidates or query_parity or forced_fallback or odd_shapes or scan_bound" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
tail -3 $O/pytest.log
for f in $O/serial_*.log $O/two_*.log; do echo $f; tail -2 $f | cut -c1-700; done
