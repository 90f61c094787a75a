mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -rf -k "build_parity or odd_shapes or full_size_sampled and c4 or pp_build" > gpurun_out/pytest_codes.log 2>&1; echo pytest rc=$? > gpurun_out/rc.txt
: > gpurun_out/e_cw.log
for cw in 16 8; do for st in "3,4" "2,4" "4,2"; do
  echo "cw $cw st $st" >> gpurun_out/e_cw.log
  NRLSH_CODES_CW=$cw NRLSH_CODES_STAGES=$st timeout 120 python tools/run_stage.py build --reps 3 2>&1 | tail -1 >> gpurun_out/e_cw.log
done; done
echo "scale cw16" >> gpurun_out/e_cw.log
timeout 200 python tools/run_stage.py build --config scale --reps 2 2>&1 | tail -1 >> gpurun_out/e_cw.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k3_codes" -c 1 -o gpurun_out/prof_codes python tools/run_stage.py build --reps 1 > gpurun_out/ncu_codes.log 2>&1
echo ncu rc=$? >> gpurun_out/rc.txt
