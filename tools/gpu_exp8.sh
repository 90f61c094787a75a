mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
: > gpurun_out/e_stages.log
for cfg in "3,4" "2,4" "2,6" "4,3" "3,3" "2,3" "4,2"; do
  echo "cfg $cfg" >> gpurun_out/e_stages.log
  NRLSH_CODES_STAGES=$cfg timeout 120 python tools/run_stage.py build --reps 3 >> gpurun_out/e_stages.log 2>&1
done
echo "cfg scale" >> gpurun_out/e_stages.log
timeout 200 python tools/run_stage.py build --config scale --reps 2 >> gpurun_out/e_stages.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k3_codes" -c 1 -o gpurun_out/prof_codes python tools/run_stage.py build --reps 1 > gpurun_out/ncu_codes.log 2>&1
echo ncu rc=$? > gpurun_out/rc.txt
