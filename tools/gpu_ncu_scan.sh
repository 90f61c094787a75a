# ncu --set full of one k6_scan launch on c4 and on scale (source view imported)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 300 python tools/run_stage.py query --reps 1 > gpurun_out/plain_query.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k6_scan" -c 1 -o gpurun_out/prof_scan python tools/run_stage.py query --reps 1 > gpurun_out/ncu_scan.log 2>&1
echo ncu rc=$? > gpurun_out/rc.txt
if [ -n "$SCALE" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k6_scan" -c 1 -o gpurun_out/prof_scan_scale python tools/run_stage.py query --config scale --nq 4096 --reps 1 > gpurun_out/ncu_scan_scale.log 2>&1
echo ncu scale rc=$? >> gpurun_out/rc.txt
fi
