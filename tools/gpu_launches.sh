mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python tools/run_stage.py query --reps 1 > gpurun_out/ncu_launch.log 2>&1
echo rc=$? > gpurun_out/rc.txt
