mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_step.csv python bench.py --no-scale --no-cpu-baseline --no-latency --no-e2e --steps 1 --warmup 1 > gpurun_out/ncu_launch.log 2>&1
echo rc=$? > gpurun_out/rc.txt
