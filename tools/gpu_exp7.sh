mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -rf -k "build_parity or odd_shapes or full_size or test_query_parity or pp_build or rerank_tensor" > gpurun_out/pytest_codes.log 2>&1; echo pytest rc=$? > gpurun_out/rc.txt
B="python bench.py --no-scale --no-cpu-baseline --no-latency --no-e2e --steps 10 --warmup 3"
timeout 300 $B > gpurun_out/e_codes.json 2>&1
timeout 200 python tools/run_stage.py build --config scale --reps 2 > gpurun_out/e_scale_build.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k3_codes" -c 1 -o gpurun_out/prof_codes python tools/run_stage.py build --reps 1 > gpurun_out/ncu_codes.log 2>&1
echo ncu rc=$? >> gpurun_out/rc.txt
