mkdir -p gpurun_out
(timeout 900 python -m pytest tests -x -q -m gpu -k "build or odd or degenerate or full_size or smoke or uniform" 2>&1 | tail -2
for cf in 2,4 2,2; do echo "CFG=$cf"; NRLSH_CODES_CFG=$cf timeout 600 python bench.py --no-cpu-baseline --no-latency --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], {k:round(v['ms_per_step'],3) for k,v in d['stage_ms_per_step'].items() if k in ('norms','partition','scatter','codes')})"; done
) > gpurun_out/exp.log 2>&1
