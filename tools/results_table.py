"""Markdown tables for BASELINE.md §4 from a bench line and a sweep JSON.
usage: python tools/results_table.py BENCH_JSON SWEEP_JSON"""
import json
import sys

bench = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
rows = json.load(open(sys.argv[2]))
print(f"Bench line (c4, 64-bit, m=128, T=1%, step = build + 10,000 queries + exact top-10): "
      f"{bench['value']:,.0f} queries/s, {bench['ms_per_step']:.2f} ms/step, recall@10 "
      f"{bench.get('recall_at_10', float('nan')):.4f}; e2e (host buffers) "
      f"{bench['e2e']['value']:,.0f} queries/s.\n")
print("| config | L_h | m | T (share of n) | queries/s | recall@k | build (ms) |")
print("|---|---|---|---|---|---|---|")
for r in rows:
    rk = f"{r['recall_at_k']:.4f}" + (f" (@10: {r['recall_at_10']:.4f})" if "recall_at_10" in r else "")
    print(f"| {r['config']} | {r['code_bits']} | {r['num_parts']} | {r['probe_budget']:,} "
          f"({100 * r['budget_frac']:.3g}%) | {r['queries_per_s']:,.0f} | {rk} | {r['build_ms']:.2f} |")
