"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python tools/launch_summary.py launches.csv OUT.md [--last-step-from KERNEL]
With --last-step-from K, only launches from the last occurrence of kernel K on
are counted (the timed step of `bench.py --steps 1`), so the shares are one
step's.  ncu serialises launches and runs them cold, so compare SHARES with the
CUDA-event stage times of bench.py, not absolute durations.
"""
import collections
import csv
import re
import sys


def main():
    path, out = sys.argv[1], sys.argv[2]
    start_k = None
    if "--last-step-from" in sys.argv:
        start_k = sys.argv[sys.argv.index("--last-step-from") + 1]
    rows = [r for r in csv.reader(open(path)) if len(r) >= 15 and r[0] != "ID"]
    launches = []
    for r in rows:
        if r[12] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[4]).replace("void ", "").replace("nrlsh::", "")
        v = float(r[14].replace(",", ""))
        us = v / 1e3 if r[13] == "ns" else (v * 1e3 if r[13] == "ms" else v)
        launches.append((name, us))
    if start_k:
        idx = max(i for i, (n, _) in enumerate(launches) if n.startswith(start_k))
        launches = launches[idx:]
    agg = collections.OrderedDict()
    for n, us in launches:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    lines = [f"launches: {len(launches)}; total device time {tot / 1e3:.3f} ms (ncu, serialised, "
             "cold caches)", "", "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for n, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {n} | {c} | {us / 1e3:.3f} | {us / tot:.1%} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
