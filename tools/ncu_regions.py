"""Per-SASS-line executed-instruction and stall-sample dump of one kernel from an ncu
report, grouped into runs of lines with the same execution count (loop bodies).
usage: python tools/ncu_regions.py REPORT KERNEL_REGEX [out_lines.txt]"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

rep, kre = sys.argv[1], sys.argv[2]
def page(p):
    return subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", "--kernel-name", f"regex:{kre}",
                           "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(page("raw"))))
h = rows[0]
for name in ("gpu__time_duration.sum", "smsp__inst_executed.sum",
             "smsp__issue_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
             "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
             "launch__grid_size", "dram__bytes_read.sum", "dram__bytes_write.sum"):
    if name in h:
        print(f"{name:62s} {rows[2][h.index(name)]}")
rows = list(csv.reader(io.StringIO(page("source"))))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
body = [r for r in rows[hi + 1:] if r and r[0] not in ("Address", "Kernel Name")]
ie, isrc, iss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
f = lambda x: float(x or 0)
cnt = [f(r[ie]) / 1e6 for r in body]
st = [f(r[iss]) for r in body]
txt = [r[isrc].strip() for r in body]
if len(sys.argv) > 3:
    with open(sys.argv[3], "w") as o:
        for i in range(len(body)):
            o.write(f"{i:5d} {cnt[i]:8.2f} {st[i]:7.0f} {txt[i][:90]}\n")
tot, tst = sum(cnt), sum(st)
ops = Counter()
for t, n in zip(txt, cnt):
    op = re.sub(r"^@!?U?P\d+\s+", "", t).split()[0] if t else ""
    ops[op.split(".")[0]] += n
print(f"warp-instructions {tot:.1f}M; by opcode: " + ", ".join(f"{k} {v:.1f}" for k, v in ops.most_common(12)))
prev, start = None, 0
for i, c in enumerate(cnt + [None]):
    if prev is None:
        prev, start = c, i
        continue
    if c is None or abs(c - prev) > 0.02 * max(prev, 0.05):
        n, s = sum(cnt[start:i]), sum(st[start:i])
        if n > tot * 0.006 or s > tst * 0.01:
            print(f"{start:5d}-{i - 1:5d} x{prev:6.2f}M  instr {n:7.1f}M ({n / tot:5.1%})  stalls {s / tst:5.1%}   {txt[start][:50]}")
        prev, start = c, i
