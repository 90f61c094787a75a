"""Hot SASS lines of one kernel from an ncu report (--page source).
usage: python tools/ncu_source.py REPORT KERNEL_REGEX [min_share]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.008
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# the report may hold several kernels: keep the first block after its header
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr_i]
body = []
for r in rows[hdr_i + 1:]:
    if not r or r[0] in ("Address", "Kernel Name"):
        break
    body.append(r)
i_s = h.index("Warp Stall Sampling (All Samples)")
i_e = h.index("Instructions Executed")
tot = sum(float(x[i_s] or 0) for x in body)
ti = sum(float(x[i_e] or 0) for x in body)
print(f"samples {tot:.0f}  instructions {ti:.3g}")
for idx, x in enumerate(body):
    sv = float(x[i_s] or 0)
    if sv > tot * thr:
        print(f"{idx:5d} {sv / tot:6.1%} {x[i_e]:>10} {x[1][:90]}")
