"""Hot SASS lines of one kernel from an ncu report (--page source), with the
dominant stall reasons per line.
usage: python tools/ncu_source.py REPORT KERNEL_REGEX [min_share] [--range A B]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
thr = float(sys.argv[3]) if len(sys.argv) > 3 and not sys.argv[3].startswith("--") else 0.008
rng = None
if "--range" in sys.argv:
    i = sys.argv.index("--range")
    rng = (int(sys.argv[i + 1]), int(sys.argv[i + 2]))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr_i]
body = []
for r in rows[hdr_i + 1:]:
    if not r or r[0] in ("Address", "Kernel Name"):
        break
    body.append(r)
i_s = h.index("Warp Stall Sampling (All Samples)")
i_e = h.index("Instructions Executed")
i_t = h.index("Thread Instructions Executed")
stall_cols = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
f = lambda x: float(x or 0)
tot = sum(f(x[i_s]) for x in body)
ti = sum(f(x[i_e]) for x in body)
print(f"samples {tot:.0f}  warp-instructions {ti:.3g}")
for idx, x in enumerate(body):
    sv = f(x[i_s])
    if (rng and rng[0] <= idx <= rng[1]) or (not rng and sv > tot * thr):
        st = sorted(((f(x[i]), n) for i, n in stall_cols), reverse=True)[:2]
        sts = " ".join(f"{n}:{v:.0f}" for v, n in st if v > 0)
        act = f(x[i_t]) / max(1.0, f(x[i_e]))
        print(f"{idx:5d} {sv / tot:6.1%} {x[i_e]:>10} a{act:4.1f} {x[1][:70]:70s} {sts}")
