"""Summarise ncu reports (.ncu-rep) into a compact markdown table + JSON.

usage: python tools/ncu_summary.py OUT_PREFIX REPORT [REPORT ...]
Writes OUT_PREFIX.md (one row per profiled launch: duration, DRAM bytes, DRAM %,
L2 hit rate, SM / pipe utilisation, occupancy, registers, top stall reasons)
and OUT_PREFIX.json (the same numbers, machine-readable; `bench.py` reads the
per-kernel DRAM bytes from profiles/traffic.json for the `traffic` key).
"""
import csv
import io
import json
import re
import subprocess
import sys

FIELDS = {
    "dur_us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "mem_pct": "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "occ_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "alu_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "lsu_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "xu_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fp64_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "tensor_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm_ghz": "sm__cycles_elapsed.avg.per_second",
}


def _num(s):
    try:
        return float(s.replace(",", ""))
    except Exception:
        return None


def read_report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    idx = {name: i for i, name in enumerate(h)}
    res = []
    for r in rows[2:]:
        d = {"kernel": re.sub(r"\(.*", "", r[idx["Kernel Name"]]).replace("void ", ""),
             "grid": r[idx["Grid Size"]], "block": r[idx["Block Size"]]}
        for k, f in FIELDS.items():
            if f in idx:
                v = _num(r[idx[f]])
                u = units[idx[f]]
                if v is not None and k == "dur_us":
                    v = v / 1e3 if u == "ns" else (v * 1e3 if u == "ms" else v)
                if v is not None and k in ("dram_rd", "dram_wr"):
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                    v = v * scale
                d[k] = v
        stalls = {}
        for i, name in enumerate(h):
            m = re.match(r"smsp__pcsamp_warps_issue_stalled_([a-z_]+)$", name)
            if m and not name.endswith("_not_issued"):
                v = _num(r[i])
                if v:
                    stalls[m.group(1)] = v
        tot = sum(stalls.values()) or 1.0
        d["stalls"] = {k: round(v / tot, 3) for k, v in
                       sorted(stalls.items(), key=lambda x: -x[1])[:4]}
        res.append(d)
    return res


def main():
    prefix, reps = sys.argv[1], sys.argv[2:]
    allr = []
    for p in reps:
        for d in read_report(p):
            d["report"] = p.split("/")[-1]
            allr.append(d)
    with open(prefix + ".json", "w") as f:
        json.dump(allr, f, indent=1)
    cols = ["kernel", "dur_us", "dram_rd", "dram_wr", "dram_pct", "l2_hit", "sm_pct", "alu_pct",
            "fma_pct", "lsu_pct", "fp64_pct", "tensor_pct", "occ_pct", "regs", "sm_ghz"]
    lines = ["| " + " | ".join(cols + ["top stalls"]) + " |",
             "|" + "---|" * (len(cols) + 1)]
    for d in allr:
        vals = []
        for c in cols:
            v = d.get(c)
            if isinstance(v, float):
                v = f"{v / 1e6:.1f}MB" if c in ("dram_rd", "dram_wr") else f"{v:.3g}"
            vals.append(str(v))
        st = ", ".join(f"{k} {v:.0%}" for k, v in d["stalls"].items())
        lines.append("| " + " | ".join(vals + [st]) + " |")
    with open(prefix + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
