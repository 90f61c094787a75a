"""profiles/traffic.json from ncu --set full summaries (tools/ncu_summary.py JSON):
dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged per kernel class,
in the profile slots bench.py reports (`traffic` of each roofline entry).

usage: python tools/traffic_from_ncu.py OUT.json QUERY_SUMMARY.json [GT_SUMMARY.json] --source TEXT
QUERY_SUMMARY: a capture of `tools/run_stage.py query` (build + one query sub-batch:
the member-mode filter is the re-rank); GT_SUMMARY: of `run_stage.py gtseed`."""
import json
import sys

SLOTS = [("k6_pilot", "pilot"), ("k6_scan", "scan"), ("k7_select", "select"), ("k1_norms", "norms"),
         ("k3_codes", "codes")]


def per_slot(rows, mapping):
    acc = {}
    for r in rows:
        for prefix, slot in mapping:
            if r["kernel"].startswith(prefix):
                acc.setdefault(slot, []).append((r.get("dram_rd") or 0) + (r.get("dram_wr") or 0))
    return {k: sum(v) / len(v) for k, v in acc.items()}


def main():
    args = [a for a in sys.argv[1:]]
    src = ""
    if "--source" in args:
        i = args.index("--source")
        src = args[i + 1]
        del args[i:i + 2]
    out, q = args[0], args[1]
    rows = json.load(open(q))
    res = per_slot(rows, SLOTS + [("gt_filter_tc", "rerank")])
    if len(args) > 2:
        res.update(per_slot(json.load(open(args[2])), [("gt_filter_tc", "gt_filter")]))
    res["_source"] = src
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
