#!/usr/bin/env python
"""bench.py — RANGE-LSH hot path on B200 (driver contract: one JSON line on rank 0).

A step is one pass of the whole hot path over one
batch of synthetic input: index build (norms, percentile partition, transform +
SRP codes, rank table), the batched query (query codes, Hamming scan + metric +
filter, top-T select, exact re-rank + top-k) and the exact brute-force ground
truth used for recall@10.  Default workload: BASELINE.json configs[3] (c4,
ImageNet-SIFT-shaped, "index build time and batched query throughput"),
64-bit codes, probe budget 1% of n.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
                  [--config c4|scale|...] [--bits 64] [--budget-permille 10]

Multi-GPU (torchrun): every rank builds the same index and answers its own
query shard (queries are independent units) — weak scaling, no data-path
collective; torch.distributed is used for the barrier and the max-over-ranks
time only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
# measured on this pool's B200 by tools/ubench.cu (profiles/r01/ubench_popc.txt):
# 4.569e12 POPC/s at 1965 MHz = 15.7 POPC/clk/SM x 148 SM (guide value 16/clk/SM)
POPC_PEAK_PER_S = 4.569e12
FFMA_PEAK_FLOPS = 148 * 128 * 2 * 1.965e9       # 74.4 TFLOP/s fp32 SIMT (128 FMA/clk/SM)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--bits", type=int, default=None)
    ap.add_argument("--parts", type=int, default=None)
    ap.add_argument("--budget-permille", type=float, default=None,
                    help="probe budget T as per-mille of n (default: config's largest budget)")
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-scale", dest="scale", action="store_false",
                    help="skip the scale (configs[4]) sub-record")
    ap.add_argument("--scale-steps", type=int, default=3)
    ap.add_argument("--sweep-m", action="store_true",
                    help="with --sweep: m in {1,32,64,128,256} at the paper's bit accounting")
    ap.add_argument("--sweep", default=None,
                    help="comma-separated configs: per probe budget queries/s and recall@k "
                         "(no driver line; writes --sweep-out)")
    ap.add_argument("--sweep-out", default=None)
    ap.add_argument("--proj", default="shared", choices=["shared", "per_partition"],
                    help="sub-index projections (DESIGN.md reading Q4; NEXT-4)")
    ap.add_argument("--scheme", default="percentile", choices=["percentile", "uniform"],
                    help="partitioning (Alg. 1 l.4; uniform = Fig. 3(a), NEXT-2)")
    ap.add_argument("--sweep-parts", default=None,
                    help="with --sweep: comma-separated m values instead of the config's")
    return ap.parse_args()


def workload(args):
    cfg = workloads.CONFIGS[args.config]
    L = args.bits or cfg.code_bits[-1]
    m = args.parts or cfg.num_parts[0]
    nq = args.nq or cfg.nq
    if args.budget_permille is not None:
        T = int(np.ceil(args.budget_permille * cfg.n / 1000.0))
    else:
        T = max(cfg.budget_list())
    desc = {
        "workload": f"{cfg.name}: n={cfg.n:,} d={cfg.d} {cfg.norm_law} norms x unit Gaussian "
                    f"directions, {L}-bit SRP codes, m={m} percentile sub-datasets, "
                    f"{nq:,} unit queries (sub-batches of {cfg.query_batch}), top-{cfg.k}, "
                    f"T={T:,} ({T / cfg.n:.2%} of n); step = build + query batch + exact "
                    f"ground truth",
        "n": cfg.n, "d": cfg.d, "code_bits": L, "num_parts": m, "nq_per_gpu": nq, "k": cfg.k,
        "probe_budget": T, "query_batch": cfg.query_batch, "seed": cfg.seed,
        "l2": "flushed between timed steps (512 MiB write)",
    }
    return cfg, L, m, nq, T, desc


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.rows = []
        self.proc = None
        self.gpu = gpu_index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for nm, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- roofline
def load_peaks():
    try:
        with open(PEAKS_FILE) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def roofline_for(slot, ms_total, count, info, peaks, peaks_src):
    """Algorithmic work of a stage over the timed steps / its device time there (CUDA
    events on the launching stream around the stage's launches)."""
    if count == 0 or ms_total <= 0:
        return None
    steps = info["steps"]
    per_launch_s = ms_total / count / 1e3
    n, d, L, W, nq = info["n"], info["d"], info["L"], info["W"], info["nq"]
    T, k, m = info["T"], info["k"], info["m"]
    traffic = info.get("traffic", {}).get(slot)
    if slot == "scan":
        # L/32 POPC per (query, item) pair the scan must evaluate;
        # pairs of sub-datasets whose radius is < 0 are skipped exactly.  POPCs issued:
        # W per pair, minus the W/2 the one-POPC-per-word-pair lower bound saves on the
        # pairs it decides alone, plus W/2 on the pairs where it ran and did not
        ops = (info["scanned_pairs"] * W - info["lb_decided_pairs"] * W
               + info["lb_pairs"] * (W // 2)) / count
        # (the library's own count of the POPCs issued, nrlsh_last_scan_popc: it knows
        # which bound ran where — the coarse first bound costs half of the pair bound)
        if info.get("scan_popc"):
            ops = info["scan_popc"] / count
        ach = ops / per_launch_s
        return {"bound": "alu", "kernel": "k6_scan (XOR+POPC Hamming scan + metric filter)",
                "achieved": ach / 1e12, "peak": POPC_PEAK_PER_S / 1e12, "unit": "TPOPC/s",
                "frac": ach / POPC_PEAK_PER_S, "traffic": traffic,
                "popc_per_pair": ops * count / max(1, info["scanned_pairs"]),
                "pairs_decided_per_s": info["scanned_pairs"] / (ms_total / 1e3),
                "pairs_decided_frac": info["scanned_pairs"] * W / (ms_total / 1e3) / POPC_PEAK_PER_S,
                "peak_source": "tools/ubench.cu measured POPC rate (profiles/r01/ubench_popc.txt)",
                "logical_pairs_per_s": nq * n * steps / (ms_total / 1e3),
                # SURVEY §8(d) "code-scan GB/s": code bytes compared (all n items per query)
                # and the codes actually scanned (skipped sub-datasets excluded), per second
                "code_scan_logical_gbs": nq * n * steps * L / 8 / (ms_total / 1e3) / 1e9,
                "code_scan_actual_gbs": info["scanned_pairs"] * L / 8 / (ms_total / 1e3) / 1e9,
                "dram_gbs": (traffic / per_launch_s / 1e9) if traffic else None}
    if slot == "gt_filter" or (slot == "rerank" and info.get("rerank_path") == "tensor"):
        # one bf16 pass over every item per query; the re-rank's member-mode pass
        # multiplies only the tiles of sub-datasets holding candidates (its own count)
        # the pairs each filter actually multiplied (tile pruning skips the rest)
        # (the counters are already summed over the timed steps)
        pairs = info["gt_filter_pairs"] if slot == "gt_filter" else info["rerank_filter_pairs"]
        fl = 2.0 * pairs * d / count
        ach = fl / per_launch_s
        if slot == "rerank":
            pk = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")) * 1e12
            return {"bound": "tensor", "kernel": "rerank (tcgen05 bf16 filter pass, member mode)",
                    "achieved": ach / 1e12, "peak": pk / 1e12, "unit": "TFLOP/s",
                    "frac": ach / pk, "traffic": traffic,
                    "peak_source": f"MEASURED_PEAKS.json bf16 sustained ({peaks_src})"}
        if info.get("gt_tensor"):
            pk = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")) * 1e12
            return {"bound": "tensor", "kernel": "gt_filter (tcgen05 bf16)", "achieved": ach / 1e12,
                    "peak": pk / 1e12, "unit": "TFLOP/s", "frac": ach / pk, "traffic": traffic,
                    "peak_source": f"MEASURED_PEAKS.json bf16 sustained ({peaks_src})"}
        return {"bound": "alu", "kernel": "gt_filter_simt (fp32 FFMA filter GEMM)",
                "achieved": ach / 1e12, "peak": FFMA_PEAK_FLOPS / 1e12, "unit": "TFLOP/s",
                "frac": ach / FFMA_PEAK_FLOPS, "traffic": traffic,
                "peak_source": "148 SM x 128 FFMA/clk x 2 x 1965 MHz"}
    hbm = peaks["hbm_gbs"] * 1e9
    if slot == "rerank":
        by = info["score_bytes"] / count
    elif slot in ("codes", "norms"):
        by = (n * d * 4.0 + (n * W * 4.0 if slot == "codes" else n * 8.0)) * steps / count
    else:
        return None
    ach = by / per_launch_s
    return {"bound": "hbm", "kernel": slot, "achieved": ach / 1e9, "peak": hbm / 1e9,
            "unit": "GB/s", "frac": ach / hbm, "traffic": traffic,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peaks_src})"}


def load_traffic():
    """dram bytes per launch from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except Exception:
        return {}


# ----------------------------------------------------------------- CPU oracle
def cpu_oracle_step(cfg, X, Q, L, m, T, k, nq_full, nsample, threads):
    """The oracle, as it stands, on the host cores: full index build (Alg. 1) over
    all n items, then `nsample` whole queries (codes, candidates, re-rank) plus
    their exact top-k; returns extrapolated seconds for the full step."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    t0 = time.perf_counter()
    nv = oracle.norm2(X)
    part, perm, off, V = oracle.partition(nv, m)
    A = oracle.projection(cfg.seed, X.shape[1] + 1, L)
    R, _ = oracle.rank_table(np.sqrt(V), L, 0.01)
    codes = oracle.item_codes_parallel(X, part, V, nv, A, threads=threads)
    t_build = time.perf_counter() - t0

    def one(q):
        a, _ = oracle.query(X, codes, part, R, A, q, T, k)
        b, _ = oracle.exact_topk(X, q, k)
        return a, b

    t1 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, list(Q[:nsample])))
    t_q = (time.perf_counter() - t1) / nsample       # wall seconds per query at `threads`
    return t_build, t_q, t_build + nq_full * t_q


# ----------------------------------------------------------------- main arms
def max_over_ranks(x, dist, device=None):
    """Max of a per-rank float over all ranks (identity without torch.distributed)."""
    if dist is None:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(units_per_rank, world, ms_max):
    """Weak scaling: every rank answers its own `units_per_rank` queries; the job
    rate is all ranks' units over the slowest rank's time."""
    return world * units_per_rank / (ms_max / 1e3)


def rank_queries(cfg, nq, rank):
    """Rank r's query shard: an independent seeded stream (queries are independent
    units, so the index is replicated and nothing is exchanged on the data path)."""
    return workloads.make_queries(cfg, nq=nq, shard=rank)


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args):
    """The oracle arm (--impl reference): rank 0 only; the oracle as it stands on
    the host cores, same config/metric/unit as the native arm."""
    world, rank, local = dist_setup(args)
    if rank != 0:
        return
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    cfg, L, m, nq, T, desc = workload(args)
    X = workloads.make_items(cfg)
    Q = workloads.make_queries(cfg, nq=8 * (args.warmup + args.steps))
    threads = os.cpu_count() or 1
    nsample = 8
    t0 = time.perf_counter()
    nv = oracle.norm2(X)
    part, perm, off, V = oracle.partition(nv, m)
    A = oracle.projection(cfg.seed, X.shape[1] + 1, L)
    R, _ = oracle.rank_table(np.sqrt(V), L, 0.01)
    codes = oracle.item_codes_parallel(X, part, V, nv, A, threads=threads)
    t_build = time.perf_counter() - t0

    def one(q):
        oracle.query(X, codes, part, R, A, q, T, cfg.k)
        oracle.exact_topk(X, q, cfg.k)

    tq = []
    for i in range(args.warmup + args.steps):
        t1 = time.perf_counter()
        with ThreadPoolExecutor(max_workers=threads) as ex:
            list(ex.map(one, list(Q[i * nsample:(i + 1) * nsample])))
        if i >= args.warmup:
            tq.append((time.perf_counter() - t1) / nsample)
    t_q = float(np.mean(tq)) if tq else 0.0
    t_step = t_build + nq * t_q
    value = nq / t_step
    sample = (f"oracle build over all {cfg.n:,} items once ({t_build:.1f} s, item codes on "
              f"{threads} threads) + per step {nsample} whole queries (codes, candidates, "
              f"re-rank, exact top-k) on {threads} threads ({t_q * 1e3:.0f} ms/query wall), "
              f"extrapolated to a {nq:,}-query step")
    line = {"impl": "reference", "metric": "queries/s at fixed probe budget with recall@10",
            "value": value, "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": desc,
            "cpu_baseline": {"value": value, "unit": "queries/s", "cores": threads,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def measure_path(P, torch, cfg, L, m, T, Xd, Qd, steps, warmup, stream, flush, dist=None):
    """Time `steps` whole steps (build + query batch + exact ground truth), each
    phase bracketed by CUDA events on the launching stream; per-stage device time
    from the library's own events; the work counters the rooflines need."""
    k = cfg.k

    def step(ev=None):
        if ev:
            ev[0].record(stream)
        idx = P.Index(Xd, L, m, seed=cfg.seed, query_batch=cfg.query_batch)
        if ev:
            ev[1].record(stream)
        ids, sc = idx.query(Qd, k, T)
        qstats = P.last_query_stats()
        qstats.update(P.last_scan_stats())
        rinfo = P.last_rerank_path()
        if ev:
            ev[2].record(stream)
        # ground truth, warm-started from the LSH answers (certified; the result
        # does not depend on the seeds — tests/test_gpu_parity.py)
        gid, gsc = idx.exact_topk(Qd, k, seed_ids=ids)
        gstats = P.last_exact_stats()
        if ev:
            ev[3].record(stream)
        idx.close()
        return ids, gid, qstats, rinfo, gstats

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    P.profile_read(reset=True)
    P.profile_enable(True)
    launches0 = P.launch_count()
    acc = {"scanned_pairs": 0, "lb_pairs": 0, "lb_decided_pairs": 0, "scan_popc": 0, "buffer_entries": 0,
           "fallback_queries": 0, "rerank_filter_pairs": 0,
           "rerank_overflow": 0, "gt_filter_pairs": 0, "gt_survivors": 0}
    evs = []
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(steps):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ids, gid, qstats, rinfo, gstats = step(ev)
        evs.append(ev)
        acc["scanned_pairs"] += qstats["scanned_pairs"]
        acc["lb_pairs"] += qstats["bound_pairs"]
        acc["lb_decided_pairs"] += qstats["bound_decided_pairs"]
        acc["scan_popc"] += qstats.get("popc_ops", 0)
        acc["buffer_entries"] += qstats["buffer_entries"]
        acc["fallback_queries"] += qstats["fallback_queries"]
        acc["rerank_filter_pairs"] += rinfo["filter_pairs"]
        acc["rerank_overflow"] += rinfo["overflow_redone"]
        acc["gt_filter_pairs"] += gstats["filter_pairs"]
        acc["gt_survivors"] += gstats["sum_survivors"]
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = P.launch_count() - launches0
    P.profile_enable(False)
    prof = P.profile_read(reset=True)
    ms = [e[0].elapsed_time(e[3]) for e in evs]
    ids_h, gid_h = ids.cpu().numpy(), gid.cpu().numpy()
    rec = float(np.mean([len(set(a.tolist()) & set(b.tolist())) / k for a, b in zip(ids_h, gid_h)]))
    rec10 = float(np.mean([len(set(a[:10].tolist()) & set(b[:10].tolist())) / 10
                           for a, b in zip(ids_h, gid_h)]))
    return {"ms_all": ms, "ms_step": float(np.mean(ms)),
            "build_ms": float(np.mean([e[0].elapsed_time(e[1]) for e in evs])),
            "query_ms": float(np.mean([e[1].elapsed_time(e[2]) for e in evs])),
            "query_ms_all": [e[1].elapsed_time(e[2]) for e in evs],
            "gt_ms": float(np.mean([e[2].elapsed_time(e[3]) for e in evs])),
            "prof": prof, "launches": launches, "acc": acc, "recall_at_k": rec,
            "recall_at_10": rec10, "rerank_path": rinfo["path"]}


def rooflines(r, cfg, L, m, nq, T, steps, peaks, peaks_src):
    """SURVEY.md §8(d) rooflines from one measure_path() result: the dominant
    kernel, every stage's own, and the build / query totals."""
    prof, acc = r["prof"], r["acc"]
    W = 1 if L <= 32 else (2 if L <= 64 else 4)
    info = {"n": cfg.n, "d": cfg.d, "L": L, "W": W, "nq": nq, "T": T, "k": cfg.k, "m": m,
            "scanned_pairs": acc["scanned_pairs"], "lb_pairs": acc["lb_pairs"],
            "lb_decided_pairs": acc["lb_decided_pairs"], "scan_popc": acc["scan_popc"],
            "traffic": load_traffic(), "steps": steps,
            "rerank_path": r["rerank_path"], "rerank_filter_pairs": acc["rerank_filter_pairs"],
            "gt_filter_pairs": acc["gt_filter_pairs"],
            "score_bytes": float(nq) * T * cfg.d * 4.0 * steps, "gt_tensor": True}
    live = {n_: v for n_, v in prof.items() if v[1] > 0}
    dom = max(live.items(), key=lambda x: x[1][0])
    roof = roofline_for(dom[0], dom[1][0], dom[1][1], info, peaks, peaks_src)
    scan_roof = roofline_for("scan", *prof["scan"], info, peaks, peaks_src) if prof["scan"][1] else None
    others = {s_: roofline_for(s_, *prof[s_], info, peaks, peaks_src)
              for s_ in ("gt_filter", "rerank", "codes", "norms") if prof.get(s_, (0, 0))[1]}
    hbm = peaks["hbm_gbs"] * 1e9
    bf16 = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")) * 1e12
    n, d = cfg.n, cfg.d
    # build (Alg. 1): X read twice (exact ranks precede hashing) + codes + ~32 B/item
    # of keys / permutation
    b_bytes = 2.0 * n * d * 4 + n * L / 8.0 + 32.0 * n
    build_dev = sum(prof.get(s_, (0, 0))[0] for s_ in ("norms", "partition", "scatter", "codes")) / steps
    build = {"bound": "hbm", "algorithmic_bytes": b_bytes, "t_roof_ms": b_bytes / hbm * 1e3,
             "t_measured_ms": r["build_ms"], "frac": b_bytes / hbm * 1e3 / r["build_ms"],
             "t_device_stages_ms": build_dev, "frac_device_stages": b_bytes / hbm * 1e3 / build_dev,
             "peak_gbs": peaks["hbm_gbs"], "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peaks_src})"}
    # query: t_codes + max(popc, hbm)_scan + t_select + t_rerank
    nsub = -(-nq // cfg.query_batch)
    t_codes = 2.0 * nq * d * L / FFMA_PEAK_FLOPS
    t_scan_hbm = nsub * n * W * 4.0 / hbm
    t_sel = acc["buffer_entries"] / steps * 8.0 / hbm
    def q_roof(popcs, rr_pairs):
        t_scan = max(popcs / POPC_PEAK_PER_S, t_scan_hbm)
        t_rr = rr_pairs * 2.0 * d / bf16
        t = t_codes + t_scan + t_sel + t_rr
        return {"t_roof_ms": t * 1e3, "frac": t * 1e3 / r["query_ms"],
                "terms_ms": {"codes": t_codes * 1e3, "scan": t_scan * 1e3, "select": t_sel * 1e3,
                             "rerank": t_rr * 1e3}}
    query = {"t_measured_ms": r["query_ms"],
             # every (query, item) pair scanned; every probed candidate scored on the tensor pipe
             "logical": q_roof(float(nq) * n * W, float(nq) * T),
             # the POPCs the scan issued after exact sub-dataset skipping and the lower
             # bound, the pairs the re-rank's filter multiplied
             "actual": q_roof((acc["scan_popc"] or (acc["scanned_pairs"] * W - acc["lb_decided_pairs"] * W
                                                    + acc["lb_pairs"] * (W // 2))) / steps,
                              acc["rerank_filter_pairs"] / steps),
             "peaks": {"popc_per_s": POPC_PEAK_PER_S, "hbm_gbs": peaks["hbm_gbs"],
                       "bf16_tflops": bf16 / 1e12, "ffma_tflops": FFMA_PEAK_FLOPS / 1e12}}
    return roof, scan_roof, others, build, query


def run_native(args):
    import torch
    world, rank, local = dist_setup(args)
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        dist = None
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_1809_08782_b200 as P

    cfg, L, m, nq, T, desc = workload(args)
    t_gen = time.perf_counter()
    X = workloads.make_items(cfg)
    Q = rank_queries(cfg, nq, rank)
    t_gen = time.perf_counter() - t_gen
    Xd = torch.from_numpy(X).to(dev)
    Qd = torch.from_numpy(Q).to(dev)
    k = cfg.k
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    sampler = ClockSampler(local)
    sampler.start()
    r = measure_path(P, torch, cfg, L, m, T, Xd, Qd, args.steps, args.warmup, stream, flush, dist)
    clocks = sampler.stop()
    ms_step = max_over_ranks(r["ms_step"], dist, dev)
    value = whole_job_rate(nq, world, ms_step)
    prof = r["prof"]

    # -------- end to end through the public API with HOST buffers (pinned)
    # latency mode: 1 and 2 queries per call, index resident; the scan
    # is then bound by streaming the codes of the probed sub-datasets from HBM
    latency = []
    if not args.no_latency:
        idx = P.Index(Xd, L, m, seed=cfg.seed, query_batch=cfg.query_batch)
        for nql in (1, 2):
            Ql = Qd[:nql].contiguous()
            for _ in range(3):
                idx.query(Ql, k, T)
            P.profile_read(reset=True)
            P.profile_enable(True)
            ts = []
            for _ in range(20):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                idx.query(Ql, k, T)
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            P.profile_enable(False)
            pr = P.profile_read(reset=True)
            qs = P.last_query_stats()
            scan_ms = pr["scan"][0] / max(1, pr["scan"][1])
            latency.append({"nq": nql, "ms_median": float(np.median(ts)),
                            "scan_ms": scan_ms,
                            "code_scan_actual_gbs": qs["scanned_pairs"] * L / 8 / (scan_ms / 1e3) / 1e9,
                            "code_scan_logical_gbs": nql * cfg.n * L / 8 / (scan_ms / 1e3) / 1e9})
        idx.close()
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(X).pin_memory()
        Qh = torch.from_numpy(Q).pin_memory()
        oid = torch.empty((nq, k), dtype=torch.int64).pin_memory()
        osc = torch.empty((nq, k), dtype=torch.float32).pin_memory()
        gid2 = torch.empty((nq, k), dtype=torch.int64).pin_memory()
        gsc2 = torch.empty((nq, k), dtype=torch.float32).pin_memory()
        e2e_ms = []
        for it in range(args.e2e_steps + 1):   # iteration 0: untimed warm-up (pool growth)
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            idx = P.Index(Xh, L, m, seed=cfg.seed, query_batch=cfg.query_batch)
            idx.query(Qh, k, T, out_ids=oid, out_scores=osc)
            idx.exact_topk(Qh, k, out_ids=gid2, out_scores=gsc2, seed_ids=oid)
            idx.close()
            torch.cuda.synchronize()
            if it > 0:
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2 = float(np.mean(e2e_ms))
        e2 = max_over_ranks(e2, dist, dev)
        e2e = {"value": whole_job_rate(nq, world, e2), "unit": "queries/s",
               "h2d_bytes_per_step": int(X.nbytes + 2 * Q.nbytes),
               "d2h_bytes_per_step": int(2 * (oid.numel() * 8 + osc.numel() * 4)),
               "ms_per_step": e2, "ms_all": e2e_ms}
        del Xh, Qh

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peaks, peaks_src = load_peaks()
    stage = {name: {"ms_per_step": v[0] / args.steps, "launches_per_step": v[1] / args.steps}
             for name, v in prof.items() if v[1] > 0}
    roof, scan_roof, others, build_roof, query_roof = rooflines(r, cfg, L, m, nq, T, args.steps,
                                                                peaks, peaks_src)
    # the same kernels with the sub-batches on one stream (after the timed region,
    # untimed): in the timed region two sub-batches share the GPU, so each kernel's
    # CUDA-event duration there includes the other stream's work
    iso = None
    if world == 1:
        os.environ["NRLSH_QUERY_SERIAL"] = "1"
        try:
            ri = measure_path(P, torch, cfg, L, m, T, Xd, Qd, 2, 1, stream, flush)
        finally:
            del os.environ["NRLSH_QUERY_SERIAL"]
        iroof, iscan, iothers, _, _ = rooflines(ri, cfg, L, m, nq, T, 2, peaks, peaks_src)
        iso = {"note": "sub-batches serialised on one stream (NRLSH_QUERY_SERIAL=1), 2 untimed "
                       "steps after the timed region: kernel efficiency without stream overlap",
               "ms_per_step": ri["ms_step"], "roofline": iroof, "scan_roofline": iscan,
               "other_rooflines": iothers,
               "stage_ms_per_step": {nm: v[0] / 2 for nm, v in ri["prof"].items() if v[1] > 0}}
        if roof and iroof and roof.get("kernel") == iroof.get("kernel"):
            roof["frac_serial_stream"] = iroof["frac"]
            roof["note"] = ("timed region: two sub-batch streams share the GPU, so the kernel's "
                            "CUDA-event span includes the other stream's work; frac_serial_stream: "
                            "the same kernel with the sub-batches on one stream")

    # -------- scale (BASELINE configs[4]) in the same run: a sub-record, not the headline
    scale = None
    if args.scale and world == 1 and cfg.name != "scale":
        del Xd, Qd
        torch.cuda.empty_cache()
        scfg = workloads.CONFIGS["scale"]
        sL, sm_ = scfg.code_bits[-1], scfg.num_parts[0]
        sT = max(scfg.budget_list())
        sX = torch.from_numpy(workloads.make_items(scfg)).to(dev)
        sQ = torch.from_numpy(workloads.make_queries(scfg)).to(dev)
        rs = measure_path(P, torch, scfg, sL, sm_, sT, sX, sQ, args.scale_steps, 2, stream, flush)
        sroof, sscan, sothers, sbuild, squery = rooflines(rs, scfg, sL, sm_, scfg.nq, sT,
                                                          args.scale_steps, peaks, peaks_src)
        scale = {"workload": f"scale: n={scfg.n:,} d={scfg.d} {scfg.norm_law} norms, {sL}-bit codes, "
                             f"m={sm_}, {scfg.nq:,} queries (sub-batches of {scfg.query_batch}), "
                             f"top-{scfg.k}, T={sT:,}",
                 "value": scfg.nq / (rs["ms_step"] / 1e3), "unit": "queries/s",
                 "ms_per_step": rs["ms_step"], "ms_all": rs["ms_all"], "steps": args.scale_steps,
                 "warmup": 2, "query_ms_all": rs["query_ms_all"], "build_ms": rs["build_ms"], "query_ms": rs["query_ms"], "gt_ms": rs["gt_ms"],
                 "recall_at_100": rs["recall_at_k"], "recall_at_10": rs["recall_at_10"],
                 "scan_frac": sscan["frac"] if sscan else None, "build_frac": sbuild["frac"],
                 "build_roofline": sbuild, "query_roofline": squery, "roofline": sroof,
                 "stage_ms_per_step": {nm: v[0] / args.scale_steps for nm, v in rs["prof"].items()
                                       if v[1] > 0},
                 "counters": rs["acc"]}
        del sX, sQ
        torch.cuda.empty_cache()

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = os.cpu_count() or 1
        nsample = 8
        t_build, t_q, t_step = cpu_oracle_step(cfg, X, Q, L, m, T, k, nq, nsample, threads)
        cpu = {"value": nq / t_step, "unit": "queries/s", "cores": threads, "kind": "oracle",
               "sample": f"oracle build over all {cfg.n:,} items ({t_build:.1f} s; item codes "
                         f"on {threads} threads) + {nsample} whole queries incl. exact top-k "
                         f"({t_q * 1e3:.0f} ms/query wall on {threads} threads), extrapolated "
                         f"to {nq:,} queries"}

    line = {
        "metric": "queries/s at fixed probe budget with recall@10",
        "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32 codes / f32 scores",
        "data": "synthetic", "config": desc,
        "recall_at_10": r["recall_at_10"],
        "stage_ms_per_step": stage,
        "phase_ms_per_step": {"build": r["build_ms"], "query": r["query_ms"], "ground_truth": r["gt_ms"]},
        "roofline": roof, "scan_roofline": scan_roof, "other_rooflines": others,
        "rooflines_serial_stream": iso,
        "build_roofline": build_roof, "query_roofline": query_roof,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(r["launches"]),
        "latency_mode": latency,
        "scale": scale,
        "clocks": clocks,
        "notes": {"input_gen_s": t_gen, "peaks": peaks_src,
                  "step_ms_all": r["ms_all"], "rerank_path": r["rerank_path"],
                  "counters_per_step": {k_: v / args.steps for k_, v in r["acc"].items()}},
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def _sweep_plan(cfg, m_sweep=False):
    """(code_bits, num_parts, budgets, index_bits_in_budget) runs of a config: its
    stated budgets plus the paper's 2^i probe grid (Fig. 2 x-axis)
    where BASELINE.json asks for recall curves (c3, c4).  m_sweep (SURVEY §8(f)
    NEXT-1): m = 1 (SIMPLE-LSH) against m in {32, 64, 128, 256} at the paper's bit
    accounting, L_h = code_bits - ceil(log2 m)."""
    Ts = sorted(set(cfg.budget_list()) | set(t for t in cfg.extra_T if t <= cfg.n))
    runs = []
    if m_sweep:
        for L in cfg.code_bits:
            for m in (1, 32, 64, 128, 256):
                if m <= cfg.n:
                    runs.append((L, m, Ts, True))
        return runs
    for L in cfg.code_bits:
        for m in cfg.num_parts:
            runs.append((L, m, Ts, False))
    return runs


def run_sweep(args):
    """queries/s (nrlsh_query only, device-resident queries, CUDA events) and
    recall@k against the exact top-k, at every probe budget of each config."""
    import torch
    import paper_1809_08782_b200 as P
    dev = torch.device("cuda", 0)
    rows = []
    for name in args.sweep.split(","):
        cfg = workloads.CONFIGS[name]
        X = workloads.make_items(cfg)
        Q = workloads.make_queries(cfg)
        Xd = torch.from_numpy(X).to(dev)
        Qd = torch.from_numpy(Q).to(dev)
        k = cfg.k
        gt = None
        plan = _sweep_plan(cfg, args.sweep_m)
        if args.sweep_parts:
            ms = [int(v) for v in args.sweep_parts.split(",")]
            Ts0, ib0 = plan[0][2], plan[0][3]
            plan = [(L, m_, Ts0, ib0) for L in cfg.code_bits for m_ in ms]
        for L, m, Ts, ibits in plan:
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            idx = P.Index(Xd, L, m, seed=cfg.seed, query_batch=cfg.query_batch,
                          index_bits_in_budget=ibits, proj=args.proj, scheme=args.scheme)
            e1.record()
            torch.cuda.synchronize()
            build_ms = e0.elapsed_time(e1)
            if gt is None:
                gt, _ = idx.exact_topk(Qd, k)
                gt = gt.cpu().numpy()
            for T in Ts:
                idx.query(Qd[: min(len(Q), 256)], k, T)          # warm-up
                ms = []
                for _ in range(3):
                    e0.record()
                    ids, sc = idx.query(Qd, k, T)
                    e1.record()
                    torch.cuda.synchronize()
                    ms.append(e0.elapsed_time(e1))
                ids = ids.cpu().numpy()
                rec = float(np.mean([len(set(a.tolist()) & set(b.tolist())) / k
                                     for a, b in zip(ids, gt)]))
                row = {"config": name, "n": cfg.n, "d": cfg.d, "code_bits": L, "num_parts": m,
                       "proj": args.proj, "scheme": args.scheme,
                       "hash_bits": idx.hash_bits, "index_bits_in_budget": ibits,
                       "nq": len(Q), "k": k, "probe_budget": int(T), "budget_frac": T / cfg.n,
                       "queries_per_s": len(Q) / (float(np.median(ms)) / 1e3),
                       "query_ms": float(np.median(ms)), "recall_at_k": rec,
                       "build_ms": build_ms}
                if k > 10:   # recall@10: the first 10 returned against the true top-10
                    row["recall_at_10"] = float(np.mean([
                        len(set(a[:10].tolist()) & set(b[:10].tolist())) / 10
                        for a, b in zip(ids, gt)]))
                rows.append(row)
                print(json.dumps(row), flush=True)
            idx.close()
        del Xd, Qd
        torch.cuda.empty_cache()
    if args.sweep_out:
        with open(args.sweep_out, "w") as f:
            json.dump(rows, f, indent=1)


def main():
    args = parse()
    if args.sweep:
        run_sweep(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_native(args)


if __name__ == "__main__":
    main()
