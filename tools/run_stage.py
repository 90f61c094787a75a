"""Run one stage of the hot path on a BASELINE config (for ncu / quick timing).
usage: python tools/run_stage.py {gt,query,build} [--config c4] [--nq 1024] [--bits 64] [--T N]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_08782_b200 as P  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("stage")
ap.add_argument("--config", default="c4")
ap.add_argument("--nq", type=int, default=1024)
ap.add_argument("--bits", type=int, default=None)
ap.add_argument("--T", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
L = a.bits or cfg.code_bits[-1]
T = a.T or max(cfg.budget_list())
X = torch.from_numpy(workloads.make_items(cfg)).cuda()
Q = torch.from_numpy(workloads.make_queries(cfg, nq=a.nq)).cuda()
idx = P.Index(X, L, cfg.num_parts[0], seed=cfg.seed, query_batch=cfg.query_batch)
P.profile_enable(True)
for r in range(a.reps):
    P.profile_read(reset=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if a.stage == "gt":
        ids, sc = idx.exact_topk(Q, cfg.k)
        st = P.last_exact_stats()
    elif a.stage == "gtseed":
        if r == 0:
            seeds, _ = idx.query(Q, cfg.k, T)
        ids, sc = idx.exact_topk(Q, cfg.k, seed_ids=seeds)
        st = P.last_exact_stats()
    elif a.stage == "query":
        ids, sc = idx.query(Q, cfg.k, T)
        st = P.last_query_stats()
        st.update(P.last_rerank_stats())
    else:
        idx2 = P.Index(X, L, cfg.num_parts[0], seed=cfg.seed)
        st = {}
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    prof = {k: round(v[0], 3) for k, v in P.profile_read().items() if v[1]}
    print(f"rep {r}: {dt * 1e3:.2f} ms wall; stats {st}; stages(ms) {prof}", flush=True)
