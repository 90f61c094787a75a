"""Single-query latency on c4: wall and CUDA-event time per call, stage times, launches.
usage: python tools/latency_probe.py [--nq 1] [--reps 50]"""
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
ap.add_argument("--config", default="c4")
ap.add_argument("--nq", type=int, default=1)
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
L = cfg.code_bits[-1]
T = max(cfg.budget_list())
X = torch.from_numpy(workloads.make_items(cfg)).cuda()
Q = torch.from_numpy(workloads.make_queries(cfg, nq=a.nq)).cuda()
idx = P.Index(X, L, cfg.num_parts[0], seed=cfg.seed, query_batch=cfg.query_batch)
for _ in range(5):
    idx.query(Q, cfg.k, T)
torch.cuda.synchronize()
wall, dev = [], []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    idx.query(Q, cfg.k, T)
    e1.record()
    torch.cuda.synchronize()
    wall.append((time.perf_counter() - t0) * 1e3)
    dev.append(e0.elapsed_time(e1))
P.profile_enable(True)
P.profile_read(reset=True)
idx.query(Q, cfg.k, T)
torch.cuda.synchronize()
prof = {k: round(v[0], 4) for k, v in P.profile_read(reset=True).items() if v[1]}
P.profile_enable(False)
print(f"nq={a.nq} T={T}: wall median {np.median(wall):.3f} ms, device median {np.median(dev):.3f} ms, "
      f"launches {P.last_query_stats()['kernel_launches']}, path {P.last_rerank_path()['path']}")
print("stages (ms):", prof)
