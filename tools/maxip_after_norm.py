"""Fig. 1(c)/(d) diagnostic:
the distribution over queries of the maximum inner product after the normalisation
of SIMPLE-LSH (every item divided by the global maximum 2-norm U) and of RANGE-LSH
(an item of sub-dataset j divided by its local maximum U_j), on a config's
synthetic items and queries.

  SIMPLE:  max_i q.x_i / U
  RANGE:   max_j ( max_{i in S_j} q.x_i ) / U_j          (m sub-datasets, Alg. 1)

Reading: Fig. 1(d) plots, per query, the largest normalised inner product over all
sub-datasets — the quantity whose size sets rho_j = G(c, S0/U_j).  The
per-sub-dataset maxima come from the library's exact top-1 (nrlsh_exact_topk) on
each sub-dataset's rows; U and U_j from the index's partition (V_j = U_j^2).
Off the hot path: a diagnostic, GPU only.
usage: python tools/maxip_after_norm.py [config] [num_parts] [nq] [out.json]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_08782_b200 as P  # noqa: E402
import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 32
cfg = workloads.CONFIGS[name]
nq = min(int(sys.argv[3]) if len(sys.argv) > 3 else 2000, cfg.nq)
X = torch.from_numpy(workloads.make_items(cfg)).cuda()
Q = torch.from_numpy(workloads.make_queries(cfg, nq)).cuda()
idx = P.Index(X, 32, m, seed=cfg.seed)
_, perm, off, V = idx.partition()
U = np.sqrt(np.asarray(V, dtype=np.float64))
perm_d = torch.from_numpy(np.asarray(perm, dtype=np.int64)).cuda()
best = np.full((m, nq), -np.inf)
for j in range(m):
    rows = X.index_select(0, perm_d[int(off[j]):int(off[j + 1])]).contiguous()
    _, sc = P.exact_topk(rows, Q, 1)
    best[j] = sc.double().cpu().numpy()[:, 0]
simple = best.max(axis=0) / U.max()
rng = (best / U[:, None]).max(axis=0)
edges = np.linspace(-0.2, 1.0, 25)


def summary(v):
    h, _ = np.histogram(np.clip(v, edges[0], edges[-1]), bins=edges)
    return {"mean": float(v.mean()), "median": float(np.median(v)),
            "p10": float(np.quantile(v, 0.1)), "p90": float(np.quantile(v, 0.9)),
            "hist_fraction": (h / len(v)).round(4).tolist()}


out = {"config": name, "num_parts": m, "nq": nq, "n": int(cfg.n), "d": int(cfg.d),
       "U": float(U.max()), "U_j_min": float(U.min()), "U_j_median": float(np.median(U)),
       "bin_edges": edges.round(3).tolist(),
       "simple_lsh": summary(simple), "range_lsh": summary(rng)}
print(json.dumps({k: v for k, v in out.items() if k != "bin_edges"}))
if len(sys.argv) > 4:
    json.dump(out, open(sys.argv[4], "w"), indent=1)
idx.close()
