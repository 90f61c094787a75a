"""Debug: how much of n the Cauchy-Schwarz tile pruning keeps per 256-query pair."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_08782_b200 as P  # noqa: E402
import workloads  # noqa: E402

cfg = workloads.CONFIGS["c4"]
X = workloads.make_items(cfg)
Q = workloads.make_queries(cfg, nq=1024)
Xd, Qd = torch.from_numpy(X).cuda(), torch.from_numpy(Q).cuda()
idx = P.Index(Xd, 64, 128, seed=cfg.seed)
norms = np.sort(np.linalg.norm(X.astype(np.float64), axis=1))
ids, sc = idx.query(Qd, 10, 23404)
gt, gsc = idx.exact_topk(Qd, 10)
th_lsh = sc[:, 9].cpu().numpy()
th_gt = gsc[:, 9].cpu().numpy()
qn = np.linalg.norm(Q.astype(np.float64), axis=1)
for name, th in (("lsh seeds", th_lsh), ("true 10th", th_gt)):
    t = th / qn
    print(name, "theta/|q| percentiles 0,1,10,50,90:", np.round(np.percentile(t, [0, 1, 10, 50, 90]), 2))
    keep = []
    for g in range(4):
        tau = t[g * 256:(g + 1) * 256].min()
        keep.append(1 - np.searchsorted(norms, tau) / len(norms))
    print("  kept share of n per pair:", np.round(keep, 5))
print("norm percentiles 50,99,99.9,99.99,max:", np.round(np.percentile(norms, [50, 99, 99.9, 99.99, 100]), 2))
