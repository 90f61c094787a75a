"""Debug: share of n in sub-datasets holding any candidate of a 256-query group."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_08782_b200 as P  # noqa: E402
import workloads  # noqa: E402

cfg = workloads.CONFIGS["c4"]
X = torch.from_numpy(workloads.make_items(cfg)).cuda()
Q = torch.from_numpy(workloads.make_queries(cfg, nq=1024)).cuda()
for L in (64, 32):
    idx = P.Index(X, L, 128, seed=cfg.seed)
    norm2, perm, off, V = idx.partition()
    part_of_id = np.empty(idx.n, np.int64)
    for j in range(128):
        part_of_id[perm[off[j]:off[j + 1]]] = j
    sizes = np.diff(off)
    for T in (2341, 23404, 65536):
        ids, _ = idx.candidates(T, queries=Q)
        pj = part_of_id[ids.cpu().numpy().astype(np.int64)]
        fr = []
        for g in range(4):
            act = np.unique(pj[g * 256:(g + 1) * 256])
            fr.append(sizes[act].sum() / idx.n)
        per_q = np.mean([sizes[np.unique(pj[q])].sum() / idx.n for q in range(0, 1024, 64)])
        print(f"L={L} T={T}: active share per 256-group {np.round(fr, 3)}, per query {per_q:.3f}", flush=True)
