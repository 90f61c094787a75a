"""Debug: one query's sampled vs true cumulative counts along the structure order."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_08782_b200 as P  # noqa: E402
import workloads  # noqa: E402

cfg = workloads.CONFIGS["c4"]
qi = int(sys.argv[1]) if len(sys.argv) > 1 else 828
X = torch.from_numpy(workloads.make_items(cfg)).cuda()
Q = torch.from_numpy(workloads.make_queries(cfg)).cuda()
idx = P.Index(X, 64, 128, seed=cfg.seed, index_bits_in_budget=True)
L = idx.hash_bits
m = 128
codes = torch.from_numpy(idx.codes().astype(np.int64)).cuda() & 0xFFFFFFFF
_, perm, off, _ = idx.partition()
part = torch.zeros(idx.n, dtype=torch.int64, device="cuda")
for j in range(m):
    part[int(off[j]):int(off[j + 1])] = j
R = torch.from_numpy(idx.rank_table().astype(np.int64)).cuda().reshape(-1)
qc = idx.query_codes(Q[qi:qi + 1]).to(torch.int64) & 0xFFFFFFFF


def popc(v):
    c = torch.zeros_like(v)
    for b in range(32):
        c += (v >> b) & 1
    return c


h = popc(codes[:, 0] ^ qc[0, 0]) + popc(codes[:, 1] ^ qc[0, 1])
r = R[part * (L + 1) + h]
NR = m * (L + 1)
true_hist = torch.bincount(r, minlength=NR).cpu().numpy()
stride = 64
samp = torch.arange(0, idx.n, stride, device="cuda")
s_hist = torch.bincount(r[samp], minlength=NR).cpu().numpy()
ct, cs = np.cumsum(true_hist), np.cumsum(s_hist)
for T in (2341, 4096):
    target = T + 4.0 * math.sqrt(T * stride) + stride
    need = max(16, math.ceil(target / stride))
    B = int(np.searchsorted(cs, need))
    print(f"T={T} need={need} B={B} sampled<=B={cs[B]} true<=B={ct[B]} cell B: true {true_hist[B]} sampled {s_hist[B]}")
    for b in range(max(0, B - 5), B + 1):
        print("   r", b, "true", true_hist[b], "samp", s_hist[b], "cum", ct[b], cs[b])
