"""Debug: emulate the pilot bound (sampled histogram) vs the true per-query counts."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1809_08782_b200 as P  # noqa: E402
import workloads  # noqa: E402

cfg = workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
L = int(sys.argv[2]) if len(sys.argv) > 2 else 32
nq = 256
X = torch.from_numpy(workloads.make_items(cfg)).cuda()
Q = torch.from_numpy(workloads.make_queries(cfg, nq=nq)).cuda()
idx = P.Index(X, L, cfg.num_parts[0], seed=cfg.seed, query_batch=cfg.query_batch)
n, m = idx.n, cfg.num_parts[0]
codes = torch.from_numpy(idx.codes().astype(np.int64)).cuda()          # [n, W]
_, perm, offsets, _ = idx.partition()
part = torch.zeros(n, dtype=torch.int64, device="cuda")
for j in range(m):
    part[int(offsets[j]):int(offsets[j + 1])] = j
R = torch.from_numpy(idx.rank_table().astype(np.int64)).cuda().reshape(-1)
qc = idx.query_codes(Q).to(torch.int64) & 0xFFFFFFFF
codes &= 0xFFFFFFFF
stride = min(64, max(1, n // 32768))
samp = torch.arange(0, n, stride, device="cuda")
NR = m * (L + 1)


def popc(v):
    c = torch.zeros_like(v)
    for b in range(32):
        c += (v >> b) & 1
    return c


for T in (128, 256, 512, 2048):
    target = T + 4.0 * math.sqrt(T * stride) + stride
    need = max(1, math.ceil(target / stride))
    C = int(max(T, 2.0 * T + 16.0 * math.sqrt(T * stride) + 4096.0))
    bad_lo = bad_hi = 0
    worst = []
    for q in range(nq):
        h = torch.zeros(n, dtype=torch.int64, device="cuda")
        for w in range(codes.shape[1]):
            h += popc(codes[:, w] ^ qc[q, w])
        r = R[part * (L + 1) + h]
        true_hist = torch.bincount(r, minlength=NR)
        s_hist = torch.bincount(r[samp], minlength=NR)
        cs = torch.cumsum(s_hist, 0)
        B = int(torch.searchsorted(cs, torch.tensor([need], device="cuda"))[0].clamp(max=NR - 1))
        cnt = int(true_hist[:B + 1].sum())
        if cnt < T: bad_lo += 1
        if cnt > C: bad_hi += 1
        if q < 4 or cnt < T or cnt > C:
            worst.append((q, B, int(cs[B]), cnt, int(true_hist[B])))
    print(f"T={T} need={need} C={C}: cnt<T {bad_lo}/{nq}, cnt>C {bad_hi}/{nq}; samples {worst[:8]}", flush=True)
