import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1809_08782_b200 as P, workloads, oracle
cfg = workloads.CONFIGS["c3"]
X = workloads.make_items(cfg); Q = workloads.make_queries(cfg)
Xd = torch.from_numpy(X).cuda(); Qd = torch.from_numpy(Q).cuda()
idx = P.Index(Xd, 64, 64, seed=0)
norm2, perm, off, V = idx.partition()
A = idx.projection(); R = idx.rank_table()
codes_pos = idx.codes()
pos_of = np.empty(len(X), np.int64); pos_of[perm] = np.arange(len(X))
codes = codes_pos[pos_of]
part = (np.searchsorted(off, pos_of, side="right") - 1).astype(np.int32)
gt, _ = idx.exact_topk(Qd, 10); gt = gt.cpu().numpy()
for nq in [24, 1024, 2048, 10000]:
    for T in [4096, 8192, 65536]:
        ids, sc = idx.query(Qd[:nq], 10, T)
        ids = ids.cpu().numpy()
        rec = np.mean([len(set(a) & set(b)) / 10 for a, b in zip(ids, gt[:nq])])
        st = P.last_query_stats()
        bad = []
        for qi in [0, 1, nq // 2, nq - 1]:
            a, s = oracle.query(X, codes, part, R, A, Q[qi], T, 10)
            if not np.array_equal(a, ids[qi]): bad.append(qi)
        print(f"nq={nq} T={T} recall={rec:.4f} stats={st} mismatching(sampled)={bad}", flush=True)
