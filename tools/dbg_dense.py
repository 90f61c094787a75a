import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1809_08782_b200 as P, workloads, oracle
cfg = workloads.CONFIGS["tiny"]
X = workloads.make_items(cfg); Q = workloads.make_queries(cfg)[:24]
Xd = torch.from_numpy(X).cuda(); Qd = torch.from_numpy(Q).cuda()
idx = P.Index(Xd, 32, 8, seed=0)
norm2, perm, off, V = idx.partition()
pos_of = np.empty(len(X), np.int64); pos_of[perm] = np.arange(len(X))
part = np.searchsorted(off, pos_of, side="right") - 1
for T in [100, 1428, 10000]:
    os.environ.pop("NRLSH_NO_DENSE", None)
    a, sa = idx.query(Qd, 10, T)
    os.environ["NRLSH_NO_DENSE"] = "1"
    b, sb = idx.query(Qd, 10, T)
    a, b = a.cpu().numpy(), b.cpu().numpy()
    bad = [qi for qi in range(len(Q)) if not np.array_equal(a[qi], b[qi])]
    print("T", T, "mismatching queries", len(bad))
    for qi in bad[:3]:
        miss = [i for i in b[qi] if i not in a[qi]]
        print(" q", qi, "dense", a[qi][:10], "ref", b[qi][:10], "missing", miss, "parts", [int(part[i]) for i in miss], "pos", [int(pos_of[i]) for i in miss])
