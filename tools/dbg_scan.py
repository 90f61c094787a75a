import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_1809_08782_b200 as P, workloads, oracle
cfg = workloads.CONFIGS["tiny"]
X = workloads.make_items(cfg); Q = workloads.make_queries(cfg)
idx = P.Index(torch.from_numpy(X).cuda(), 32, 8, seed=0)
try:
    ids, rk = idx.candidates(100, queries=torch.from_numpy(Q[:16]).cuda())
    print("ok", ids[0][:5])
except Exception as e:
    print("ERR", e)
