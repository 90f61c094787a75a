import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1809_08782_b200 as P, workloads
cfg = workloads.CONFIGS["c4"]
X = torch.from_numpy(workloads.make_items(cfg)).cuda()
Q = torch.from_numpy(workloads.make_queries(cfg)).cuda()
idx = P.Index(X, 64, 128, seed=cfg.seed, query_batch=1024, index_bits_in_budget=True)
for T in (2341, 4096):
    for b in range(0, 10000, 1024):
        idx.candidates(T, queries=Q[b:b + 1024].contiguous())
        st = P.last_query_stats()
        if st["fallback_queries"]:
            print("T", T, "batch", b, st, flush=True)
            for qq in range(b, min(b + 1024, 10000)):
                idx.candidates(T, queries=Q[qq:qq + 1].contiguous())
                if P.last_query_stats()["fallback_queries"]:
                    print("  alone fails:", qq, flush=True)
print("done")
