import os, sys
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1809_08782_b200 as P, workloads
cfg = workloads.CONFIGS["c4"]
X = torch.from_numpy(workloads.make_items(cfg)).cuda()
Q = torch.from_numpy(workloads.make_queries(cfg)).cuda()
for m in (64, 128, 256):
    idx = P.Index(X, 64, m, seed=cfg.seed, query_batch=1024, index_bits_in_budget=True)
    for T in (2341, 4096):
        idx.query(Q[:256], 10, T)
        P.profile_enable(True); P.profile_read(reset=True)
        torch.cuda.synchronize()
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); idx.query(Q, 10, T); e1.record(); torch.cuda.synchronize()
        pr={k: round(v[0],3) for k,v in P.profile_read(reset=True).items() if v[1]}
        print(m, idx.hash_bits, T, round(e0.elapsed_time(e1),2), P.last_query_stats(), P.last_rerank_path(), pr, flush=True)
    idx.close()
