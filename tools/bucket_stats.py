"""Bucket-balance diagnostics: distinct codes
and the largest bucket, for SIMPLE-LSH (m = 1) and RANGE-LSH (m sub-datasets, a bucket
= (sub-dataset, code)), on a config's synthetic items.
usage: python tools/bucket_stats.py [config] [code_bits] [out.json]"""
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
L = int(sys.argv[2]) if len(sys.argv) > 2 else 32
cfg = workloads.CONFIGS[name]
X = torch.from_numpy(workloads.make_items(cfg)).cuda()
rows = []
for m in sorted({1, *cfg.num_parts, 32, 128}):
    if m > cfg.n:
        continue
    idx = P.Index(X, L, m, seed=cfg.seed)
    codes = idx.codes()                      # partition order
    _, perm, off, _ = idx.partition()
    part = np.repeat(np.arange(m, dtype=np.uint32), np.diff(off))
    keys = np.ascontiguousarray(np.column_stack([part, codes.astype(np.uint32)]))
    _, counts = np.unique(keys.view(np.dtype((np.void, keys.dtype.itemsize * keys.shape[1]))),
                          return_counts=True)
    row = {"config": name, "code_bits": L, "num_parts": m, "n": int(idx.n),
           "buckets": int(len(counts)), "largest_bucket": int(counts.max()),
           "items_in_largest_1pct_buckets": int(np.sort(counts)[::-1][:max(1, len(counts) // 100)].sum())}
    rows.append(row)
    print(json.dumps(row), flush=True)
    idx.close()
if len(sys.argv) > 3:
    json.dump(rows, open(sys.argv[3], "w"), indent=1)
