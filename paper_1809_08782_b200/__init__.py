"""B200-native norm-ranging LSH (RANGE-LSH, arXiv 1809.08782) for MIPS.

Python face of ``libnrlsh.so`` (C ABI in ``include/nrlsh.h``): index build
(Alg. 1), batched query (Alg. 2 + multi-probe over the sorted (U_j, l)
structure), exact brute-force top-k.  All compute runs in the library's
hand-written sm_100a kernels; PyTorch only provides device memory and streams.
"""
from ._native import (EXPORTS, LIB_PATH, Index, NrlshError, exact_topk, last_exact_stats,
                      last_query_stats, last_rerank_path, last_rerank_stats, last_scan_stats, launch_count, lib, profile_enable,
                      profile_read)

__all__ = ["Index", "exact_topk", "last_query_stats", "last_scan_stats", "last_rerank_path", "last_rerank_stats", "NrlshError", "lib",
           "LIB_PATH", "EXPORTS", "profile_enable", "profile_read", "launch_count",
           "last_exact_stats"]
