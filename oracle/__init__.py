"""CPU fp64 oracle for the norm-ranging LSH hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1809_08782_b200``) never imports it and shares no code
with it.  This module is argument marshalling (numpy <-> ctypes) around
``nrlsh_oracle.c``; every step of the arithmetic lives in that C file, which
cites the paper passage each function follows.

Parity status: every function is pinned by tests/test_oracle_pins.py except
recall against the paper's own datasets ("parity unpinned").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nrlsh_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
             "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _declare(_lib)
    return _lib


_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int32
_u64 = C.c_uint64
_f64 = C.c_double


def _declare(L):
    L.orc_norm2.argtypes = [_p, _i64, _i32, _p]
    L.orc_norm2.restype = None
    L.orc_partition.argtypes = [_p, _i64, _i32, _p, _p, _p, _p]
    L.orc_partition.restype = C.c_int
    L.orc_partition_uniform.argtypes = [_p, _i64, _i32, _p, _p, _p, _p]
    L.orc_partition_uniform.restype = C.c_int
    L.orc_transform.argtypes = [_p, _i32, _f64, _f64, _p]
    L.orc_transform.restype = None
    L.orc_projection.argtypes = [_u64, _i32, _i32, _p]
    L.orc_projection.restype = None
    L.orc_item_codes.argtypes = [_p, _i64, _i32, _p, _p, _p, _p, _i32, _p, _p]
    L.orc_item_codes.restype = C.c_int
    L.orc_query_codes.argtypes = [_p, _i64, _i32, _p, _i32, _p, _p]
    L.orc_query_codes.restype = C.c_int
    L.orc_hamming.argtypes = [_p, _p, _i32]
    L.orc_hamming.restype = _i32
    L.orc_s_hat.argtypes = [_f64, _i32, _i32, _f64]
    L.orc_s_hat.restype = _f64
    L.orc_rank_table.argtypes = [_p, _i32, _i32, _f64, _p, _p]
    L.orc_rank_table.restype = C.c_int
    L.orc_candidates.argtypes = [_p, _p, _i64, _i32, _p, _p, _i32, _i64, _p, _p]
    L.orc_candidates.restype = _i64
    L.orc_rerank.argtypes = [_p, _i64, _i32, _p, _p, _i64, _i32, _p, _p]
    L.orc_rerank.restype = C.c_int
    L.orc_exact_topk.argtypes = [_p, _i64, _i32, _p, _i32, _p, _p]
    L.orc_exact_topk.restype = C.c_int
    L.orc_query.argtypes = [_p, _i64, _i32, _p, _p, _p, _i32, _p, _i32, _p, _i64, _i32,
                            _p, _p]
    L.orc_query.restype = C.c_int
    L.orc_projection_pp.argtypes = [_u64, _i32, _i32, _i32, _p]
    L.orc_projection_pp.restype = None
    L.orc_item_codes_pp.argtypes = [_p, _i64, _i32, _p, _p, _p, _p, _i32, _p, _p]
    L.orc_item_codes_pp.restype = C.c_int
    L.orc_query_codes_pp.argtypes = [_p, _i64, _i32, _p, _i32, _i32, _p, _p]
    L.orc_query_codes_pp.restype = C.c_int
    L.orc_candidates_pp.argtypes = [_p, _p, _i64, _i32, _p, _p, _i32, _i64, _p, _p]
    L.orc_candidates_pp.restype = _i64
    L.orc_query_pp.argtypes = [_p, _i64, _i32, _p, _p, _p, _i32, _p, _i32, _p, _i64, _i32,
                               _p, _p]
    L.orc_query_pp.restype = C.c_int


def _c(a, dtype):
    a = np.ascontiguousarray(a, dtype=dtype)
    return a


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _check(rc, what):
    if rc < 0:
        raise ValueError(f"oracle {what} failed with code {rc}")


# ---------------------------------------------------------------- build side
def norm2(X):
    X = _c(X, np.float32)
    n, d = X.shape
    out = np.empty(n, np.float64)
    lib().orc_norm2(_ptr(X), n, d, _ptr(out))
    return out


def partition(norm2_, m, scheme="percentile"):
    """Returns (part[n] int32, perm[n] int32, offsets[m+1] int64, V[m] fp64)."""
    nv = _c(norm2_, np.float64)
    n = nv.shape[0]
    part = np.empty(n, np.int32)
    perm = np.empty(n, np.int32)
    offsets = np.empty(m + 1, np.int64)
    V = np.empty(m, np.float64)
    fn = lib().orc_partition if scheme == "percentile" else lib().orc_partition_uniform
    _check(fn(_ptr(nv), n, m, _ptr(part), _ptr(perm), _ptr(offsets), _ptr(V)), "partition")
    return part, perm, offsets, V


def transform(x, Vj, norm2x):
    x = _c(x, np.float32)
    d = x.shape[0]
    out = np.empty(d + 1, np.float64)
    lib().orc_transform(_ptr(x), d, float(Vj), float(norm2x), _ptr(out))
    return out


def projection(seed, rows, L):
    A = np.empty((rows, L), np.float32)
    lib().orc_projection(C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), rows, L, _ptr(A))
    return A


def item_codes(X, part, V, norm2_, A, want_z=False):
    X = _c(X, np.float32)
    n, d = X.shape
    A = _c(A, np.float32)
    L = A.shape[1]
    assert A.shape[0] == d + 1
    codes = np.empty((n, (L + 31) // 32), np.uint32)
    z = np.empty((n, L), np.float64) if want_z else None
    part = _c(part, np.int32)
    V = _c(V, np.float64)
    nv = _c(norm2_, np.float64)
    rc = lib().orc_item_codes(_ptr(X), n, d, _ptr(part), _ptr(V), _ptr(nv), _ptr(A), L,
                              _ptr(codes), _ptr(z) if z is not None else None)
    _check(rc, "item_codes")
    return (codes, z) if want_z else codes


def item_codes_parallel(X, part, V, norm2_, A, threads=None, chunk=1 << 15):
    """item_codes over row chunks on host threads (ctypes releases the GIL); each
    item's arithmetic is unchanged -- the oracle is a per-item function."""
    from concurrent.futures import ThreadPoolExecutor
    X = _c(X, np.float32)
    n = X.shape[0]
    L = A.shape[1]
    out = np.empty((n, (L + 31) // 32), np.uint32)
    part = _c(part, np.int32)
    nv = _c(norm2_, np.float64)

    def work(r0):
        r1 = min(n, r0 + chunk)
        out[r0:r1] = item_codes(X[r0:r1], part[r0:r1], V, nv[r0:r1], A)

    with ThreadPoolExecutor(max_workers=threads or os.cpu_count()) as ex:
        list(ex.map(work, range(0, n, chunk)))
    return out


def query_codes(Q, A, want_z=False):
    Q = _c(Q, np.float32)
    nq, d = Q.shape
    A = _c(A, np.float32)
    L = A.shape[1]
    qcodes = np.empty((nq, (L + 31) // 32), np.uint32)
    z = np.empty((nq, L), np.float64) if want_z else None
    rc = lib().orc_query_codes(_ptr(Q), nq, d, _ptr(A), L, _ptr(qcodes),
                               _ptr(z) if z is not None else None)
    _check(rc, "query_codes")
    return (qcodes, z) if want_z else qcodes


def hamming(a, b):
    a = _c(a, np.uint32)
    b = _c(b, np.uint32)
    return int(lib().orc_hamming(_ptr(a), _ptr(b), a.shape[0]))


def s_hat(Uj, h, L, eps):
    return float(lib().orc_s_hat(float(Uj), int(h), int(L), float(eps)))


def rank_table(U, L, eps=0.01):
    """Returns (R[m, L+1] uint16, order[m*(L+1)] int32 = j*(L+1)+h by position)."""
    U = _c(U, np.float64)
    m = U.shape[0]
    R = np.empty((m, L + 1), np.uint16)
    order = np.empty(m * (L + 1), np.int32)
    _check(lib().orc_rank_table(_ptr(U), m, L, float(eps), _ptr(R), _ptr(order)), "rank_table")
    return R, order


def candidates(codes, part, qcode, R, T):
    """codes in item-id order.  Returns (ids[T'] int32, rank[T'] uint16)."""
    codes = _c(codes, np.uint32)
    n, W = codes.shape
    R = _c(R, np.uint16)
    m, L = R.shape[0], R.shape[1] - 1
    Tp = min(int(T), n)
    ids = np.empty(Tp, np.int32)
    rk = np.empty(Tp, np.uint16)
    got = lib().orc_candidates(_ptr(codes), _ptr(_c(part, np.int32)), n, L,
                               _ptr(_c(qcode, np.uint32)), _ptr(R), m, int(T),
                               _ptr(ids), _ptr(rk))
    _check(got, "candidates")
    return ids[:got], rk[:got]


def rerank(X, q, cand_ids, k):
    X = _c(X, np.float32)
    n, d = X.shape
    cand = _c(cand_ids, np.int32)
    ids = np.empty(k, np.int64)
    sc = np.empty(k, np.float64)
    _check(lib().orc_rerank(_ptr(X), n, d, _ptr(_c(q, np.float32)), _ptr(cand), cand.shape[0],
                            k, _ptr(ids), _ptr(sc)), "rerank")
    return ids, sc


def exact_topk(X, q, k):
    X = _c(X, np.float32)
    n, d = X.shape
    ids = np.empty(k, np.int64)
    sc = np.empty(k, np.float64)
    _check(lib().orc_exact_topk(_ptr(X), n, d, _ptr(_c(q, np.float32)), k, _ptr(ids),
                                _ptr(sc)), "exact_topk")
    return ids, sc


def query(X, codes, part, R, A, q, T, k):
    X = _c(X, np.float32)
    n, d = X.shape
    codes = _c(codes, np.uint32)
    R = _c(R, np.uint16)
    L = R.shape[1] - 1
    ids = np.empty(k, np.int64)
    sc = np.empty(k, np.float64)
    rc = lib().orc_query(_ptr(X), n, d, _ptr(codes), _ptr(_c(part, np.int32)), _ptr(R),
                         R.shape[0], _ptr(_c(A, np.float32)), L, _ptr(_c(q, np.float32)),
                         int(T), int(k), _ptr(ids), _ptr(sc))
    _check(rc, "query")
    return ids, sc


# ---------------------------------------- per-sub-dataset projections (NEXT-4)
def projection_pp(seed, m, rows, L):
    """A_all [m, rows, L]: A_j from seed ^ j."""
    A = np.empty((m, rows, L), np.float32)
    lib().orc_projection_pp(C.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), m, rows, L, _ptr(A))
    return A


def item_codes_pp(X, part, V, norm2_, A_all, want_z=False):
    X = _c(X, np.float32)
    n, d = X.shape
    A_all = _c(A_all, np.float32)
    L = A_all.shape[2]
    assert A_all.shape[1] == d + 1
    codes = np.empty((n, (L + 31) // 32), np.uint32)
    z = np.empty((n, L), np.float64) if want_z else None
    rc = lib().orc_item_codes_pp(_ptr(X), n, d, _ptr(_c(part, np.int32)), _ptr(_c(V, np.float64)),
                                 _ptr(_c(norm2_, np.float64)), _ptr(A_all), L, _ptr(codes),
                                 _ptr(z) if z is not None else None)
    _check(rc, "item_codes_pp")
    return (codes, z) if want_z else codes


def item_codes_pp_parallel(X, part, V, norm2_, A_all, threads=None, chunk=1 << 15):
    from concurrent.futures import ThreadPoolExecutor
    X = _c(X, np.float32)
    n = X.shape[0]
    L = A_all.shape[2]
    out = np.empty((n, (L + 31) // 32), np.uint32)
    part = _c(part, np.int32)
    nv = _c(norm2_, np.float64)

    def work(r0):
        r1 = min(n, r0 + chunk)
        out[r0:r1] = item_codes_pp(X[r0:r1], part[r0:r1], V, nv[r0:r1], A_all)

    with ThreadPoolExecutor(max_workers=threads or os.cpu_count()) as ex:
        list(ex.map(work, range(0, n, chunk)))
    return out


def query_codes_pp(Q, A_all, want_z=False):
    """qcodes [nq, m, W] (and z [nq, m, L])."""
    Q = _c(Q, np.float32)
    nq, d = Q.shape
    A_all = _c(A_all, np.float32)
    m, L = A_all.shape[0], A_all.shape[2]
    W = (L + 31) // 32
    qc = np.empty((nq, m, W), np.uint32)
    z = np.empty((nq, m, L), np.float64) if want_z else None
    rc = lib().orc_query_codes_pp(_ptr(Q), nq, d, _ptr(A_all), m, L, _ptr(qc),
                                  _ptr(z) if z is not None else None)
    _check(rc, "query_codes_pp")
    return (qc, z) if want_z else qc


def candidates_pp(codes, part, qcodes_m, R, T):
    """qcodes_m [m, W]: the query's code under each sub-index's projection."""
    codes = _c(codes, np.uint32)
    n, W = codes.shape
    R = _c(R, np.uint16)
    m, L = R.shape[0], R.shape[1] - 1
    Tp = min(int(T), n)
    ids = np.empty(Tp, np.int32)
    rk = np.empty(Tp, np.uint16)
    got = lib().orc_candidates_pp(_ptr(codes), _ptr(_c(part, np.int32)), n, L,
                                  _ptr(_c(qcodes_m, np.uint32)), _ptr(R), m, int(T),
                                  _ptr(ids), _ptr(rk))
    _check(got, "candidates_pp")
    return ids[:got], rk[:got]


def query_pp(X, codes, part, R, A_all, q, T, k):
    X = _c(X, np.float32)
    n, d = X.shape
    R = _c(R, np.uint16)
    L = R.shape[1] - 1
    ids = np.empty(k, np.int64)
    sc = np.empty(k, np.float64)
    rc = lib().orc_query_pp(_ptr(X), n, d, _ptr(_c(codes, np.uint32)), _ptr(_c(part, np.int32)),
                            _ptr(R), R.shape[0], _ptr(_c(A_all, np.float32)), L,
                            _ptr(_c(q, np.float32)), int(T), int(k), _ptr(ids), _ptr(sc))
    _check(rc, "query_pp")
    return ids, sc


# ------------------------------------------------------------- whole index
class OracleIndex:
    """Alg. 1 end to end on the CPU (D1-D5, D8-D9)."""

    def __init__(self, X, code_bits, num_parts, seed, eps=0.01, scheme="percentile",
                 proj="shared"):
        self.X = _c(X, np.float32)
        n, d = self.X.shape
        self.L = int(code_bits)
        self.m = int(num_parts)
        self.eps = float(eps)
        self.norm2 = norm2(self.X)
        self.part, self.perm, self.offsets, self.V = partition(self.norm2, self.m, scheme)
        self.U = np.sqrt(self.V)
        self.proj = proj
        self.A = projection(seed, d + 1, self.L)
        # per-sub-dataset projections (A_all[j] = A_j; A_all[0] == A)
        self.A_all = projection_pp(seed, self.m, d + 1, self.L) if proj == "per_partition" else None
        self.R, self.order = rank_table(self.U, self.L, self.eps)

    def codes(self, want_z=False):
        if self.proj == "per_partition":
            return item_codes_pp(self.X, self.part, self.V, self.norm2, self.A_all, want_z=want_z)
        return item_codes(self.X, self.part, self.V, self.norm2, self.A, want_z=want_z)

    def query_codes(self, Q, want_z=False):
        if self.proj == "per_partition":
            return query_codes_pp(Q, self.A_all, want_z=want_z)
        return query_codes(Q, self.A, want_z=want_z)

    def candidates(self, codes, qcode, T):
        if self.proj == "per_partition":
            return candidates_pp(codes, self.part, qcode, self.R, T)
        return candidates(codes, self.part, qcode, self.R, T)

    def query(self, codes, q, T, k):
        if self.proj == "per_partition":
            return query_pp(self.X, codes, self.part, self.R, self.A_all, q, T, k)
        return query(self.X, codes, self.part, self.R, self.A, q, T, k)


def recall_at_k(ret_ids, true_ids):
    """D12: |returned ∩ truth| / k, macro-averaged over queries (rows)."""
    ret_ids = np.asarray(ret_ids)
    true_ids = np.asarray(true_ids)
    k = true_ids.shape[1]
    tot = 0.0
    for r, t in zip(ret_ids, true_ids):
        tot += len(set(int(x) for x in r if x >= 0) & set(int(x) for x in t if x >= 0)) / k
    return tot / max(1, ret_ids.shape[0])
