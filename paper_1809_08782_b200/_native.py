"""ctypes binding of libnrlsh.so (include/nrlsh.h) — argument marshalling only.

Every step of the method runs in the library's sm_100a kernels; this module
only converts torch tensors / numpy arrays into pointers, allocates outputs and
maps status codes to exceptions.  There is no fallback: if the shared library
is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnrlsh.so")

_STATUS = {0: "OK", 1: "EINVAL", 2: "ENONFINITE", 3: "EZERONORM", 4: "ENOMEM", 5: "ECUDA",
           6: "ENOTIMPL"}

EXPORTS = [
    "nrlsh_default_options", "nrlsh_build", "nrlsh_build_ex", "nrlsh_query", "nrlsh_exact_topk",
    "nrlsh_free", "nrlsh_last_error", "nrlsh_get_info", "nrlsh_get_partition",
    "nrlsh_get_projection", "nrlsh_get_rank_table", "nrlsh_get_codes", "nrlsh_set_codes",
    "nrlsh_query_codes", "nrlsh_query_candidates", "nrlsh_last_query_stats", "nrlsh_last_scan_stats", "nrlsh_last_scan_popc",
    "nrlsh_index_exact_topk", "nrlsh_exact_topk_seeded", "nrlsh_index_exact_topk_seeded",
    "nrlsh_last_rerank_stats", "nrlsh_last_rerank_path", "nrlsh_profile_enable", "nrlsh_profile_read",
    "nrlsh_profile_slot_name", "nrlsh_launch_count", "nrlsh_last_exact_stats", "nrlsh_get_proj",
]


class NrlshError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status
        self.code = _STATUS.get(status, str(status))


class Options(C.Structure):
    _fields_ = [("eps", C.c_double), ("scheme", C.c_int32), ("index_bits_in_budget", C.c_int32),
                ("query_batch", C.c_int32), ("proj", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c \"import __graft_entry__ as g; "
                "g.build()\"` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        p, i64, i32, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64
        st = C.c_int
        L.nrlsh_default_options.argtypes = [C.POINTER(Options)]
        L.nrlsh_default_options.restype = None
        L.nrlsh_build.argtypes = [p, i64, i32, i32, i32, u64, C.POINTER(p), p]
        L.nrlsh_build.restype = st
        L.nrlsh_build_ex.argtypes = [p, i64, i32, i32, i32, u64, C.POINTER(Options), C.POINTER(p), p]
        L.nrlsh_build_ex.restype = st
        L.nrlsh_query.argtypes = [p, p, i64, i32, i64, p, p, p]
        L.nrlsh_query.restype = st
        L.nrlsh_exact_topk.argtypes = [p, i64, i32, p, i64, i32, p, p, p]
        L.nrlsh_exact_topk.restype = st
        L.nrlsh_free.argtypes = [p]
        L.nrlsh_free.restype = None
        L.nrlsh_last_error.argtypes = []
        L.nrlsh_last_error.restype = C.c_char_p
        L.nrlsh_get_info.argtypes = [p, p, p, p, p, p]
        L.nrlsh_get_info.restype = st
        L.nrlsh_get_proj.argtypes = [p, p]
        L.nrlsh_get_proj.restype = st
        L.nrlsh_get_partition.argtypes = [p, p, p, p, p]
        L.nrlsh_get_partition.restype = st
        L.nrlsh_get_projection.argtypes = [p, p]
        L.nrlsh_get_projection.restype = st
        L.nrlsh_get_rank_table.argtypes = [p, p]
        L.nrlsh_get_rank_table.restype = st
        L.nrlsh_get_codes.argtypes = [p, p]
        L.nrlsh_get_codes.restype = st
        L.nrlsh_set_codes.argtypes = [p, p]
        L.nrlsh_set_codes.restype = st
        L.nrlsh_query_codes.argtypes = [p, p, i64, p, p]
        L.nrlsh_query_codes.restype = st
        L.nrlsh_query_candidates.argtypes = [p, p, p, i64, i64, p, p, p]
        L.nrlsh_query_candidates.restype = st
        L.nrlsh_last_query_stats.argtypes = [p, p, p, p]
        L.nrlsh_last_query_stats.restype = st
        L.nrlsh_last_scan_stats.argtypes = [p, p]
        L.nrlsh_last_scan_stats.restype = st
        L.nrlsh_last_scan_popc.argtypes = [p]
        L.nrlsh_last_scan_popc.restype = st
        L.nrlsh_index_exact_topk.argtypes = [p, p, i64, i32, p, p, p]
        L.nrlsh_index_exact_topk.restype = st
        L.nrlsh_exact_topk_seeded.argtypes = [p, i64, i32, p, i64, i32, p, i32, p, p, p]
        L.nrlsh_exact_topk_seeded.restype = st
        L.nrlsh_index_exact_topk_seeded.argtypes = [p, p, i64, i32, p, i32, p, p, p]
        L.nrlsh_index_exact_topk_seeded.restype = st
        L.nrlsh_profile_enable.argtypes = [C.c_int]
        L.nrlsh_profile_enable.restype = None
        L.nrlsh_profile_read.argtypes = [p, p, i32, C.c_int]
        L.nrlsh_profile_read.restype = C.c_int
        L.nrlsh_profile_slot_name.argtypes = [i32]
        L.nrlsh_profile_slot_name.restype = C.c_char_p
        L.nrlsh_last_rerank_stats.argtypes = [p]
        L.nrlsh_last_rerank_stats.restype = st
        L.nrlsh_last_rerank_path.argtypes = [p, p, p]
        L.nrlsh_last_rerank_path.restype = st
        L.nrlsh_last_exact_stats.argtypes = [p, p, p, p]
        L.nrlsh_last_exact_stats.restype = st
        L.nrlsh_launch_count.argtypes = []
        L.nrlsh_launch_count.restype = C.c_int64
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise NrlshError(rc, lib().nrlsh_last_error().decode())


def _ptr(a):
    """Pointer of a torch tensor (device or host) or numpy array (host)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return C.c_void_p(a.ctypes.data)
    assert a.is_contiguous()
    return C.c_void_p(a.data_ptr())


_NP_OF = {"float32": np.float32, "int64": np.int64, "int32": np.int32, "uint32": np.uint32,
          "uint16": np.uint16}


def _want(a, name, dtypes, shape=None, device=None):
    """Validate an array before its raw pointer crosses the ABI (which cannot check
    dtype, width or device itself): C-contiguous, one of `dtypes` (numpy names;
    int32/uint32 and int16/uint16 are interchangeable bit containers), `shape` (None
    entries are free), and for torch tensors on the index's device (or the host)."""
    if a is None:
        raise ValueError(f"{name} is None")
    if isinstance(a, np.ndarray):
        dt = a.dtype.name
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name} must be C-contiguous")
    else:
        dt = str(a.dtype).replace("torch.", "")
        if not a.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if device is not None and a.is_cuda and a.device != device:
            raise ValueError(f"{name} is on {a.device}, the index on {device}")
    alias = {"int32": "uint32", "uint32": "int32", "int16": "uint16", "uint16": "int16"}
    if dt not in dtypes and alias.get(dt) not in dtypes:
        raise TypeError(f"{name} must be {'/'.join(dtypes)}, got {dt}")
    if shape is not None:
        got = tuple(a.shape)
        if len(got) != len(shape) or any(w is not None and g != w for g, w in zip(got, shape)):
            raise ValueError(f"{name} must have shape {shape} (None = any), got {got}")
    return a


def _dev_of(a):
    return None if isinstance(a, np.ndarray) or not a.is_cuda else a.device


def _stream(stream):
    if stream is not None:
        return C.c_void_p(int(stream))
    try:
        import torch
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    except Exception:
        pass
    return None


def _is_np(a):
    return isinstance(a, np.ndarray)


def _empty_like_io(ref, shape, np_dtype, torch_dtype):
    if _is_np(ref):
        return np.empty(shape, np_dtype)
    import torch
    return torch.empty(shape, dtype=torch_dtype, device=ref.device)


class Index:
    """An nrlsh_index handle (Alg. 1).  Keeps the item buffer alive (borrowed)."""

    def __init__(self, items, code_bits, num_parts, seed=0, eps=0.01, scheme="percentile",
                 index_bits_in_budget=False, query_batch=0, stream=None, proj="shared"):
        _want(items, "items", ("float32",), (None, None))
        self._items = items
        self._device = _dev_of(items)
        opt = Options()
        lib().nrlsh_default_options(C.byref(opt))
        opt.eps = float(eps)
        opt.scheme = {"percentile": 0, "uniform": 1}[scheme]
        opt.index_bits_in_budget = 1 if index_bits_in_budget else 0
        opt.query_batch = int(query_batch)
        opt.proj = {"shared": 0, "per_partition": 1}[proj]
        n, d = items.shape
        h = C.c_void_p()
        _check(lib().nrlsh_build_ex(_ptr(items), n, d, int(code_bits), int(num_parts),
                                    C.c_uint64(seed & (2 ** 64 - 1)), C.byref(opt), C.byref(h),
                                    _stream(stream)))
        self._h = h
        ni, di, hb, npart, w = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(lib().nrlsh_get_info(h, C.byref(ni), C.byref(di), C.byref(hb), C.byref(npart),
                                    C.byref(w)))
        self.n, self.d, self.hash_bits, self.num_parts, self.words = (
            ni.value, di.value, hb.value, npart.value, w.value)
        pj = C.c_int32()
        _check(lib().nrlsh_get_proj(h, C.byref(pj)))
        self.proj = "per_partition" if pj.value == 1 else "shared"
        # query codes per query: one, or one per sub-index (A_j)
        self.qm = self.num_parts if self.proj == "per_partition" else 1

    def _qshape(self, nq):
        return (nq, self.qm, self.words) if self.qm > 1 else (nq, self.words)

    def close(self):
        if getattr(self, "_h", None):
            lib().nrlsh_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- query
    def query(self, queries, k, probe_budget, out_ids=None, out_scores=None, stream=None):
        _want(queries, "queries", ("float32",), (None, self.d), self._device)
        nq = queries.shape[0]
        if out_ids is None:
            out_ids = _empty_like_io(queries, (nq, k), np.int64, _torch_dtype("int64"))
        if out_scores is None:
            out_scores = _empty_like_io(queries, (nq, k), np.float32, _torch_dtype("float32"))
        _want(out_ids, "out_ids", ("int64",), (nq, k), self._device)
        _want(out_scores, "out_scores", ("float32",), (nq, k), self._device)
        _check(lib().nrlsh_query(self._h, _ptr(queries), nq, int(k), int(probe_budget),
                                 _ptr(out_ids), _ptr(out_scores), _stream(stream)))
        return out_ids, out_scores

    def exact_topk(self, queries, k, out_ids=None, out_scores=None, stream=None, seed_ids=None):
        """Ground truth against the index's own items (no re-staging of host items).
        seed_ids [nq x ks] int64 (optional): warm-start ids, e.g. query()'s answers;
        the result does not depend on them."""
        _want(queries, "queries", ("float32",), (None, self.d), self._device)
        nq = queries.shape[0]
        if out_ids is None:
            out_ids = _empty_like_io(queries, (nq, k), np.int64, _torch_dtype("int64"))
        if out_scores is None:
            out_scores = _empty_like_io(queries, (nq, k), np.float32, _torch_dtype("float32"))
        _want(out_ids, "out_ids", ("int64",), (nq, k), self._device)
        _want(out_scores, "out_scores", ("float32",), (nq, k), self._device)
        if seed_ids is not None:
            _want(seed_ids, "seed_ids", ("int64",), (nq, None), self._device)
        if seed_ids is None:
            _check(lib().nrlsh_index_exact_topk(self._h, _ptr(queries), nq, int(k), _ptr(out_ids),
                                                _ptr(out_scores), _stream(stream)))
        else:
            _check(lib().nrlsh_index_exact_topk_seeded(
                self._h, _ptr(queries), nq, int(k), _ptr(seed_ids), int(seed_ids.shape[1]),
                _ptr(out_ids), _ptr(out_scores), _stream(stream)))
        return out_ids, out_scores

    def query_codes(self, queries, stream=None):
        _want(queries, "queries", ("float32",), (None, self.d), self._device)
        nq = queries.shape[0]
        out = _empty_like_io(queries, self._qshape(nq), np.uint32, _torch_dtype("int32"))
        _check(lib().nrlsh_query_codes(self._h, _ptr(queries), nq, _ptr(out), _stream(stream)))
        return out

    def candidates(self, probe_budget, queries=None, qcodes=None, stream=None):
        ref = queries if queries is not None else qcodes
        if queries is not None:
            _want(queries, "queries", ("float32",), (None, self.d), self._device)
        if qcodes is not None:
            _want(qcodes, "qcodes", ("uint32",), self._qshape(None), self._device)
            if queries is not None and queries.shape[0] != qcodes.shape[0]:
                raise ValueError("queries and qcodes disagree on nq")
        nq = ref.shape[0]
        T = min(int(probe_budget), self.n)
        ids = _empty_like_io(ref, (nq, T), np.int32, _torch_dtype("int32"))
        rk = _empty_like_io(ref, (nq, T), np.uint16, _torch_dtype("int16"))
        _check(lib().nrlsh_query_candidates(self._h, _ptr(queries), _ptr(qcodes), nq,
                                            int(probe_budget), _ptr(ids), _ptr(rk),
                                            _stream(stream)))
        return ids, rk

    # -------------------------------------------------------------- hooks (host copies)
    def partition(self):
        norm2 = np.empty(self.n, np.float64)
        perm = np.empty(self.n, np.int32)
        offsets = np.empty(self.num_parts + 1, np.int64)
        V = np.empty(self.num_parts, np.float64)
        _check(lib().nrlsh_get_partition(self._h, _ptr(norm2), _ptr(perm), _ptr(offsets),
                                         _ptr(V)))
        return norm2, perm, offsets, V

    def projection(self):
        """A [(d+1) x L_h]; per-sub-dataset projections: [m x (d+1) x L_h], A[j] = A_j."""
        shp = (self.d + 1, self.hash_bits)
        A = np.empty(((self.qm,) + shp) if self.qm > 1 else shp, np.float32)
        _check(lib().nrlsh_get_projection(self._h, _ptr(A)))
        return A

    def rank_table(self):
        R = np.empty((self.num_parts, self.hash_bits + 1), np.uint16)
        _check(lib().nrlsh_get_rank_table(self._h, _ptr(R)))
        return R

    def codes(self):
        c = np.empty((self.n, self.words), np.uint32)
        _check(lib().nrlsh_get_codes(self._h, _ptr(c)))
        return c

    def set_codes(self, codes):
        codes = np.ascontiguousarray(codes, dtype=np.uint32)
        assert codes.shape == (self.n, self.words)
        _check(lib().nrlsh_set_codes(self._h, _ptr(codes)))


def _torch_dtype(name):
    import torch
    return getattr(torch, name)


def exact_topk(items, queries, k, out_ids=None, out_scores=None, stream=None, seed_ids=None):
    _want(items, "items", ("float32",), (None, None))
    n, d = items.shape
    dev = _dev_of(items)
    _want(queries, "queries", ("float32",), (None, d), dev)
    nq = queries.shape[0]
    if out_ids is None:
        out_ids = _empty_like_io(queries, (nq, k), np.int64, _torch_dtype("int64"))
    if out_scores is None:
        out_scores = _empty_like_io(queries, (nq, k), np.float32, _torch_dtype("float32"))
    _want(out_ids, "out_ids", ("int64",), (nq, k), dev)
    _want(out_scores, "out_scores", ("float32",), (nq, k), dev)
    if seed_ids is not None:
        _want(seed_ids, "seed_ids", ("int64",), (nq, None), dev)
    if seed_ids is None:
        _check(lib().nrlsh_exact_topk(_ptr(items), n, d, _ptr(queries), nq, int(k), _ptr(out_ids),
                                      _ptr(out_scores), _stream(stream)))
    else:
        _check(lib().nrlsh_exact_topk_seeded(_ptr(items), n, d, _ptr(queries), nq, int(k),
                                             _ptr(seed_ids), int(seed_ids.shape[1]), _ptr(out_ids),
                                             _ptr(out_scores), _stream(stream)))
    return out_ids, out_scores


def last_rerank_stats():
    a = C.c_int64()
    _check(lib().nrlsh_last_rerank_stats(C.byref(a)))
    return {"rescored_fp32": a.value}


RERANK_PATHS = {0: "gather", 1: "tensor"}


def last_rerank_path():
    """Which re-rank implementation the last query on this thread used, and how many
    of its queries overflowed the tensor-core survivor list (re-ranked by gather)."""
    a, b, c = C.c_int32(), C.c_int64(), C.c_int64()
    _check(lib().nrlsh_last_rerank_path(C.byref(a), C.byref(b), C.byref(c)))
    return {"path": RERANK_PATHS.get(a.value, str(a.value)), "overflow_redone": b.value,
            "filter_pairs": c.value}


def last_query_stats():
    a, b, c, e = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    _check(lib().nrlsh_last_query_stats(C.byref(a), C.byref(b), C.byref(c), C.byref(e)))
    return {"fallback_queries": a.value, "kernel_launches": b.value, "scanned_pairs": c.value,
            "buffer_entries": e.value}


def last_scan_stats():
    """Pairs of the last query on which the scan's lower bound ran / which it decided alone."""
    a, b = C.c_int64(), C.c_int64()
    _check(lib().nrlsh_last_scan_stats(C.byref(a), C.byref(b)))
    p = C.c_int64()
    _check(lib().nrlsh_last_scan_popc(C.byref(p)))
    return {"bound_pairs": a.value, "bound_decided_pairs": b.value, "popc_ops": p.value}


def last_exact_stats():
    a, b, c, e = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    _check(lib().nrlsh_last_exact_stats(C.byref(a), C.byref(b), C.byref(c), C.byref(e)))
    return {"max_survivors": a.value, "sum_survivors": b.value, "overflow_queries": c.value,
            "filter_pairs": e.value}


def profile_enable(on=True):
    lib().nrlsh_profile_enable(1 if on else 0)


def profile_read(reset=False):
    """{slot name: (total ms, ranges)} of the library's per-kernel-class CUDA events."""
    n = 32
    ms = (C.c_double * n)()
    cnt = (C.c_int64 * n)()
    k = lib().nrlsh_profile_read(ms, cnt, n, 1 if reset else 0)
    return {lib().nrlsh_profile_slot_name(i).decode(): (ms[i], cnt[i]) for i in range(k)}


def launch_count():
    return int(lib().nrlsh_launch_count())
