"""GPU <-> oracle parity of every step of the hot path, through the C ABI.

Rules (BASELINE.json north_star):
  * partition (perm, offsets, V), norms, projection, rank table: bit-exact;
  * codes: bit-exact except bits whose fp64 projection |z| < 1e-5 * ||P(x)|| (= 1e-5);
  * Hamming scores, candidate sets (and their (R, id) order), returned ids:
    bit-exact when both sides are given identical codes;
  * inner products within 1e-4 relative; top-k ids equal except at ties within it.
Sizes: small cases the oracle finishes in seconds (several tiles + ragged
tails), and BASELINE.json's full sizes on sampled outputs.
"""
import os

import numpy as np
import pytest

import oracle
import workloads

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _P():
    import paper_1809_08782_b200 as P
    return P


@pytest.fixture(scope="session", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    P = _P()
    P.lib()


_DATA = {}


def dataset(cfg, n=None, nq=None):
    key = (cfg.name, n, nq)
    if key not in _DATA:
        c = cfg if n is None else workloads.scaled(cfg, n, nq or cfg.nq)
        X = workloads.make_items(c)
        Q = workloads.make_queries(c, nq=nq or c.nq)
        _DATA[key] = (c, X, Q)
    return _DATA[key]


def bits_of(codes, L):
    c = np.ascontiguousarray(codes, dtype=np.uint32)
    b = ((c[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(c.shape[0], -1)
    return b[:, :L].astype(bool)


def assert_codes_match(gpu_codes, orc_codes, z, L, band=1e-5):
    diff = bits_of(gpu_codes, L) != bits_of(orc_codes, L)
    bad = diff & (np.abs(z[:, :L]) >= band)
    assert not bad.any(), f"{bad.sum()} code bits differ with |z| >= {band}"
    # bits beyond L are zero on both sides
    if gpu_codes.shape[1] * 32 > L:
        allb = ((np.ascontiguousarray(gpu_codes)[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1)
        assert not allb.reshape(gpu_codes.shape[0], -1)[:, L:].any()
    return int(diff.sum())


def assert_topk_match(ids, scores, ref_ids, ref_scores, X, q, rtol=1e-4):
    """Scores within rtol of the oracle's fp64 values, relative to the larger of
    |score| and |q||x| (reading of north_star's "1e-4 relative": a score
    that cancels to ~0 carries fp32 rounding of size ~|q||x|); ids equal except
    where the swapped items' exact scores differ by no more than that tolerance."""
    ids = np.asarray(ids)
    valid = ref_ids >= 0
    assert np.array_equal(ids >= 0, valid)
    s_ref = ref_scores[valid]
    qn = float(np.linalg.norm(q.astype(np.float64)))
    xn = np.linalg.norm(X[ref_ids[valid]].astype(np.float64), axis=1)
    tol = rtol * np.maximum(np.abs(s_ref), qn * xn)
    got_s = np.asarray(scores)[valid].astype(np.float64)
    assert np.all(np.abs(got_s - s_ref) <= tol), (got_s, s_ref, tol)
    if np.array_equal(ids, ref_ids):
        return
    # differing positions must be near-ties: compare exact scores of the returned items
    got = ids[valid].astype(np.int64)
    exact = X[got].astype(np.float64) @ q.astype(np.float64)
    assert np.all(np.abs(exact - s_ref) <= tol), (ids, ref_ids)


def band_mask(gq, oq, frac=0.9):
    """Queries whose GPU and oracle query codes agree (a query bit inside the 1e-5
    band may differ, and then the probe order may legitimately differ).  At least
    `frac` of the queries must be comparable, so a test cannot pass by skipping."""
    same = np.array([np.array_equal(a, b) for a, b in zip(gq, oq)])
    assert same.mean() >= frac, f"only {same.sum()} of {len(same)} query codes agree"
    return same


# ------------------------------------------------------------------ configs
SMALL = [
    ("tiny", None, None, 32, 8),
    ("c2", None, 200, 64, 32),
    ("c3", 40_000, 64, 64, 64),
    ("c3", 40_000, 64, 64, 1),
    ("c3", None, 64, 64, 64),        # c3 at its full n (Yahoo!Music-shaped)
    ("c3", None, 64, 64, 1),         #   and plain SIMPLE-LSH on it
    ("c4", 300_000, 32, 32, 128),    # pilot stride > 1 (n > 2^18)
    ("c4", 300_000, 32, 64, 128),
    ("scale", 70_000, 16, 128, 256),
]


def _ids(case):
    return "-".join(str(x) for x in case)


@pytest.fixture(scope="session")
def built():
    cache = {}

    def get(name, n, nq, L, m, **kw):
        key = (name, n, nq, L, m, tuple(sorted(kw.items())))
        if key not in cache:
            P = _P()
            cfg, X, Q = dataset(workloads.CONFIGS[name], n, nq)
            Xd = torch.from_numpy(X).cuda()
            idx = P.Index(Xd, L, m, seed=cfg.seed, **kw)
            orc = oracle.OracleIndex(X, idx.hash_bits, m, seed=cfg.seed,
                                     eps=kw.get("eps", 0.01),
                                     scheme=kw.get("scheme", "percentile"))
            cache[key] = (cfg, X, Q, Xd, idx, orc)
        return cache[key]
    return get


@pytest.mark.parametrize("case", SMALL, ids=_ids)
def test_build_parity(built, case):
    cfg, X, Q, Xd, idx, orc = built(*case)
    norm2, perm, offsets, V = idx.partition()
    assert np.array_equal(norm2.view(np.uint64), orc.norm2.view(np.uint64))   # bit-exact
    assert np.array_equal(perm, orc.perm)
    assert np.array_equal(offsets, orc.offsets)
    assert np.array_equal(V, orc.V)
    assert np.array_equal(idx.projection(), orc.A)
    assert np.array_equal(idx.rank_table(), orc.R)
    ocodes, z = orc.codes(want_z=True)
    gcodes = idx.codes()[np.argsort(perm, kind="stable")]
    assert_codes_match(gcodes, ocodes, z, idx.hash_bits)


@pytest.mark.parametrize("case", SMALL, ids=_ids)
def test_query_codes_parity(built, case):
    cfg, X, Q, Xd, idx, orc = built(*case)
    g = idx.query_codes(torch.from_numpy(Q).cuda()).cpu().numpy().view(np.uint32)
    o, z = oracle.query_codes(Q, orc.A, want_z=True)
    assert_codes_match(g, o, z, idx.hash_bits)


def _budgets(cfg, n):
    Ts = sorted(set([1, 7, 100, (n + 99) // 100, n // 7, n, n + 5]
                    + [min(cfg.T(b), n) for b in cfg.budgets]))
    return [t for t in Ts if t >= 1]


@pytest.mark.parametrize("case", SMALL, ids=_ids)
def test_candidates_parity(built, case):
    """Identical codes -> identical candidate sets, ranks and (R, id) order."""
    cfg, X, Q, Xd, idx, orc = built(*case)
    n = X.shape[0]
    ocodes = orc.codes()
    idx.set_codes(ocodes[orc.perm])
    qc = oracle.query_codes(Q, orc.A)
    nq = min(len(Q), 16)
    qcd = torch.from_numpy(qc[:nq].view(np.int32)).cuda()
    for T in _budgets(cfg, n):
        gid, grk = idx.candidates(T, qcodes=qcd)
        gid = gid.cpu().numpy()
        grk = grk.cpu().numpy().view(np.uint16)
        for qi in range(nq):
            oid, ork = oracle.candidates(ocodes, orc.part, qc[qi], orc.R, T)
            order = np.lexsort((gid[qi], grk[qi]))
            assert np.array_equal(gid[qi][order], oid), (T, qi)
            assert np.array_equal(grk[qi][order], ork), (T, qi)


@pytest.mark.parametrize("case", SMALL, ids=_ids)
def test_query_parity(built, case):
    """End-to-end nrlsh_query with the oracle's codes injected."""
    cfg, X, Q, Xd, idx, orc = built(*case)
    n = X.shape[0]
    ocodes = orc.codes()
    idx.set_codes(ocodes[orc.perm])
    nq = min(len(Q), 24)
    Qd = torch.from_numpy(Q[:nq]).cuda()
    gq = idx.query_codes(Qd).cpu().numpy().view(np.uint32)
    oq = oracle.query_codes(Q[:nq], orc.A)
    k = cfg.k
    same = band_mask(gq, oq)
    for T in [t for t in _budgets(cfg, n) if t <= n][:5] + [n]:
        ids, sc = idx.query(Qd, k, T)
        ids, sc = ids.cpu().numpy(), sc.cpu().numpy()
        for qi in range(nq):
            if not same[qi]:
                continue     # a query bit inside the 1e-5 band: different probe order allowed
            a, s = oracle.query(X, ocodes, orc.part, orc.R, orc.A, Q[qi], T, k)
            assert_topk_match(ids[qi], sc[qi], a, s, X, Q[qi])


@pytest.mark.parametrize("name,n,nq,k", [("tiny", None, 50, 10), ("c2", None, 40, 10),
                                         ("c3", 60_000, 24, 10), ("scale", 80_000, 8, 100)])
def test_exact_topk_parity(name, n, nq, k):
    P = _P()
    cfg, X, Q = dataset(workloads.CONFIGS[name], n, nq)
    Q = Q[:nq]
    ids, sc = P.exact_topk(torch.from_numpy(X).cuda(), torch.from_numpy(Q).cuda(), k)
    ids, sc = ids.cpu().numpy(), sc.cpu().numpy()
    for qi in range(len(Q)):
        a, s = oracle.exact_topk(X, Q[qi], k)
        assert_topk_match(ids[qi], sc[qi], a, s, X, Q[qi])


@pytest.mark.parametrize("name,n,nq,k", [("c2", None, 40, 10), ("c3", 60_000, 300, 10),
                                         ("scale", 80_000, 8, 100)])
def test_exact_topk_seeded_matches_unseeded(name, n, nq, k):
    """Warm-start seeds change only the filter's starting threshold: any seed list
    (the LSH answers, the true answers, random ids, junk: -1 / out of range /
    repeats, fewer than k valid) gives the unseeded result, which matches the oracle."""
    P = _P()
    cfg, X, Q = dataset(workloads.CONFIGS[name], n, nq)
    Q = Q[:nq]
    Xd, Qd = torch.from_numpy(X).cuda(), torch.from_numpy(Q).cuda()
    base, bsc = P.exact_topk(Xd, Qd, k)
    base, bsc = base.cpu().numpy(), bsc.cpu().numpy()
    for qi in range(min(nq, 12)):
        a, s_ = oracle.exact_topk(X, Q[qi], k)
        assert_topk_match(base[qi], bsc[qi], a, s_, X, Q[qi])
    rng = np.random.default_rng(5)
    n_ = X.shape[0]
    seeds = {
        "truth": base.copy(),
        "random": rng.integers(0, n_, size=(nq, 3 * k)),
        "junk": np.where(rng.random((nq, 2 * k)) < 0.5, -1, n_ + 7).astype(np.int64),
        "repeats": np.repeat(base[:, :1], k + 3, axis=1),
        "short": base[:, : max(1, k // 2)].copy(),
    }
    m = 8 if name != "scale" else 1
    idx = P.Index(Xd, 64, m, seed=cfg.seed)
    lsh, _ = idx.query(Qd, k, max(k, n_ // 100))
    seeds["lsh"] = lsh.cpu().numpy()
    for nm, sd in seeds.items():
        got, gsc = P.exact_topk(Xd, Qd, k, seed_ids=torch.from_numpy(np.ascontiguousarray(sd, np.int64)).cuda())
        assert np.array_equal(got.cpu().numpy(), base), nm
        assert np.array_equal(gsc.cpu().numpy(), bsc), nm
        got2, _ = idx.exact_topk(Qd, k, seed_ids=np.ascontiguousarray(sd, np.int64))
        assert np.array_equal(got2.cpu().numpy(), base), nm


# --------------------------------------------------------------- edge cases
def test_full_budget_equals_brute_force(built):
    cfg, X, Q, Xd, idx, orc = built("tiny", None, None, 32, 8)
    P = _P()
    Qd = torch.from_numpy(Q[:20]).cuda()
    a, sa = idx.query(Qd, 10, X.shape[0])
    b, sb = P.exact_topk(Xd, Qd, 10)
    assert np.array_equal(a.cpu().numpy(), b.cpu().numpy())


def test_budget_below_k_pads(built):
    cfg, X, Q, Xd, idx, orc = built("tiny", None, None, 32, 8)
    ids, sc = idx.query(torch.from_numpy(Q[:5]).cuda(), 10, 3)
    ids, sc = ids.cpu().numpy(), sc.cpu().numpy()
    assert np.all(ids[:, 3:] == -1) and np.all(np.isneginf(sc[:, 3:]))
    assert np.all(ids[:, :3] >= 0)


def test_host_pointers_match_device(built):
    """HOST buffers through the same ABI (the e2e path) give the same answers."""
    P = _P()
    cfg, X, Q, Xd, idx, orc = built("tiny", None, None, 32, 8)
    idx_h = P.Index(X, 32, 8, seed=cfg.seed)          # numpy -> host pointer, owned copy
    assert np.array_equal(idx_h.codes(), idx.codes())
    a, sa = idx_h.query(Q[:10], 10, 100)
    b, sb = idx.query(torch.from_numpy(Q[:10]).cuda(), 10, 100)
    assert np.array_equal(a, b.cpu().numpy()) and np.array_equal(sa, sb.cpu().numpy())
    g1, _ = P.exact_topk(X, Q[:10], 10)
    g2, _ = P.exact_topk(Xd, torch.from_numpy(Q[:10]).cuda(), 10)
    assert np.array_equal(g1, g2.cpu().numpy())


def test_m_equals_n_and_m1_degenerate():
    P = _P()
    cfg, X, Q = dataset(workloads.CONFIGS["tiny"], 200, 8)
    for m in (1, 200):
        idx = P.Index(torch.from_numpy(X).cuda(), 32, m, seed=3)
        orc = oracle.OracleIndex(X, 32, m, seed=3)
        _, perm, off, V = idx.partition()
        assert np.array_equal(perm, orc.perm) and np.array_equal(V, orc.V)
        ocodes = orc.codes()
        idx.set_codes(ocodes[orc.perm])
        qc = oracle.query_codes(Q, orc.A)
        gid, grk = idx.candidates(50, qcodes=torch.from_numpy(qc.view(np.int32)).cuda())
        for qi in range(len(Q)):
            oid, ork = oracle.candidates(ocodes, orc.part, qc[qi], orc.R, 50)
            g = gid[qi].cpu().numpy()
            r = grk[qi].cpu().numpy().view(np.uint16)
            o = np.lexsort((g, r))
            assert np.array_equal(g[o], oid)


@pytest.mark.parametrize("kind", ["all_equal", "duplicates", "zeros"])
def test_degenerate_norms(kind):
    """Ties in the ranking, duplicated items, zero-norm items and a
    sub-dataset of zero vectors (V_j = 0).  n > 2048 forces the multi-level
    refinement of the exact selection."""
    P = _P()
    rng = np.random.default_rng(5)
    n, d = 50_000, 16
    X = rng.standard_normal((n, d)).astype(np.float32)
    if kind == "all_equal":
        X = (X / np.linalg.norm(X, axis=1, keepdims=True)).astype(np.float32)
        X[:, 0] = 1.0
        X[:, 1:] = 0.0
        X[::2, 0] = 0.0
        X[::2, 1] = 1.0            # every norm exactly 1, two directions
    elif kind == "duplicates":
        X[: n // 2] = X[n // 2:]
    else:
        X[: n // 3] = 0.0
    idx = P.Index(torch.from_numpy(X).cuda(), 64, 16, seed=9)
    orc = oracle.OracleIndex(X, 64, 16, seed=9)
    norm2, perm, off, V = idx.partition()
    assert np.array_equal(perm, orc.perm) and np.array_equal(V, orc.V)
    ocodes, z = orc.codes(want_z=True)
    gc = idx.codes()[np.argsort(perm, kind="stable")]
    assert_codes_match(gc, ocodes, z, 64)


def test_uniform_scheme_and_bit_accounting():
    """NEXT-2 uniform partitioning and NEXT-1 index bits inside the
    code budget (32 bits with 32 sub-datasets -> 27 hash bits)."""
    P = _P()
    cfg, X, Q = dataset(workloads.CONFIGS["c3"], 20_000, 16)
    idx = P.Index(torch.from_numpy(X).cuda(), 32, 32, seed=1, scheme="uniform",
                  index_bits_in_budget=True)
    assert idx.hash_bits == 27
    orc = oracle.OracleIndex(X, 27, 32, seed=1, scheme="uniform")
    _, perm, off, V = idx.partition()
    assert np.array_equal(perm, orc.perm) and np.array_equal(off, orc.offsets)
    assert np.array_equal(V, orc.V)
    assert np.array_equal(idx.rank_table(), orc.R)
    ocodes, z = orc.codes(want_z=True)
    assert_codes_match(idx.codes()[np.argsort(perm, kind="stable")], ocodes, z, 27)
    idx.set_codes(ocodes[orc.perm])
    qc = oracle.query_codes(Q, orc.A)
    gid, grk = idx.candidates(300, qcodes=torch.from_numpy(qc.view(np.int32)).cuda())
    for qi in range(len(Q)):
        oid, ork = oracle.candidates(ocodes, orc.part, qc[qi], orc.R, 300)
        g = gid[qi].cpu().numpy()
        r = grk[qi].cpu().numpy().view(np.uint16)
        o = np.lexsort((g, r))
        assert np.array_equal(g[o], oid) and np.array_equal(r[o], ork)


@pytest.mark.parametrize("mode", ["parallel", "serial", "parallel+serial"])
def test_forced_fallback_path(built, mode, monkeypatch):
    """The exact fallback (taken when the pilot bound under/overflows) gives the
    same candidates as the oracle; forced for every query via a test switch.  Modes:
    the all-SM re-do (up to 64 failed queries per sub-batch), the one-CTA-per-query
    kernel, and both (100 failed queries: 64 + 36)."""
    cfg, X, Q, Xd, idx, orc = built("c4", 300_000, 32, 32, 128)
    monkeypatch.setenv("NRLSH_TEST_FORCE_FALLBACK", "1")
    if mode == "serial":
        monkeypatch.setenv("NRLSH_FALLBACK_SERIAL", "1")
    P = _P()
    ocodes = orc.codes()
    idx.set_codes(ocodes[orc.perm])
    nq = 100 if mode == "parallel+serial" else 6
    Qm = np.concatenate([Q] * (nq // len(Q) + 1))[:nq]
    qc = oracle.query_codes(Qm, orc.A)
    gid, grk = idx.candidates(2000, qcodes=torch.from_numpy(qc.view(np.int32)).cuda())
    assert P.last_query_stats()["fallback_queries"] == nq
    for qi in ([0, 1, 63, 64, 99] if nq == 100 else range(6)):
        oid, ork = oracle.candidates(ocodes, orc.part, qc[qi], orc.R, 2000)
        g = gid[qi].cpu().numpy()
        r = grk[qi].cpu().numpy().view(np.uint16)
        o = np.lexsort((g, r))
        assert np.array_equal(g[o], oid) and np.array_equal(r[o], ork)


def test_errors():
    P = _P()
    X = np.random.default_rng(0).standard_normal((1000, 8)).astype(np.float32)
    Xb = X.copy()
    Xb[17, 3] = np.nan
    with pytest.raises(P.NrlshError) as e:
        P.Index(torch.from_numpy(Xb).cuda(), 32, 4)
    assert e.value.code == "ENONFINITE" and "17" in str(e.value)
    idx = P.Index(torch.from_numpy(X).cuda(), 32, 4)
    Qz = np.random.default_rng(1).standard_normal((9, 8)).astype(np.float32)
    Qz[7] = 0.0
    with pytest.raises(P.NrlshError) as e:
        idx.query(torch.from_numpy(Qz).cuda(), 5, 10)
    assert e.value.code == "EZERONORM" and "7" in str(e.value)
    with pytest.raises(P.NrlshError) as e:
        idx.query(torch.from_numpy(X[:3]).cuda(), 0, 10)
    assert e.value.code == "EINVAL"
    with pytest.raises(P.NrlshError) as e:
        idx.query(torch.from_numpy(X[:3]).cuda(), 5, 0)
    assert e.value.code == "EINVAL"


# ------------------------------------------------------- the bench's re-rank path
def _headline_rerank_check(P, cfg, X, Q, idx, ocodes, part, R, A, L):
    """The path bench.py times, at full size: the default re-rank selection with
    more than one sub-batch (a ragged last one) and several 256-query pairs per
    sub-batch — at c4 the tensor-core member-mode filter with bound-sorted query
    pairs, proportional CTA shares and tile pruning (Alg. 2 l.6).  Every
    query's ids and fp32 scores equal the gather path's bit for bit, and sampled
    queries equal the oracle's answer (the oracle's codes are injected)."""
    n = X.shape[0]
    if cfg.name == "c4":
        T, nqh = cfg.T((1, 100)), cfg.query_batch + 300       # the bench's T; 1024 + 300
    else:
        T, nqh = n // 200, 1100                                 # T >= n/300: the tensor path
    Qh = np.ascontiguousarray(Q[:nqh])
    Qd = torch.from_numpy(Qh).cuda()
    os.environ.pop("NRLSH_RERANK_TC", None)
    ti, ts = idx.query(Qd, cfg.k, T)
    info = P.last_rerank_path()
    assert info["path"] == "tensor", info
    assert info["filter_pairs"] > 0
    try:
        os.environ["NRLSH_RERANK_TC"] = "0"
        gi, gs = idx.query(Qd, cfg.k, T)
        assert P.last_rerank_path()["path"] == "gather"
    finally:
        os.environ.pop("NRLSH_RERANK_TC", None)
    assert torch.equal(gi, ti)
    assert torch.equal(gs.view(torch.int32), ts.view(torch.int32))
    ti, ts = ti.cpu().numpy(), ts.cpu().numpy()
    gq = idx.query_codes(Qd).cpu().numpy().view(np.uint32)
    qc = oracle.query_codes(Qh, A)
    rng = np.random.default_rng(2)
    sample = sorted(set([q for q in (0, 255, 256, 1023, 1024, cfg.query_batch - 1,
                                     cfg.query_batch, nqh - 1) if q < nqh]
                        + rng.choice(nqh, 14, replace=False).tolist()))
    same = band_mask(gq[sample], qc[sample], 0.8)
    for s_, qi in zip(same, sample):
        if s_:
            a, sc = oracle.query(X, ocodes, part, R, A, Qh[qi], T, cfg.k)
            assert_topk_match(ti[qi], ts[qi], a, sc, X, Qh[qi])


def test_rerank_path_selection(built, monkeypatch):
    """The automatic re-rank rule (api.cu): the tensor-core filter iff T >= n/300 and
    a full sub-batch's Qmax * T >= 1.28 n; both sides of each threshold."""
    cfg, X, Q, Xd, idx, orc = built("c4", 300_000, 32, 64, 128)
    P = _P()
    monkeypatch.delenv("NRLSH_RERANK_TC", raising=False)
    n = X.shape[0]
    Qrep = np.ascontiguousarray(np.concatenate([Q] * 20)[:600])
    assert n == 300_000            # n / 300 = 1000; 1.28 n = 384,000
    for nq, T, want in [(500, 1000, "tensor"), (500, 999, "gather"), (384, 1000, "tensor"),
                        (383, 1000, "gather"), (300, 1280, "tensor"), (300, 1279, "gather"),
                        (1, n, "gather"), (600, 10, "gather")]:
        idx.query(torch.from_numpy(Qrep[:nq]).cuda(), 10, T)
        assert P.last_rerank_path()["path"] == want, (nq, T)


def test_sub_batch_streams_identical(built, monkeypatch):
    """Sub-batches on one, two or three streams (api.cu: a workspace set per stream)
    give bit-identical answers and candidates, on the tensor-core re-rank (T = 1%) and
    the gather path (T = 0.1%); the ground truth likewise in sub-batches of 1,024 on
    one or two streams and of 4,096."""
    cfg, X, Q, Xd, idx, orc = built("c4", 300_000, 32, 64, 128)
    P = _P()
    n = X.shape[0]
    nq = 2600   # three sub-batches of <= 1,024
    Qd = torch.from_numpy(np.ascontiguousarray(np.concatenate([Q] * 82)[:nq])).cuda()
    for T, path in ((n // 100, "tensor"), (n // 1000, "gather")):
        res = []
        for env in ({"NRLSH_QUERY_SERIAL": "1"}, {}, {"NRLSH_QUERY_STREAMS": "3"}):
            for kk in ("NRLSH_QUERY_SERIAL", "NRLSH_QUERY_STREAMS"):
                monkeypatch.delenv(kk, raising=False)
            for kk, vv in env.items():
                monkeypatch.setenv(kk, vv)
            ids, sc = idx.query(Qd, cfg.k, T)
            assert P.last_rerank_path()["path"] == path
            cid, crk = idx.candidates(T, queries=Qd[:1100])
            res.append((ids.cpu().numpy(), sc.cpu().numpy().view(np.int32),
                        np.sort(cid.cpu().numpy(), axis=1)))
        for r in res[1:]:
            for a, b in zip(res[0], r):
                assert np.array_equal(a, b), T
    monkeypatch.delenv("NRLSH_QUERY_STREAMS", raising=False)
    monkeypatch.delenv("NRLSH_QUERY_SERIAL", raising=False)
    seeds, _ = idx.query(Qd, cfg.k, n // 100)
    gts = []
    for env in ({"NRLSH_GT_BATCH": "1024", "NRLSH_QUERY_SERIAL": "1"}, {"NRLSH_GT_BATCH": "1024"}, {}):
        for kk in ("NRLSH_GT_BATCH", "NRLSH_QUERY_SERIAL"):
            monkeypatch.delenv(kk, raising=False)
        for kk, vv in env.items():
            monkeypatch.setenv(kk, vv)
        gi, gsc = idx.exact_topk(Qd, cfg.k, seed_ids=seeds)
        gts.append((gi.cpu().numpy(), gsc.cpu().numpy().view(np.int32)))
    for g in gts[1:]:
        assert np.array_equal(gts[0][0], g[0]) and np.array_equal(gts[0][1], g[1])
    for qi in (0, nq - 1):
        a, sa = oracle.exact_topk(X, Q[qi % len(Q)], cfg.k)
        assert_topk_match(gts[-1][0][qi], gts[-1][1][qi].view(np.float32), a, sa, X, Q[qi % len(Q)])


@pytest.mark.parametrize("nq", [513, 700])
def test_rerank_tensor_multi_pair_matches_gather(built, nq, monkeypatch):
    """Several 256-query pairs per sub-batch with a ragged last pair, under the
    automatic selection (bound-sorted pairs, proportional CTA shares, pruning):
    bit-identical to the gather path at T = n/100 and n/3."""
    cfg, X, Q, Xd, idx, orc = built("c4", 300_000, 32, 64, 128)
    P = _P()
    n = X.shape[0]
    Qd = torch.from_numpy(np.ascontiguousarray(np.concatenate([Q] * 25)[:nq])).cuda()
    for T in (n // 100, n // 3):
        monkeypatch.delenv("NRLSH_RERANK_TC", raising=False)
        ti, ts = idx.query(Qd, cfg.k, T)
        assert P.last_rerank_path()["path"] == "tensor", T
        monkeypatch.setenv("NRLSH_RERANK_TC", "0")
        gi, gs = idx.query(Qd, cfg.k, T)
        assert torch.equal(gi, ti) and torch.equal(gs.view(torch.int32), ts.view(torch.int32)), T


# ------------------------------------------------------- full (BASELINE) sizes
@pytest.mark.parametrize("name,L,m", [("c4", 64, 128), ("c4", 32, 128), ("scale", 128, 256)])
def test_full_size_sampled(name, L, m):
    """BASELINE.json full sizes, in the launch configuration bench.py times:
    partition bit-exact over all n; every code bit (band-exempt); candidates and
    top-k on sampled queries with the oracle's codes injected; ground truth on
    sampled queries."""
    P = _P()
    cfg = workloads.CONFIGS[name]
    _, X, Q = dataset(cfg)
    Xd = torch.from_numpy(X).cuda()
    idx = P.Index(Xd, L, m, seed=cfg.seed)
    n = X.shape[0]
    nv = oracle.norm2(X)
    norm2, perm, off, V = idx.partition()
    assert np.array_equal(norm2.view(np.uint64), nv.view(np.uint64))
    part, operm, ooff, oV = oracle.partition(nv, m)
    assert np.array_equal(perm, operm) and np.array_equal(off, ooff) and np.array_equal(V, oV)
    A = oracle.projection(cfg.seed, X.shape[1] + 1, L)
    assert np.array_equal(idx.projection(), A)
    R, _ = oracle.rank_table(np.sqrt(oV), L, 0.01)
    assert np.array_equal(idx.rank_table(), R)
    ocodes = oracle.item_codes_parallel(X, part, oV, nv, A)
    pos_of_id = np.empty(n, np.int64)
    pos_of_id[perm] = np.arange(n)
    gcodes = idx.codes()[pos_of_id]
    rows = np.nonzero((gcodes != ocodes).any(axis=1))[0]
    assert len(rows) < max(10, n // 1000)
    if len(rows):
        oc, z = oracle.item_codes(X[rows], part[rows], oV, nv[rows], A, want_z=True)
        assert_codes_match(gcodes[rows], oc, z, L)
    idx.set_codes(ocodes[perm])
    qs = Q[:6]
    qc = oracle.query_codes(qs, A)
    T = min(cfg.T(cfg.budgets[0]), n)
    gid, grk = idx.candidates(T, qcodes=torch.from_numpy(qc.view(np.int32)).cuda())
    gid, grk = gid.cpu().numpy(), grk.cpu().numpy().view(np.uint16)
    for qi in range(len(qs)):
        oid, ork = oracle.candidates(ocodes, part, qc[qi], R, T)
        o = np.lexsort((gid[qi], grk[qi]))
        assert np.array_equal(gid[qi][o], oid) and np.array_equal(grk[qi][o], ork)
    Qd = torch.from_numpy(qs).cuda()
    gq = idx.query_codes(Qd).cpu().numpy().view(np.uint32)
    ids, sc = idx.query(Qd, cfg.k, T)
    ids, sc = ids.cpu().numpy(), sc.cpu().numpy()
    same = band_mask(gq, qc, 0.8)
    for qi in range(len(qs)):
        if same[qi]:
            a, s = oracle.query(X, ocodes, part, R, A, qs[qi], T, cfg.k)
            assert_topk_match(ids[qi], sc[qi], a, s, X, qs[qi])
    _headline_rerank_check(P, cfg, X, Q, idx, ocodes, part, R, A, L)
    gt_ids, gt_sc = P.exact_topk(Xd, torch.from_numpy(Q[:3]).cuda(), cfg.k)
    gt_ids, gt_sc = gt_ids.cpu().numpy(), gt_sc.cpu().numpy()
    for qi in range(3):
        a, s = oracle.exact_topk(X, Q[qi], cfg.k)
        assert_topk_match(gt_ids[qi], gt_sc[qi], a, s, X, Q[qi])


@pytest.mark.parametrize("case", [("c4", 300_000, 32, 64, 128), ("scale", 70_000, 16, 128, 256),
                                  ("tiny", None, None, 32, 8), ("c3", 40_000, 64, 64, 1)], ids=_ids)
def test_candidates_parity_tensor_scan(built, case, monkeypatch):
    """NEXT-3: the opt-in tcgen05 int8 Hamming scan (scan_tc.cu, NRLSH_SCAN_TC=1) gives
    the oracle's candidate sets, ranks and (R, id) order (identical codes injected),
    across budgets from 1 to n."""
    monkeypatch.setenv("NRLSH_SCAN_TC", "1")
    cfg, X, Q, Xd, idx, orc = built(*case)
    idx = _P().Index(Xd, case[3], case[4], seed=cfg.seed)   # (its +-1 rows are made at build)
    n = X.shape[0]
    ocodes = orc.codes()
    idx.set_codes(ocodes[orc.perm])
    qc = oracle.query_codes(Q, orc.A)
    nq = min(len(Q), 16)
    qcd = torch.from_numpy(qc[:nq].view(np.int32)).cuda()
    for T in _budgets(cfg, n):
        gid, grk = idx.candidates(T, qcodes=qcd)
        gid = gid.cpu().numpy()
        grk = grk.cpu().numpy().view(np.uint16)
        for qi in range(nq):
            oid, ork = oracle.candidates(ocodes, orc.part, qc[qi], orc.R, T)
            order = np.lexsort((gid[qi], grk[qi]))
            assert np.array_equal(gid[qi][order], oid), (T, qi)
            assert np.array_equal(grk[qi][order], ork), (T, qi)


@pytest.mark.parametrize("bound", ["default", "off", "always", "coarse_always"])
@pytest.mark.parametrize("case", [("c4", 300_000, 32, 64, 128), ("scale", 70_000, 16, 128, 256),
                                  ("tiny", None, None, 32, 8), ("c4", 300_000, 32, 32, 4),
                                  ("c3", 40_000, 64, 64, 1)], ids=_ids)
def test_candidates_parity_scan_bound(built, case, bound, monkeypatch):
    """The popcount scan's pair lower bound (sum over word pairs of
    popcount((x_a ^ q_a) | (x_b ^ q_b)) <= h, tried first at small radii) changes no
    candidate: with the bound at its default radii, off, and tried at every radius,
    the candidate sets, ranks and (R, id) order equal the oracle's (identical codes
    injected), across budgets from 1 to n."""
    P = _P()
    monkeypatch.setenv("NRLSH_SCAN_LBMAX", {"default": "", "off": "-1", "always": "255",
                                            "coarse_always": "255"}[bound])
    if bound == "default":
        monkeypatch.delenv("NRLSH_SCAN_LBMAX")
    # (the coarser first bound — one POPC per item at 128 bits, per two items at 64 —
    # at every radius too)
    if bound == "coarse_always":
        monkeypatch.setenv("NRLSH_SCAN_LB0MAX", "255")
    else:
        monkeypatch.delenv("NRLSH_SCAN_LB0MAX", raising=False)
    cfg, X, Q, Xd, idx, orc = built(*case)
    n = X.shape[0]
    ocodes = orc.codes()
    idx.set_codes(ocodes[orc.perm])
    qc = oracle.query_codes(Q, orc.A)
    nq = min(len(Q), 16)
    qcd = torch.from_numpy(qc[:nq].view(np.int32)).cuda()
    for T in _budgets(cfg, n):
        gid, grk = idx.candidates(T, qcodes=qcd)
        gid = gid.cpu().numpy()
        grk = grk.cpu().numpy().view(np.uint16)
        for qi in range(nq):
            oid, ork = oracle.candidates(ocodes, orc.part, qc[qi], orc.R, T)
            order = np.lexsort((gid[qi], grk[qi]))
            assert np.array_equal(gid[qi][order], oid), (T, qi)
            assert np.array_equal(grk[qi][order], ork), (T, qi)
        st = P.last_scan_stats()
        qs = P.last_query_stats()
        W = (case[3] + 31) // 32
        # POPCs issued: at most W per scanned pair plus the bounds' (W/2 + W/4), at
        # least one per two pairs
        assert 0 < st["popc_ops"] <= qs["scanned_pairs"] * (W + W / 2 + W / 4)
        assert st["popc_ops"] * 2 >= qs["scanned_pairs"]
        if bound in ("always", "coarse_always") and case[3] > 32:
            assert st["bound_pairs"] > 0
        if bound == "off" or case[3] <= 32:
            assert st["bound_pairs"] == 0


def test_scan_rows_full(built, monkeypatch):
    """Candidate rows too small for the pilot's estimate (NRLSH_TEST_BUFFER_TIGHT: T plus
    one sub-dataset): the scan's dense runs, lane spills and stage copy-out hit the end of
    the row (their guarded stores), the counts overflow, and the exact fallback redoes
    those queries — the candidates still equal the oracle's."""
    cfg, X, Q, Xd, idx, orc = built("c4", 300_000, 32, 64, 128)
    P = _P()
    monkeypatch.setenv("NRLSH_TEST_BUFFER_TIGHT", "1")
    ocodes = orc.codes()
    idx.set_codes(ocodes[orc.perm])
    qc = oracle.query_codes(Q, orc.A)
    qcd = torch.from_numpy(qc.view(np.int32)).cuda()
    T = 30_000
    gid, grk = idx.candidates(T, qcodes=qcd)
    assert P.last_query_stats()["fallback_queries"] > 0
    gid, grk = gid.cpu().numpy(), grk.cpu().numpy().view(np.uint16)
    for qi in range(0, len(Q), 4):
        oid, ork = oracle.candidates(ocodes, orc.part, qc[qi], orc.R, T)
        o = np.lexsort((gid[qi], grk[qi]))
        assert np.array_equal(gid[qi][o], oid) and np.array_equal(grk[qi][o], ork)


def test_small_last_sub_batch_large_budget(built):
    """nq = one full sub-batch + a few queries, T spanning several re-rank rounds: the
    short last sub-batch splits its candidates finer than the full one (regression:
    its partial top-k lists once overflowed a buffer sized for the full sub-batch)."""
    cfg, X, Q, Xd, idx, orc = built("c2", None, 200, 64, 32)
    n = X.shape[0]
    Qbig = np.concatenate([Q] * 6)[:1024 + 9]                 # 1024 + 9 queries
    Qd = torch.from_numpy(np.ascontiguousarray(Qbig)).cuda()
    ocodes = orc.codes()
    idx.set_codes(ocodes[orc.perm])
    gq = idx.query_codes(Qd).cpu().numpy().view(np.uint32)
    oq = oracle.query_codes(Qbig, orc.A)
    same = band_mask(gq, oq)
    for T in (1777, n // 2):
        ids, sc = idx.query(Qd, cfg.k, T)
        ids, sc = ids.cpu().numpy(), sc.cpu().numpy()
        for qi in list(range(1024, 1033)) + [0, 511]:
            if not same[qi]:
                continue
            a, s = oracle.query(X, ocodes, orc.part, orc.R, orc.A, Qbig[qi], T, cfg.k)
            assert_topk_match(ids[qi], sc[qi], a, s, X, Qbig[qi])


def test_coarse_cells_no_overflow(built):
    """Few sub-datasets over heavy-tailed norms: most items of the top sub-dataset
    have ||x|| << U_j, map close to e_{d+1} and share (nearly) one code, so the
    pilot's boundary cell can hold tens of thousands of items for a tiny budget.
    The per-query capacity covers a whole sub-dataset: no query may overflow into
    the exact fallback, and the candidates still equal the oracle's."""
    cfg, X, Q, Xd, idx, orc = built("c4", 300_000, 32, 32, 4)
    P = _P()
    ocodes = orc.codes()
    idx.set_codes(ocodes[orc.perm])
    qc = oracle.query_codes(Q, orc.A)
    for T in (1, 128, 4096):
        gid, grk = idx.candidates(T, qcodes=torch.from_numpy(qc.view(np.int32)).cuda())
        assert P.last_query_stats()["fallback_queries"] == 0, T
        gid, grk = gid.cpu().numpy(), grk.cpu().numpy().view(np.uint16)
        for qi in range(4):
            oid, ork = oracle.candidates(ocodes, orc.part, qc[qi], orc.R, T)
            o = np.lexsort((gid[qi], grk[qi]))
            assert np.array_equal(gid[qi][o], oid) and np.array_equal(grk[qi][o], ork)


@pytest.mark.parametrize("case", [("c4", 300_000, 32, 64, 128), ("c4", 300_000, 32, 32, 4),
                                  ("scale", 70_000, 16, 128, 256), ("c2", None, 200, 64, 32),
                                  ("tiny", None, None, 32, 8)], ids=_ids)
def test_rerank_tensor_matches_gather(built, case, monkeypatch):
    """The tensor-core re-rank (bf16 pass over every item, certified filter against a
    running bound of the k-th best candidate score, candidate rule in the epilogue,
    fp32 re-rank of the survivors) returns exactly the gather path's answer — same
    ids, bit-identical scores — at budgets from tiny to all of n; and through its
    overflow redo (survivor lists capped at 16)."""
    cfg, X, Q, Xd, idx, orc = built(*case)
    P = _P()
    n = X.shape[0]
    Qd = torch.from_numpy(Q).cuda()
    for T in sorted({1, 7, max(1, n // 100), n // 3, n}):
        for k in (1, cfg.k, 64):
            monkeypatch.setenv("NRLSH_RERANK_TC", "0")
            gi, gs = idx.query(Qd, k, T)
            assert P.last_rerank_path()["path"] == "gather"
            monkeypatch.setenv("NRLSH_RERANK_TC", "1")
            ti, ts = idx.query(Qd, k, T)
            assert P.last_rerank_path()["path"] == "tensor"
            assert torch.equal(gi, ti), (T, k)
            assert torch.equal(gs.view(torch.int32), ts.view(torch.int32)), (T, k)
    monkeypatch.setenv("NRLSH_RERANK_TC_CAP", "16")
    T = max(1, n // 10)
    ti, ts = idx.query(Qd, cfg.k, T)
    info = P.last_rerank_path()
    assert info["path"] == "tensor" and info["overflow_redone"] > 0
    monkeypatch.setenv("NRLSH_RERANK_TC", "0")
    gi, gs = idx.query(Qd, cfg.k, T)
    assert torch.equal(gi, ti) and torch.equal(gs.view(torch.int32), ts.view(torch.int32))


@pytest.mark.parametrize("case", [("c4", 300_000, 32, 64, 128), ("scale", 70_000, 16, 128, 256),
                                  ("c3", 40_000, 64, 64, 64)], ids=_ids)
def test_tile_pruning_is_exact(built, case, monkeypatch):
    """Tile pruning of the tensor-core filter (tiles whose largest |x| cannot reach a
    query pair's seeded bound are not streamed; Cauchy-Schwarz) changes nothing: the
    index's seeded ground truth and the tensor-core re-rank equal their unpruned runs
    bit for bit (ids and fp32 scores), at budgets from tiny to all of n."""
    cfg, X, Q, Xd, idx, orc = built(*case)
    P = _P()
    n = X.shape[0]
    Qd = torch.from_numpy(np.concatenate([Q] * (300 // len(Q) + 1))[:300]).cuda()   # > 1 pair
    seeds, _ = idx.query(Qd, cfg.k, max(cfg.k, n // 100))
    for k in (1, cfg.k, 50):
        monkeypatch.delenv("NRLSH_GT_ALLTILES", raising=False)
        a, sa = idx.exact_topk(Qd, k, seed_ids=seeds)
        monkeypatch.setenv("NRLSH_GT_ALLTILES", "1")
        b, sb = idx.exact_topk(Qd, k, seed_ids=seeds)
        assert torch.equal(a, b) and torch.equal(sa.view(torch.int32), sb.view(torch.int32)), k
    monkeypatch.setenv("NRLSH_RERANK_TC", "1")
    for T in (max(1, n // 100), n // 3):
        monkeypatch.delenv("NRLSH_GT_ALLTILES", raising=False)
        a, sa = idx.query(Qd, cfg.k, T)
        monkeypatch.setenv("NRLSH_GT_ALLTILES", "1")
        b, sb = idx.query(Qd, cfg.k, T)
        assert torch.equal(a, b) and torch.equal(sa.view(torch.int32), sb.view(torch.int32)), T


# ------------------------------------------------------------------ unusual shapes
ODD = [   # (n, d, L, m): odd d (scalar loads, unskewed norm chain), partial code words
          # (L = 17, 50, 100), tiny d, d beyond the bf16 filters' range, ragged n
    (12_345, 37, 17, 7),
    (9_999, 150, 100, 5),
    (7_777, 64, 50, 9),
    (5_000, 2, 64, 3),
    (3_001, 301, 128, 61),
    (2_000, 513, 32, 10),
]


@pytest.mark.parametrize("shape", ODD, ids=_ids)
def test_odd_shapes_parity(shape):
    """Build, query (oracle codes injected) and exact top-k parity on shapes off the
    configs' grid: every kernel's scalar / ragged / fallback variant."""
    from dataclasses import replace
    n, d, L, m = shape
    P = _P()
    cfg = replace(workloads.CONFIGS["c2"], name=f"odd{n}x{d}", n=n, d=d, nq=12)
    X = workloads.make_items(cfg)
    Q = workloads.make_queries(cfg)
    Xd = torch.from_numpy(X).cuda()
    idx = P.Index(Xd, L, m, seed=3)
    orc = oracle.OracleIndex(X, idx.hash_bits, m, seed=3)
    norm2, perm, offsets, V = idx.partition()
    assert np.array_equal(norm2.view(np.uint64), orc.norm2.view(np.uint64))
    assert np.array_equal(perm, orc.perm)
    assert np.array_equal(offsets, orc.offsets)
    assert np.array_equal(V, orc.V)
    assert np.array_equal(idx.projection(), orc.A)
    assert np.array_equal(idx.rank_table(), orc.R)
    ocodes, z = orc.codes(want_z=True)
    assert_codes_match(idx.codes()[np.argsort(perm, kind="stable")], ocodes, z, idx.hash_bits)
    idx.set_codes(ocodes[orc.perm])
    Qd = torch.from_numpy(Q).cuda()
    gq = idx.query_codes(Qd).cpu().numpy().view(np.uint32)
    oq = oracle.query_codes(Q, orc.A)
    k = 10
    same = band_mask(gq, oq, 0.75)
    for T in (1, 37, (n + 99) // 100, n // 3, n):
        ids, sc = idx.query(Qd, k, T)
        ids, sc = ids.cpu().numpy(), sc.cpu().numpy()
        for qi in range(len(Q)):
            if not same[qi]:
                continue
            a, s = oracle.query(X, ocodes, orc.part, orc.R, orc.A, Q[qi], T, k)
            assert_topk_match(ids[qi], sc[qi], a, s, X, Q[qi])
    gi, gs = P.exact_topk(Xd, Qd, k)
    gi, gs = gi.cpu().numpy(), gs.cpu().numpy()
    for qi in range(len(Q)):
        a, s = oracle.exact_topk(X, Q[qi], k)
        assert_topk_match(gi[qi], gs[qi], a, s, X, Q[qi])
    idx.close()


# ------------------------------------- NEXT-4: per-sub-dataset projections A_j
PP_CASES = [("tiny", None, 40, 32, 8), ("c3", 40_000, 40, 64, 64), ("c4", 300_000, 32, 64, 128),
            ("scale", 70_000, 16, 128, 256), ("c2", None, 40, 50, 7)]


@pytest.fixture(scope="session")
def built_pp():
    cache = {}

    def get(name, n, nq, L, m):
        key = (name, n, nq, L, m)
        if key not in cache:
            P = _P()
            cfg, X, Q = dataset(workloads.CONFIGS[name], n, nq)
            Xd = torch.from_numpy(X).cuda()
            idx = P.Index(Xd, L, m, seed=cfg.seed + 5, proj="per_partition")
            orc = oracle.OracleIndex(X, idx.hash_bits, m, seed=cfg.seed + 5, proj="per_partition")
            cache[key] = (cfg, X, Q[:nq], Xd, idx, orc)
        return cache[key]
    return get


@pytest.mark.parametrize("case", PP_CASES, ids=_ids)
def test_pp_build_and_codes_parity(built_pp, case):
    """Alg. 1 l.7 with an independent projection per sub-index (
    A_j from seed XOR j): every A_j, the partition, the rank table and
    every item code (band-exempt) and query code under every A_j match the oracle."""
    cfg, X, Q, Xd, idx, orc = built_pp(*case)
    assert idx.proj == "per_partition" and idx.qm == case[4]
    A = idx.projection()
    assert A.shape == orc.A_all.shape and np.array_equal(A, orc.A_all)
    _, perm, offsets, V = idx.partition()
    assert np.array_equal(perm, orc.perm) and np.array_equal(V, orc.V)
    assert np.array_equal(idx.rank_table(), orc.R)
    ocodes, z = orc.codes(want_z=True)
    assert_codes_match(idx.codes()[np.argsort(perm, kind="stable")], ocodes, z, idx.hash_bits)
    g = idx.query_codes(torch.from_numpy(Q).cuda()).cpu().numpy().view(np.uint32)
    oq, oz = orc.query_codes(Q, want_z=True)
    assert g.shape == oq.shape
    m, W = oq.shape[1], oq.shape[2]
    assert_codes_match(g.reshape(-1, W), oq.reshape(-1, W), oz.reshape(-1, oz.shape[2]), idx.hash_bits)


@pytest.mark.parametrize("case", PP_CASES, ids=_ids)
def test_pp_candidates_and_query_parity(built_pp, case):
    """Identical codes injected: candidate sets, structure positions and (R, id)
    order, and the end-to-end answers equal the oracle's at budgets from 1 to n."""
    cfg, X, Q, Xd, idx, orc = built_pp(*case)
    n = X.shape[0]
    ocodes = orc.codes()
    idx.set_codes(ocodes[orc.perm])
    qc = orc.query_codes(Q)
    nq = min(len(Q), 12)
    qcd = torch.from_numpy(np.ascontiguousarray(qc[:nq]).view(np.int32)).cuda()
    for T in _budgets(cfg, n):
        gid, grk = idx.candidates(T, qcodes=qcd)
        gid, grk = gid.cpu().numpy(), grk.cpu().numpy().view(np.uint16)
        for qi in range(nq):
            oid, ork = orc.candidates(ocodes, qc[qi], T)
            o = np.lexsort((gid[qi], grk[qi]))
            assert np.array_equal(gid[qi][o], oid), (T, qi)
            assert np.array_equal(grk[qi][o], ork), (T, qi)
    Qd = torch.from_numpy(Q[:nq]).cuda()
    gq = idx.query_codes(Qd).cpu().numpy().view(np.uint32)
    same = band_mask(gq, qc[:nq], 0.75)
    for T in sorted({1, 37, max(1, n // 100), n // 3, n}):
        ids, sc = idx.query(Qd, cfg.k, T)
        ids, sc = ids.cpu().numpy(), sc.cpu().numpy()
        for qi in range(nq):
            if same[qi]:
                a, s = orc.query(ocodes, Q[qi], T, cfg.k)
                assert_topk_match(ids[qi], sc[qi], a, s, X, Q[qi])


def test_pp_one_sub_dataset_equals_shared():
    """m = 1: A_0 is the shared projection, so codes, query codes and answers are
    identical to the shared-A index (plain SIMPLE-LSH either way)."""
    P = _P()
    cfg, X, Q = dataset(workloads.CONFIGS["c2"], None, 40)
    Xd, Qd = torch.from_numpy(X).cuda(), torch.from_numpy(Q[:40]).cuda()
    a = P.Index(Xd, 64, 1, seed=2)
    b = P.Index(Xd, 64, 1, seed=2, proj="per_partition")
    assert np.array_equal(a.codes(), b.codes())
    assert torch.equal(a.query_codes(Qd), b.query_codes(Qd).reshape(40, -1))
    for T in (50, 1777):
        ia, sa = a.query(Qd, 10, T)
        ib, sb = b.query(Qd, 10, T)
        assert torch.equal(ia, ib) and torch.equal(sa, sb)


@pytest.mark.parametrize("case", [("c4", 300_000, 32, 64, 128), ("c3", 40_000, 40, 64, 64)], ids=_ids)
def test_pp_rerank_tensor_and_fallback(built_pp, case, monkeypatch):
    """The tensor-core re-rank (member test with the query's code under the item's
    A_j) equals the gather path bit for bit over several query pairs; the forced
    exact fallback gives the oracle's candidates."""
    cfg, X, Q, Xd, idx, orc = built_pp(*case)
    P = _P()
    n = X.shape[0]
    Qd = torch.from_numpy(np.ascontiguousarray(np.concatenate([Q] * 20)[:600])).cuda()
    for T in (n // 100, n // 3):
        monkeypatch.setenv("NRLSH_RERANK_TC", "1")
        ti, ts = idx.query(Qd, cfg.k, T)
        assert P.last_rerank_path()["path"] == "tensor"
        monkeypatch.setenv("NRLSH_RERANK_TC", "0")
        gi, gs = idx.query(Qd, cfg.k, T)
        assert torch.equal(gi, ti) and torch.equal(gs.view(torch.int32), ts.view(torch.int32)), T
    monkeypatch.delenv("NRLSH_RERANK_TC")
    ocodes = orc.codes()
    idx.set_codes(ocodes[orc.perm])
    qc = orc.query_codes(Q[:6])
    monkeypatch.setenv("NRLSH_TEST_FORCE_FALLBACK", "1")
    gid, grk = idx.candidates(2000, qcodes=torch.from_numpy(np.ascontiguousarray(qc).view(np.int32)).cuda())
    assert P.last_query_stats()["fallback_queries"] == 6
    for qi in range(6):
        oid, ork = orc.candidates(ocodes, qc[qi], 2000)
        g, r = gid[qi].cpu().numpy(), grk[qi].cpu().numpy().view(np.uint16)
        o = np.lexsort((g, r))
        assert np.array_equal(g[o], oid) and np.array_equal(r[o], ork)
