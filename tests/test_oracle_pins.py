"""Pins of the CPU oracle against what the paper and mathematics fix.

These run with ``-m "not gpu"``.  Each test pins an oracle function to
something other than itself: a closed form stated in the paper, a worked
example (tests/golden/, each with its citation), an invariant, a special case
that reduces to a textbook/library routine, or brute force on tiny inputs.
PAPER:<line> = /root/reference/PAPER.md; SPEC:<line> = /root/reference/SPEC.md.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import workloads

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _rng(s=0):
    return np.random.default_rng(s)


def _popcount_np(a):
    """Independent popcount (numpy unpackbits), for brute-force pins."""
    a = np.ascontiguousarray(a, dtype=np.uint32)
    return np.unpackbits(a.view(np.uint8), axis=-1).sum(axis=-1)


# ------------------------------------------------------------------ P1 norms
def test_norm_345():
    g = _gold("spec_examples.json")["norm_345"]
    assert oracle.norm2(np.array([g["x"]], np.float32))[0] == g["norm2"]


def test_norm_exact_on_integers():
    X = _rng(1).integers(-50, 50, size=(64, 37)).astype(np.float32)
    ref = (X.astype(np.int64) ** 2).sum(axis=1).astype(np.float64)  # exact integer arithmetic
    assert np.array_equal(oracle.norm2(X), ref)


def test_norm_vs_einsum():
    X = _rng(2).standard_normal((500, 300)).astype(np.float32)
    X64 = X.astype(np.float64)
    ref = np.einsum("ij,ij->i", X64, X64)
    got = oracle.norm2(X)
    # different summation order: bounded by d * 2^-53 relative (all terms >= 0)
    assert np.all(np.abs(got - ref) <= 300 * 2.0 ** -53 * ref)


# -------------------------------------------------------------- P2 partition
def _check_partition(nv, m, part, perm, offsets, V):
    n = nv.shape[0]
    sizes = np.diff(offsets)
    assert set(sizes.tolist()) <= {n // m, -(-n // m)}          # Q1: sizes differ by <= 1
    assert np.array_equal(np.sort(perm), np.arange(n))           # exhaustive, disjoint
    for j in range(m):
        ids = perm[offsets[j]:offsets[j + 1]]
        assert np.all(np.diff(ids) > 0)                          # ascending id inside S_j
        assert np.all(part[ids] == j)
        assert V[j] == nv[ids].max()                             # Alg.1 l.6, U_j^2
        if j + 1 < m:
            nxt = perm[offsets[j + 1]:offsets[j + 2]]
            assert nv[ids].max() <= nv[nxt].min()                # ranked ranges


def test_partition_spec_example():
    g = _gold("spec_examples.json")["partition_percentile"]
    nv = np.array(g["norms"]) ** 2
    part, perm, offsets, V = oracle.partition(nv, g["m"])
    assert part.tolist() == g["part"]
    assert np.sqrt(V).tolist() == g["U"]


def test_partition_bruteforce_rank():
    """Alg. 1 l.3-4 by brute force: rank r(i) = #{i' : (||x_i'||, i') < (||x_i||, i)}."""
    rng = _rng(3)
    nv = rng.integers(0, 6, size=53).astype(np.float64)        # many ties
    for m in (1, 2, 5, 7, 53):
        part, perm, offsets, V = oracle.partition(nv, m)
        n = nv.shape[0]
        for i in range(n):
            r = sum(1 for k in range(n) if (nv[k], k) < (nv[i], i))
            assert part[i] == (r * m) // n
        _check_partition(nv, m, part, perm, offsets, V)


@pytest.mark.parametrize("n,m", [(10_000, 8), (17_770, 32), (1000, 8), (4096, 256), (999, 333)])
def test_partition_percentiles(n, m):
    """Boundaries sit at the stated norm percentiles: U_j^2 is the (j+1)/m quantile
    under the nearest-rank (inverted-CDF) rule wherever (j+1)n/m is an integer."""
    nv = _rng(n).lognormal(0, 1, size=n) ** 2
    part, perm, offsets, V = oracle.partition(nv, m)
    _check_partition(nv, m, part, perm, offsets, V)
    checked = 0
    for j in range(m):
        # only where p*n is exact in binary floating point (numpy computes p*n in fp64)
        if ((j + 1) * n) % m == 0 and ((j + 1) / m) * n == (j + 1) * n // m:
            q = np.quantile(nv, (j + 1) / m, method="inverted_cdf")
            assert V[j] == q
            checked += 1
    assert checked >= 1


def test_partition_m1_is_simple_lsh_normaliser():
    """m = 1: U = max ||x|| over S, the SIMPLE-LSH normaliser."""
    nv = _rng(5).pareto(2.5, 1000) ** 2
    _, _, _, V = oracle.partition(nv, 1)
    assert V[0] == nv.max()


def test_partition_all_equal_norms():
    """Ties broken so the percentile split still works."""
    nv = np.full(100, 2.25)
    part, perm, offsets, V = oracle.partition(nv, 4)
    assert np.diff(offsets).tolist() == [25, 25, 25, 25]
    assert np.all(V == 2.25)
    assert part.tolist() == sum([[j] * 25 for j in range(4)], [])


def test_partition_m_gt_n_rejected():
    with pytest.raises(ValueError):
        oracle.partition(np.ones(3), 4)


def test_partition_uniform_spec_example():
    g = _gold("spec_examples.json")["partition_uniform"]
    nv = np.array(g["norms"]) ** 2
    part, perm, offsets, V = oracle.partition(nv, g["m"], scheme="uniform")
    assert part.tolist() == g["part"]


def test_partition_uniform_ranges_are_on_the_norm_not_its_square():
    """Fig. 3(a) / PAPER:1365 split the 2-norm range into equal-width intervals.
    Norms [0, 3, 4, 5], m = 2: the interval width is 2.5, so {0} | {3, 4, 5}; an
    equal-width split of ||x||^2 (width 12.5 over [0, 25]) would give {0, 3} | {4, 5}."""
    nv = np.array([0.0, 3.0, 4.0, 5.0]) ** 2
    part, perm, offsets, V = oracle.partition(nv, 2, scheme="uniform")
    assert part.tolist() == [0, 1, 1, 1]
    assert offsets.tolist() == [0, 1, 4]
    assert V.tolist() == [0.0, 25.0]


def test_partition_uniform_interior_boundaries():
    """An item exactly on an interior boundary u_j = lo + j (hi - lo) / m opens
    sub-dataset j (half-open [u_j, u_{j+1})); the maximum norm closes the last one
    (reading Q19).  All values here are exact in binary."""
    part, _, offsets, V = oracle.partition(np.array([1.0, 2.0, 3.0, 5.0]) ** 2, 2, scheme="uniform")
    assert part.tolist() == [0, 0, 1, 1]                 # 3 = lo + (hi - lo) / 2
    part, _, offsets, V = oracle.partition(np.arange(5.0) ** 2, 4, scheme="uniform")
    assert part.tolist() == [0, 1, 2, 3, 3]              # 1, 2, 3 on boundaries; 4 = max
    assert offsets.tolist() == [0, 1, 2, 3, 5]
    assert V.tolist() == [0.0, 1.0, 4.0, 16.0]
    # empty sub-datasets are allowed; their V is 0
    part, _, offsets, V = oracle.partition(np.array([1.0, 1.1, 9.0, 10.0]) ** 2, 4, scheme="uniform")
    assert part.tolist() == [0, 0, 3, 3] and offsets.tolist() == [0, 2, 2, 2, 4]
    assert V[1] == 0.0 and V[2] == 0.0
    # all norms equal: one non-empty range (hi == lo)
    part, _, offsets, _ = oracle.partition(np.full(6, 2.0), 3, scheme="uniform")
    assert part.tolist() == [0] * 6 and offsets.tolist() == [0, 6, 6, 6]


@pytest.mark.parametrize("m", [1, 3, 7, 32, 256])
def test_partition_uniform_matches_brute_force_edges(m):
    """Brute force, written independently: explicit edges lo + (hi - lo) k / m and
    a search for the interval of every norm (numpy searchsorted), on long-tailed
    norms; perm = ids grouped by interval, ascending id; V = max norm^2 per interval."""
    rng = _rng(11 + m)
    r = np.exp(rng.normal(0.0, 1.0, 20_000))
    nv = r * r
    part, perm, offsets, V = oracle.partition(nv, m, scheme="uniform")
    rr = np.sqrt(nv)
    lo, hi = rr.min(), rr.max()
    edges = lo + (hi - lo) * np.arange(m + 1) / m
    ref = np.clip(np.searchsorted(edges, rr, side="right") - 1, 0, m - 1)
    near = np.min(np.abs(rr[:, None] - edges[None, 1:-1]), axis=1) < 1e-12 * hi if m > 1 \
        else np.zeros(len(rr), bool)
    assert near.sum() <= 2
    assert np.array_equal(part[~near], ref[~near])
    assert np.array_equal(perm, np.argsort(part, kind="stable"))
    assert np.array_equal(offsets, np.concatenate([[0], np.cumsum(np.bincount(part, minlength=m))]))
    for j in range(m):
        sel = nv[part == j]
        assert V[j] == (sel.max() if len(sel) else 0.0)


# -------------------------------------------------------------- P3 transform
def test_transform_spec_examples():
    for g in _gold("spec_examples.json")["transform"]:
        x = np.array(g["x"], np.float32)
        P = oracle.transform(x, g["U"] ** 2, float((x.astype(np.float64) ** 2).sum()))
        assert np.allclose(P, g["P"], rtol=0, atol=1e-7)     # x given in fp32


def test_transform_unit_norm_and_ip():
    """Eq. (8): ||P(x)|| = 1 and P(q)^T P(x) = q^T x / U_j."""
    rng = _rng(7)
    d = 20
    X = (rng.standard_normal((200, d)) * rng.lognormal(0, 1, (200, 1))).astype(np.float32)
    nv = oracle.norm2(X)
    V = nv.max() * 1.7
    q = rng.standard_normal(d)
    q /= np.linalg.norm(q)
    q32 = q.astype(np.float32).astype(np.float64)
    for i in range(200):
        P = oracle.transform(X[i], V, nv[i])
        assert abs(np.linalg.norm(P) - 1.0) < 1e-12
        Pq = np.concatenate([q32, [0.0]])
        assert abs(Pq @ P - (q32 @ X[i].astype(np.float64)) / math.sqrt(V)) < 1e-12


def test_transform_zero_partition():
    P = oracle.transform(np.zeros(4, np.float32), 0.0, 0.0)
    assert P.tolist() == [0, 0, 0, 0, 1.0]


# ----------------------------------------------------- P4 SRP / projection
def test_projection_distribution():
    """a ~ i.i.d. N(0,1) (Eq. (4)): mean, variance, KS test;
    entries are TF32-representable (reading Q14)."""
    from scipy import stats
    A = oracle.projection(12345, 65, 2048).ravel().astype(np.float64)
    N = A.size
    assert abs(A.mean()) < 5 / math.sqrt(N)
    assert abs(A.var() - 1.0) < 5 * math.sqrt(2.0 / N)
    assert stats.kstest(A, "norm").pvalue > 1e-3
    bits = oracle.projection(12345, 65, 2048).view(np.uint32)
    assert np.all(bits & 0x1FFF == 0)
    # different seeds give different matrices; same seed is reproducible
    assert np.array_equal(oracle.projection(1, 3, 64), oracle.projection(1, 3, 64))
    assert not np.array_equal(oracle.projection(1, 3, 64), oracle.projection(2, 3, 64))


def test_sign_hash_identity_directions():
    """identity directions, v = (2, -3) -> bits [1, 0]; the appended
    coordinate t >= 0 hashes to 1 (sign(0) -> 1, reading Q13)."""
    g = _gold("spec_examples.json")["sign_hash_identity"]
    v = np.array([g["v"]], np.float32)
    A = np.zeros((3, 32), np.float32)
    A[0, 0] = 1.0
    A[1, 1] = 1.0
    A[2, 2] = 1.0
    nv = oracle.norm2(v)
    codes = oracle.item_codes(v, np.zeros(1, np.int32), nv * 4.0, nv, A)
    bits = [(int(codes[0, 0]) >> b) & 1 for b in range(3)]
    assert bits[:2] == g["bits"]
    assert bits[2] == 1
    # columns of A that are all zero project to 0 -> bit 1
    assert all(((int(codes[0, 0]) >> b) & 1) == 1 for b in range(3, 32))


@pytest.mark.parametrize("case", range(4))
def test_srp_collision_rate(case):
    """Empirical agreement of sign bits over many projections equals
    1 - acos(cos)/pi (Eq. (4)), within 4 binomial sigma."""
    L = 1 << 17
    A = oracle.projection(777 + case, 3, L)
    # item x in a sub-dataset with normaliser V; query q = e1 (unit)
    xs = [np.array([[0.0, 1.0]]), np.array([[0.5, 0.5]]), np.array([[0.6, 0.0]]),
          np.array([[-0.3, 0.2]])]
    Vs = [1.0, 1.0, 1.0, 0.25]
    x = xs[case].astype(np.float32)
    nv = oracle.norm2(x)
    codes = oracle.item_codes(x, np.zeros(1, np.int32), np.array([Vs[case]]), nv, A)
    q = np.array([[1.0, 0.0]], np.float32)
    qc = oracle.query_codes(q, A)
    agree = L - oracle.hamming(codes[0], qc[0])
    cos = float(x[0, 0]) / math.sqrt(Vs[case])        # P(q)^T P(x), both unit
    p = 1.0 - math.acos(cos) / math.pi
    sigma = math.sqrt(p * (1 - p) / L)
    assert abs(agree / L - p) < 4 * sigma


def test_collision_special_cases():
    """orthogonal -> 0.5, 45 degrees -> 0.75."""
    L = 1 << 17
    A = oracle.projection(4242, 3, L)
    for g in _gold("spec_examples.json")["collision"]:
        x = np.array([g["x"]], np.float32)
        y = np.array([g["y"]], np.float32)
        # use query codes ([v;0]) for both: plain SRP of the raw vectors
        cx = oracle.query_codes(x, A)
        cy = oracle.query_codes(y, A)
        agree = (L - oracle.hamming(cx[0], cy[0])) / L
        sigma = math.sqrt(g["p"] * (1 - g["p"]) / L)
        assert abs(agree - g["p"]) < 4 * sigma


def test_codes_scale_invariant_and_complement():
    rng = _rng(9)
    d, L = 16, 64
    A = oracle.projection(3, d + 1, L)
    q = rng.standard_normal((5, d)).astype(np.float32)
    c1 = oracle.query_codes(q, A)
    c2 = oracle.query_codes(q * 4.0, A)         # exact power-of-two scaling
    c3 = oracle.query_codes(-q, A)
    assert np.array_equal(c1, c2)
    assert np.array_equal(c1 ^ c3, np.full_like(c1, 0xFFFFFFFF))


def test_item_codes_partition_scale_invariant():
    """Scaling a whole sub-dataset by c > 0 leaves P(x), hence the codes, unchanged."""
    rng = _rng(10)
    X = rng.standard_normal((50, 8)).astype(np.float32)
    A = oracle.projection(5, 9, 32)
    nv = oracle.norm2(X)
    part = np.zeros(50, np.int32)
    c1 = oracle.item_codes(X, part, np.array([nv.max()]), nv, A)
    X2 = X * np.float32(2.0)
    nv2 = oracle.norm2(X2)
    c2 = oracle.item_codes(X2, part, np.array([nv2.max()]), nv2, A)
    assert np.array_equal(c1, c2)


def test_m1_reduces_to_simple_lsh():
    """One partition is exactly SIMPLE-LSH:
    U = max ||x||, P(x) = [x/U; sqrt(1 - ||x/U||^2)], bits = sign(a^T P(x))."""
    cfg = workloads.scaled(workloads.CONFIGS["tiny"], 400, 5)
    X = workloads.make_items(cfg)
    idx = oracle.OracleIndex(X, 32, 1, seed=11)
    codes, z = idx.codes(want_z=True)
    X64 = X.astype(np.float64)
    U = np.sqrt((X64 ** 2).sum(1)).max()
    Px = np.concatenate([X64 / U, np.sqrt(np.maximum(0, 1 - ((X64 / U) ** 2).sum(1)))[:, None]], 1)
    zz = Px @ idx.A.astype(np.float64)
    assert np.allclose(z, zz, atol=1e-12)
    bits = (zz >= 0)
    sure = np.abs(zz) > 1e-9
    got = ((codes[:, :, None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(400, 32).astype(bool)
    assert np.array_equal(got[sure], bits[sure])


# ----------------------------------------------------------- P5 rank table
def test_s_hat_spec_examples():
    for g in _gold("spec_examples.json")["s_hat"]:
        h = g["L"] - g["l"]
        assert abs(oracle.s_hat(g["U"], h, g["L"], g["eps"]) - g["s"]) < 1e-15


def test_schedule_worked_example():
    g = _gold("schedule_spec417.json")
    R, order = oracle.rank_table(np.array(g["U"]), g["L"], g["eps"])
    L = g["L"]
    got = [[g["U"][e // (L + 1)], L - (e % (L + 1))] for e in order]
    assert got == g["order_U_l"]


@pytest.mark.parametrize("m,L", [(1, 32), (8, 32), (32, 64), (256, 128)])
def test_rank_table_structure(m, L):
    """Size mL+m (PAPER:217 footnote); R is a permutation; monotone in h within
    each sub-dataset; m = 1 gives plain Hamming ranking."""
    U = np.sort(_rng(m).lognormal(0, 1, m))
    R, order = oracle.rank_table(U, L, 0.01)
    assert R.size == m * L + m
    assert np.array_equal(np.sort(R.ravel()), np.arange(m * (L + 1)))
    assert np.all(np.diff(R.astype(np.int64), axis=1) > 0)
    if m == 1:
        assert R[0].tolist() == list(range(L + 1))


@pytest.mark.parametrize("L,eps", [(32, 0.01), (64, 0.01), (128, 0.01), (64, 0.1), (27, 0.05)])
def test_eps_sign_boundary(L, eps):
    """the adjusted cos < 0 only when l < L[1/2 - eps/(2(1-eps))]."""
    bound = L * (0.5 - eps / (2 * (1 - eps)))
    for h in range(L + 1):
        l = L - h
        s = oracle.s_hat(1.0, h, L, eps)
        if l < bound - 1e-9:
            assert s < 0
        elif l > bound + 1e-9:
            assert s > 0


def test_schedule_order_is_s_hat_desc():
    U = np.array([0.3, 0.9, 1.7, 1.7])
    L = 32
    R, order = oracle.rank_table(U, L, 0.01)
    s = [U[e // (L + 1)] * math.cos(math.pi * 0.99 * (e % (L + 1)) / L) for e in order]
    assert all(s[i] >= s[i + 1] for i in range(len(s) - 1))


# ----------------------------------------------------------- P6 candidates
def test_hamming_spec_examples():
    for g in _gold("spec_examples.json")["hamming"]:
        assert oracle.hamming(np.array([g["a"]]), np.array([g["b"]])) == g["h"]


def _bruteforce_candidates(codes, part, qcode, R, T):
    """The definition D10 written as a sort of all keys (R[j(i)][h(i)], i)."""
    h = _popcount_np(codes ^ qcode[None, :])
    key = R[part, h].astype(np.int64)
    order = np.lexsort((np.arange(codes.shape[0]), key))
    return order[:T], key[order[:T]]


@pytest.mark.parametrize("L,m", [(32, 8), (64, 5), (64, 1), (27, 4)])
def test_candidates_match_sorted_keys(L, m):
    cfg = workloads.scaled(workloads.CONFIGS["tiny"], 3000, 4)
    X = workloads.make_items(cfg)[:, :32]
    idx = oracle.OracleIndex(X, L, m, seed=21)
    codes = idx.codes()
    Q = workloads.make_queries(workloads.scaled(cfg, 3000, 4))[:, :32]
    qc = oracle.query_codes(Q, idx.A)
    for qi in range(4):
        for T in (1, 17, 300, 3000, 5000):
            ids, rk = oracle.candidates(codes, idx.part, qc[qi], idx.R, T)
            bi, bk = _bruteforce_candidates(codes, idx.part, qc[qi], idx.R, min(T, 3000))
            assert np.array_equal(ids, bi)
            assert np.array_equal(rk.astype(np.int64), bk)


def test_candidates_nested_full_and_m1():
    cfg = workloads.scaled(workloads.CONFIGS["tiny"], 2000, 3)
    X = workloads.make_items(cfg)
    idx = oracle.OracleIndex(X, 32, 1, seed=5)
    codes = idx.codes()
    qc = oracle.query_codes(workloads.make_queries(cfg), idx.A)
    full, _ = oracle.candidates(codes, idx.part, qc[0], idx.R, 2000)
    assert np.array_equal(np.sort(full), np.arange(2000))          # T = n: every item
    for T in (5, 50, 500):
        c, _ = oracle.candidates(codes, idx.part, qc[0], idx.R, T)
        assert np.array_equal(c, full[:T])                           # nested in T
    # m = 1: Hamming ranking with id ties = SIMPLE-LSH multi-probe
    h = _popcount_np(codes ^ qc[0][None, :])
    assert np.array_equal(full, np.lexsort((np.arange(2000), h)))


# ------------------------------------------------------- P7 re-rank / exact
def test_brute_force_spec_example():
    g = _gold("spec_examples.json")["brute_force"]
    ids, sc = oracle.exact_topk(np.array(g["X"], np.float32), np.array(g["q"], np.float32), g["k"])
    assert ids.tolist() == g["ids"] and sc.tolist() == g["scores"]


def test_brute_force_orthogonal_ties():
    X = np.array([[0, 1, 0], [0, 0, 1], [0, 2, 2], [0, -1, 3]], np.float32)
    ids, sc = oracle.exact_topk(X, np.array([1, 0, 0], np.float32), 3)
    assert ids.tolist() == [0, 1, 2] and sc.tolist() == [0.0, 0.0, 0.0]


def test_brute_force_vs_numpy():
    rng = _rng(13)
    X = (rng.standard_normal((5000, 24)) * rng.lognormal(0, 1, (5000, 1))).astype(np.float32)
    Q = rng.standard_normal((6, 24)).astype(np.float32)
    S = Q.astype(np.float64) @ X.astype(np.float64).T
    for qi in range(6):
        ids, sc = oracle.exact_topk(X, Q[qi], 10)
        ref = np.lexsort((np.arange(5000), -S[qi]))[:10]
        assert np.array_equal(ids, ref)
        assert np.allclose(sc, S[qi, ref], rtol=1e-12, atol=0)


def test_rerank_padding_and_full_budget():
    cfg = workloads.scaled(workloads.CONFIGS["tiny"], 1500, 3)
    X = workloads.make_items(cfg)
    q = workloads.make_queries(cfg)[0]
    ids, sc = oracle.rerank(X, q, np.array([4, 9, 2], np.int32), 5)
    assert ids[3:].tolist() == [-1, -1] and np.all(np.isneginf(sc[3:]))
    # T = n: the method returns exactly the brute-force top-k
    idx = oracle.OracleIndex(X, 32, 8, seed=1)
    codes = idx.codes()
    a, sa = oracle.query(X, codes, idx.part, idx.R, idx.A, q, 1500, 10)
    b, sb = oracle.exact_topk(X, q, 10)
    assert np.array_equal(a, b) and np.array_equal(sa, sb)


def test_recall_examples():
    """equal -> 1, disjoint -> 0, 5 of 10 -> 0.5."""
    t = np.arange(10)[None, :]
    assert oracle.recall_at_k(t, t) == 1.0
    assert oracle.recall_at_k(t + 10, t) == 0.0
    assert oracle.recall_at_k(np.concatenate([t[:, :5], t[:, :5] + 100], 1), t) == 0.5


def test_bits_split_example():
    """a 16-bit code with 32 sub-datasets = 5 index bits + 11 hash bits
    (the NEXT-1 bit accounting)."""
    g = _gold("spec_examples.json")["bits_split"]
    ib = math.ceil(math.log2(g["m"]))
    assert ib == g["index_bits"] and g["code_bits"] - ib == g["hash_bits"]


def test_range_beats_simple_on_long_tail():
    """Qualitative Fig. 2 pattern -- NOT a parity pin (P8 is unpinned):
    at an equal budget range-lsh's recall is not below simple-lsh's on a
    long-tailed set, averaged over queries."""
    cfg = workloads.scaled(workloads.CONFIGS["c3"], 4000, 40)
    X = workloads.make_items(cfg)[:, :24]
    Q = workloads.make_queries(cfg)[:, :24]
    Q = Q / np.linalg.norm(Q, axis=1, keepdims=True)
    rec = {}
    for m in (1, 16):
        idx = oracle.OracleIndex(X, 32, m, seed=2)
        codes = idx.codes()
        r = []
        for q in Q:
            a, _ = oracle.query(X, codes, idx.part, idx.R, idx.A, q, 200, 10)
            b, _ = oracle.exact_topk(X, q, 10)
            r.append(len(set(a) & set(b)) / 10)
        rec[m] = np.mean(r)
    assert rec[16] >= rec[1] - 0.05


# --------------------------- NEXT-4: per-sub-dataset projections (reading Q4)
def test_pp_one_partition_is_the_shared_projection():
    """seed_j = seed XOR j, so A_0 is the shared A and m = 1 is plain
    SIMPLE-LSH: codes, query codes, candidates and answers equal the shared-A path."""
    cfg = workloads.scaled(workloads.CONFIGS["tiny"], 1500, 6)
    X = workloads.make_items(cfg)
    Q = workloads.make_queries(cfg)
    a = oracle.OracleIndex(X, 32, 1, seed=13)
    b = oracle.OracleIndex(X, 32, 1, seed=13, proj="per_partition")
    assert np.array_equal(b.A_all[0], a.A)
    ca, cb = a.codes(), b.codes()
    assert np.array_equal(ca, cb)
    qa, qb = a.query_codes(Q), b.query_codes(Q)
    assert np.array_equal(qa, qb[:, 0, :])
    for qi in range(len(Q)):
        assert np.array_equal(a.candidates(ca, qa[qi], 200)[0], b.candidates(cb, qb[qi], 200)[0])
        assert np.array_equal(a.query(ca, Q[qi], 200, 10)[0], b.query(cb, Q[qi], 200, 10)[0])


def test_pp_projections_are_independent_gaussians():
    """Each A_j is i.i.d. N(0, 1) (Eq. (4)) and A_j, A_j' are
    uncorrelated (independent hash families per sub-index)."""
    from scipy import stats
    A = oracle.projection_pp(99, 3, 65, 512).astype(np.float64)
    for j in range(3):
        assert stats.kstest(A[j].ravel(), "norm").pvalue > 1e-3
        assert np.array_equal(A[j], oracle.projection(99 ^ j, 65, 512))
    for j, jj in ((0, 1), (1, 2), (0, 2)):
        r = np.corrcoef(A[j].ravel(), A[jj].ravel())[0, 1]
        assert abs(r) < 4.0 / math.sqrt(A[j].size)


def test_pp_collision_law_per_sub_index():
    """Within sub-index j the bits of P(x) and P(q) = [q; 0] under A_j agree with
    probability 1 - acos(q.x/(U_j|q|))/pi (Eq. (4)); a query
    code taken under another sub-index's projection agrees with probability 1/2
    (independent hyperplanes) — so an item must be compared with the query's code
    of its own sub-index."""
    L = 1 << 16
    m = 2
    A_all = oracle.projection_pp(31, m, 3, L)
    X = np.array([[0.6, 0.0], [0.0, 0.9], [0.3, 0.3], [0.5, -0.5]], np.float32)
    part = np.array([0, 0, 1, 1], np.int32)
    nv = oracle.norm2(X)
    V = np.array([nv[:2].max(), nv[2:].max()])
    codes = oracle.item_codes_pp(X, part, V, nv, A_all)
    q = np.array([[1.0, 0.0]], np.float32)
    qc = oracle.query_codes_pp(q, A_all)[0]            # [m, W]
    for i in range(4):
        j = part[i]
        p = 1.0 - math.acos(float(X[i, 0]) / math.sqrt(V[j])) / math.pi
        sig = math.sqrt(p * (1 - p) / L)
        agree = (L - oracle.hamming(codes[i], qc[j])) / L
        assert abs(agree - p) < 4 * sig, (i, agree, p)
        other = (L - oracle.hamming(codes[i], qc[1 - j])) / L
        assert abs(other - 0.5) < 4 * math.sqrt(0.25 / L), (i, other)


@pytest.mark.parametrize("L,m", [(32, 8), (64, 5), (17, 3)])
def test_pp_candidates_match_sorted_keys(L, m):
    """D10 with per-sub-index query codes, against a brute-force sort of all keys
    (R[j(i)][popc(code_i ^ qcode_q[j(i)])], i) written here with numpy."""
    cfg = workloads.scaled(workloads.CONFIGS["tiny"], 2500, 4)
    X = workloads.make_items(cfg)[:, :24]
    Q = workloads.make_queries(cfg)[:, :24]
    idx = oracle.OracleIndex(X, L, m, seed=7, proj="per_partition")
    codes = idx.codes()
    qc = idx.query_codes(Q)
    for qi in range(4):
        h = _popcount_np(codes ^ qc[qi][idx.part])
        key = idx.R[idx.part, h].astype(np.int64)
        order = np.lexsort((np.arange(len(X)), key))
        for T in (1, 40, 900, 2500, 4000):
            ids, rk = idx.candidates(codes, qc[qi], T)
            t = min(T, len(X))
            assert np.array_equal(ids, order[:t])
            assert np.array_equal(rk.astype(np.int64), key[order[:t]])


def test_pp_codes_use_each_items_own_projection():
    """Every item's per-sub-index code equals the shared-A oracle code of that item
    computed with A := A_{j(i)} (D5 applied sub-index by sub-index), and the
    query codes equal the shared-A query codes under each A_j."""
    cfg = workloads.scaled(workloads.CONFIGS["c2"], 900, 5)
    X = workloads.make_items(cfg)[:, :40]
    Q = workloads.make_queries(cfg)[:, :40]
    idx = oracle.OracleIndex(X, 64, 6, seed=3, proj="per_partition")
    codes = idx.codes()
    for j in range(6):
        sel = idx.part == j
        ref = oracle.item_codes(X[sel], idx.part[sel], idx.V, idx.norm2[sel], idx.A_all[j])
        assert np.array_equal(codes[sel], ref)
    qc = idx.query_codes(Q)
    for j in range(6):
        assert np.array_equal(qc[:, j, :], oracle.query_codes(Q, idx.A_all[j]))
    # T = n: every item is probed, so the answer is the brute-force top-k
    for qi in range(len(Q)):
        a, _ = idx.query(codes, Q[qi], len(X), 10)
        b, _ = oracle.exact_topk(X, Q[qi], 10)
        assert np.array_equal(a, b)
