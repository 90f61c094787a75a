/*
 * nrlsh_oracle.c — plain, slow, obviously-correct CPU reference of the
 * norm-ranging LSH (RANGE-LSH) hot path, in fp64.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load or call this
 * library.  The product path (paper_1809_08782_b200/) never links, imports
 * or executes anything under oracle/, and this file shares no code, header,
 * table or constant generator with the CUDA path.
 *
 * Citations are to /root/reference/PAPER.md (LaTeX source of arXiv
 * 1809.08782) as PAPER:<line>, and to the readings D1..D13 / Q1..Q18 listed
 * in DESIGN.md ("Readings of the paper").
 *
 * Every function follows the paper's step order and notation:
 *   Alg. 1 (index building)
 *   Eq. (8) SIMPLE-LSH transform PAPER:83-88
 *   Eq. (4) sign random projection PAPER:53-57
 *   Eq. (12) + eps adjustment
 *   sorted (U_j, l) structure
 *   Alg. 2 (query processing)
 *   Eq. (1) MIPS
 *
 * No blocking, fusion or reordering: sums run strictly left to right.
 * Compile with -O2 -ffp-contract=off (no -ffast-math).
 *
 * Parity status of each function is stated in DESIGN.md §"Oracle pins";
 * every function here is pinned by a `-m "not gpu"` test in
 * tests/test_oracle_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_ENOMEM (-2)

/* ------------------------------------------------------------------ */
/* D2: squared 2-norm, fp64, sequential over k = 0..d-1.               */
/* Alg. 1 line 3 "Rank the items in S according to their 2-norms"     */
/* (PAPER:151).  (double)x*(double)x is exact, so fma or mul+add agree. */
/* ------------------------------------------------------------------ */
void orc_norm2(const float *X, int64_t n, int32_t d, double *norm2)
{
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int32_t k = 0; k < d; ++k) {
            double v = (double)X[i * (int64_t)d + k];
            s = s + v * v;
        }
        norm2[i] = s;
    }
}

/* ------------------------------------------------------------------ */
/* D1: percentile partition (Alg. 1 lines 3-4).         */
/* Rank by (norm2 ascending, id ascending) -- the paper breaks ties    */
/* "arbitrarily"; reading Q2 fixes ascending id.  Item of  */
/* rank r goes to sub-dataset j = floor(r*m/n) (reading Q1: half-open  */
/* rank ranges).  perm lists ids grouped by j, ascending id within j.  */
/* V[j] = max norm2 in S_j  (Alg. 1 line 6: U_j = max ||x||, U_j^2=V_j)*/
/* ------------------------------------------------------------------ */
typedef struct {
    double key;
    int64_t id;
} orc_kv;

static int orc_cmp_kv(const void *a, const void *b)
{
    const orc_kv *x = (const orc_kv *)a, *y = (const orc_kv *)b;
    if (x->key < y->key) return -1;
    if (x->key > y->key) return 1;
    if (x->id < y->id) return -1;
    if (x->id > y->id) return 1;
    return 0;
}

int orc_partition(const double *norm2, int64_t n, int32_t m,
                  int32_t *part, int32_t *perm, int64_t *offsets, double *V)
{
    if (n < 1 || m < 1 || (int64_t)m > n) return ORC_EINVAL;
    orc_kv *kv = (orc_kv *)malloc(sizeof(orc_kv) * (size_t)n);
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
    if (!kv || !cursor) { free(kv); free(cursor); return ORC_ENOMEM; }
    for (int64_t i = 0; i < n; ++i) { kv[i].key = norm2[i]; kv[i].id = i; }
    /* "Rank the items in S according to their 2-norms" */
    qsort(kv, (size_t)n, sizeof(orc_kv), orc_cmp_kv);
    /* "Partition S into m sub-datasets ... ranked in the range
        [(j-1)n/m, jn/m]" */
    for (int64_t r = 0; r < n; ++r) {
        int64_t j = (r * (int64_t)m) / n;
        part[kv[r].id] = (int32_t)j;
    }
    for (int32_t j = 0; j <= m; ++j) offsets[j] = 0;
    for (int64_t i = 0; i < n; ++i) offsets[part[i] + 1] += 1;
    for (int32_t j = 0; j < m; ++j) offsets[j + 1] += offsets[j];
    for (int32_t j = 0; j < m; ++j) cursor[j] = offsets[j];
    for (int64_t i = 0; i < n; ++i) perm[cursor[part[i]]++] = (int32_t)i;
    /* "Use U_j = max_{x in S_j} ||x|| to normalize S_j" (squared here) */
    for (int32_t j = 0; j < m; ++j) {
        double vmax = 0.0;
        int first = 1;
        for (int64_t p = offsets[j]; p < offsets[j + 1]; ++p) {
            double v = norm2[perm[p]];
            if (first || v > vmax) { vmax = v; first = 0; }
        }
        V[j] = vmax;
    }
    free(kv);
    free(cursor);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* NEXT-2 (Fig. 3(a)): uniform partitioning.  Sub-dataset  */
/* j holds items whose 2-norm lies in the j-th of m equal-width        */
/* intervals of [min ||x||, max ||x||]; empty sub-datasets allowed.     */
/* Item with ||x|| = max goes to j = m-1.  perm/offsets/V as above     */
/* (V[j] = 0 for an empty sub-dataset).                                 */
/* ------------------------------------------------------------------ */
int orc_partition_uniform(const double *norm2, int64_t n, int32_t m,
                          int32_t *part, int32_t *perm, int64_t *offsets,
                          double *V)
{
    if (n < 1 || m < 1) return ORC_EINVAL;
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
    if (!cursor) return ORC_ENOMEM;
    double lo = sqrt(norm2[0]), hi = sqrt(norm2[0]);
    for (int64_t i = 1; i < n; ++i) {
        double r = sqrt(norm2[i]);
        if (r < lo) lo = r;
        if (r > hi) hi = r;
    }
    for (int64_t i = 0; i < n; ++i) {
        double r = sqrt(norm2[i]);
        int64_t j = 0;
        if (hi > lo) {
            j = (int64_t)floor((r - lo) / (hi - lo) * (double)m);
            if (j >= m) j = m - 1;
            if (j < 0) j = 0;
        }
        part[i] = (int32_t)j;
    }
    for (int32_t j = 0; j <= m; ++j) offsets[j] = 0;
    for (int64_t i = 0; i < n; ++i) offsets[part[i] + 1] += 1;
    for (int32_t j = 0; j < m; ++j) offsets[j + 1] += offsets[j];
    for (int32_t j = 0; j < m; ++j) cursor[j] = offsets[j];
    for (int64_t i = 0; i < n; ++i) perm[cursor[part[i]]++] = (int32_t)i;
    for (int32_t j = 0; j < m; ++j) {
        double vmax = 0.0;
        for (int64_t p = offsets[j]; p < offsets[j + 1]; ++p) {
            double v = norm2[perm[p]];
            if (v > vmax) vmax = v;
        }
        V[j] = vmax;
    }
    free(cursor);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* D3: Eq. (8) applied after Alg. 1 line 6.         */
/* P(x) = [x/U_j ; sqrt(1 - ||x/U_j||^2)], written with                */
/* t = sqrt(max(0, V_j - ||x||^2)) as [x/U_j ; t/U_j].                  */
/* A sub-dataset of zero vectors (V_j = 0) maps to [0;1] (reading D3). */
/* ------------------------------------------------------------------ */
void orc_transform(const float *x, int32_t d, double Vj, double norm2x,
                   double *out)
{
    if (Vj == 0.0) {
        for (int32_t k = 0; k < d; ++k) out[k] = 0.0;
        out[d] = 1.0;
        return;
    }
    double U = sqrt(Vj);
    double diff = Vj - norm2x;
    double t = sqrt(diff > 0.0 ? diff : 0.0);
    for (int32_t k = 0; k < d; ++k) out[k] = (double)x[k] / U;
    out[d] = t / U;
}

/* ------------------------------------------------------------------ */
/* D4: projection vectors a ~ N(0, I) (Eq. (4)).           */
/* Counter-based SplitMix64 -> Box-Muller in fp64 -> fp32 -> rounded   */
/* to nearest-even TF32 (11 significant bits, reading Q14).             */
/* Entry e = k*L + b is A[k][b], k in [0, rows), b in [0, L).          */
/* (independent re-implementation of the generator documented in       */
/*  include/nrlsh.h; written separately from the library's)            */
/* ------------------------------------------------------------------ */
static uint64_t orc_splitmix64_at(uint64_t seed, uint64_t ctr)
{
    uint64_t z = seed + (ctr + 1u) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static float orc_round_tf32(double z)
{
    float f = (float)z;
    uint32_t u;
    memcpy(&u, &f, 4);
    uint32_t lsb = (u >> 13) & 1u;
    u = u + 0x0FFFu + lsb;
    u = u & 0xFFFFE000u;
    memcpy(&f, &u, 4);
    return f;
}

void orc_projection(uint64_t seed, int32_t rows, int32_t L, float *A)
{
    const double two_pi = 2.0 * 3.14159265358979323846;
    for (int64_t k = 0; k < rows; ++k) {
        for (int64_t b = 0; b < L; ++b) {
            uint64_t e = (uint64_t)(k * L + b);
            uint64_t r1 = orc_splitmix64_at(seed, 2u * e);
            uint64_t r2 = orc_splitmix64_at(seed, 2u * e + 1u);
            double u1 = (double)((r1 >> 11) + 1u) * (1.0 / 9007199254740992.0);
            double u2 = (double)(r2 >> 11) * (1.0 / 9007199254740992.0);
            double g = sqrt(-2.0 * log(u1)) * cos(two_pi * u2);
            A[k * L + b] = orc_round_tf32(g);
        }
    }
}

/* ------------------------------------------------------------------ */
/* D5: item code.  Sign random projection of P(x) (Eq. (4)):  */
/* z_b = sum_{k=0}^{d} A[k][b] * P(x)_k  (fp64, sequential);            */
/* bit b = [z_b >= 0] (sign(0) -> 1, reading Q13).  Bit b sits in word */
/* b/32 at position b%32.  codes: n x ceil(L/32) words, id order;      */
/* bits >= L are 0.                                                    */
/* z (optional, n x L) receives the fp64 projections for the parity    */
/* checker's 1e-5 exemption band.                                       */
/* ------------------------------------------------------------------ */
int orc_item_codes(const float *X, int64_t n, int32_t d,
                   const int32_t *part, const double *V, const double *norm2,
                   const float *A, int32_t L, uint32_t *codes, double *z)
{
    if (L < 1) return ORC_EINVAL;
    int32_t W = (L + 31) / 32;   /* bits >= L stay 0 (NEXT-1 bit accounting) */
    double *P = (double *)malloc(sizeof(double) * (size_t)(d + 1));
    if (!P) return ORC_ENOMEM;
    for (int64_t i = 0; i < n; ++i) {
        orc_transform(X + i * (int64_t)d, d, V[part[i]], norm2[i], P);
        for (int32_t w = 0; w < W; ++w) codes[i * W + w] = 0u;
        for (int32_t b = 0; b < L; ++b) {
            double s = 0.0;
            for (int32_t k = 0; k <= d; ++k)
                s = s + (double)A[(int64_t)k * L + b] * P[k];
            if (z) z[i * (int64_t)L + b] = s;
            if (s >= 0.0) codes[i * W + b / 32] |= (1u << (b % 32));
        }
    }
    free(P);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* D6: query code, P(q) = [q; 0] (Eq. (8)):                  */
/* bit b = [sum_{k<d} A[k][b] q_k >= 0].                                */
/* ------------------------------------------------------------------ */
int orc_query_codes(const float *Q, int64_t nq, int32_t d, const float *A,
                    int32_t L, uint32_t *qcodes, double *z)
{
    if (L < 1) return ORC_EINVAL;
    int32_t W = (L + 31) / 32;
    for (int64_t i = 0; i < nq; ++i) {
        for (int32_t w = 0; w < W; ++w) qcodes[i * W + w] = 0u;
        for (int32_t b = 0; b < L; ++b) {
            double s = 0.0;
            for (int32_t k = 0; k < d; ++k)
                s = s + (double)A[(int64_t)k * L + b] * (double)Q[i * (int64_t)d + k];
            /* the appended coordinate of P(q) is 0: A[d][b]*0 adds nothing */
            if (z) z[i * (int64_t)L + b] = s;
            if (s >= 0.0) qcodes[i * W + b / 32] |= (1u << (b % 32));
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* D7: Hamming distance h = popcount(code XOR qcode); l = L - h is the  */
/* number of identical hashes.  Plain bit loop.            */
/* ------------------------------------------------------------------ */
static int32_t orc_popcount32(uint32_t v)
{
    int32_t c = 0;
    for (int b = 0; b < 32; ++b) c += (int32_t)((v >> b) & 1u);
    return c;
}

int32_t orc_hamming(const uint32_t *a, const uint32_t *b, int32_t W)
{
    int32_t h = 0;
    for (int32_t w = 0; w < W; ++w) h += orc_popcount32(a[w] ^ b[w]);
    return h;
}

/* ------------------------------------------------------------------ */
/* D8: similarity metric, Eq. (12) with the epsilon adjustment         */
/* (PAPER:211-215):  s_hat = U_j * cos[pi (1-eps) (1 - l/L)],  and      */
/* 1 - l/L = h/L, evaluated as U_j * cos(((pi*(1-eps))*h)/L).           */
/* ------------------------------------------------------------------ */
double orc_s_hat(double Uj, int32_t h, int32_t L, double eps)
{
    const double pi = 3.14159265358979323846;
    return Uj * cos(pi * (1.0 - eps) * (double)h / (double)L);
}

/* ------------------------------------------------------------------ */
/* D9: the sorted (U_j, l) structure of PAPER:217 (size mL+m).          */
/* Entries (j, h) for j < m, 0 <= h <= L, ordered by s_hat descending   */
/* ("traversing the sorted structure", reading Q8: most similar first), */
/* ties by U_j desc, then h asc, then j asc (reading Q9).               */
/* R[j*(L+1)+h] = position of (j,h);  order[p] = j*(L+1)+h (optional). */
/* ------------------------------------------------------------------ */
typedef struct {
    double s, U;
    int32_t j, h;
} orc_sched;

static int orc_cmp_sched(const void *a, const void *b)
{
    const orc_sched *x = (const orc_sched *)a, *y = (const orc_sched *)b;
    if (x->s > y->s) return -1;
    if (x->s < y->s) return 1;
    if (x->U > y->U) return -1;
    if (x->U < y->U) return 1;
    if (x->h < y->h) return -1;
    if (x->h > y->h) return 1;
    if (x->j < y->j) return -1;
    if (x->j > y->j) return 1;
    return 0;
}

int orc_rank_table(const double *U, int32_t m, int32_t L, double eps,
                   uint16_t *R, int32_t *order)
{
    int64_t cnt = (int64_t)m * (L + 1);
    if (m < 1 || L < 1 || cnt > 65536) return ORC_EINVAL;
    orc_sched *s = (orc_sched *)malloc(sizeof(orc_sched) * (size_t)cnt);
    if (!s) return ORC_ENOMEM;
    int64_t e = 0;
    for (int32_t j = 0; j < m; ++j)
        for (int32_t h = 0; h <= L; ++h) {
            s[e].s = orc_s_hat(U[j], h, L, eps);
            s[e].U = U[j];
            s[e].j = j;
            s[e].h = h;
            ++e;
        }
    qsort(s, (size_t)cnt, sizeof(orc_sched), orc_cmp_sched);
    for (int64_t p = 0; p < cnt; ++p) {
        R[(int64_t)s[p].j * (L + 1) + s[p].h] = (uint16_t)p;
        if (order) order[p] = s[p].j * (L + 1) + s[p].h;
    }
    free(s);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* D10: candidate generation for one query = single-table multi-probe  */
/* over all sub-indexes: walk the sorted structure;   */
/* for entry (j, l) take the items of S_j that agree with the query in */
/* exactly l bits (h = L - l), in ascending id ("standard hash lookup",*/
/* reading Q10), until exactly T items are taken.                       */
/* codes: n x W words in item-id order; part[i] = sub-dataset of item i.*/
/* Output: cand_ids[T'] and cand_rank[T'] (position of (j,h)),          */
/* T' = min(T, n).  Returns T' (or a negative error).                   */
/* ------------------------------------------------------------------ */
int64_t orc_candidates(const uint32_t *codes, const int32_t *part, int64_t n,
                       int32_t L, const uint32_t *qcode, const uint16_t *R,
                       int32_t m, int64_t T, int32_t *cand_ids,
                       uint16_t *cand_rank)
{
    if (L < 1 || T < 1) return ORC_EINVAL;
    int32_t W = (L + 31) / 32;
    int64_t nent = (int64_t)m * (L + 1);
    int64_t Tp = T < n ? T : n;
    /* bucket[p] = items whose (j, h) sits at position p, in ascending id */
    int64_t *start = (int64_t *)calloc((size_t)nent + 1, sizeof(int64_t));
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)nent);
    int32_t *key = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t *items = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (!start || !fill || !key || !items) {
        free(start); free(fill); free(key); free(items);
        return ORC_ENOMEM;
    }
    for (int64_t i = 0; i < n; ++i) {
        int32_t h = orc_hamming(codes + i * W, qcode, W);
        key[i] = (int32_t)R[(int64_t)part[i] * (L + 1) + h];
        start[key[i] + 1] += 1;
    }
    for (int64_t p = 0; p < nent; ++p) start[p + 1] += start[p];
    for (int64_t p = 0; p < nent; ++p) fill[p] = start[p];
    for (int64_t i = 0; i < n; ++i) items[fill[key[i]]++] = (int32_t)i;
    /* traverse the sorted structure until the probe budget is spent */
    int64_t taken = 0;
    for (int64_t p = 0; p < nent && taken < Tp; ++p) {
        for (int64_t e = start[p]; e < start[p + 1] && taken < Tp; ++e) {
            cand_ids[taken] = items[e];
            cand_rank[taken] = (uint16_t)p;
            ++taken;
        }
    }
    free(start); free(fill); free(key); free(items);
    return taken;
}

/* ------------------------------------------------------------------ */
/* D11: verify the probed items by exact inner product (Alg. 2 line 6,  */
/* PAPER:169; reading Q12) and return the top k by (score desc, id asc).*/
/* Missing slots are padded with (-1, -inf).                            */
/* ------------------------------------------------------------------ */
typedef struct {
    double s;
    int64_t id;
} orc_scored;

static int orc_cmp_scored(const void *a, const void *b)
{
    const orc_scored *x = (const orc_scored *)a, *y = (const orc_scored *)b;
    if (x->s > y->s) return -1;
    if (x->s < y->s) return 1;
    if (x->id < y->id) return -1;
    if (x->id > y->id) return 1;
    return 0;
}

int orc_rerank(const float *X, int64_t n, int32_t d, const float *q,
               const int32_t *cand_ids, int64_t ncand, int32_t k,
               int64_t *out_ids, double *out_scores)
{
    (void)n;
    if (k < 1) return ORC_EINVAL;
    orc_scored *sc = (orc_scored *)malloc(sizeof(orc_scored) * (size_t)(ncand > 0 ? ncand : 1));
    if (!sc) return ORC_ENOMEM;
    for (int64_t c = 0; c < ncand; ++c) {
        int64_t i = cand_ids[c];
        double s = 0.0;
        for (int32_t t = 0; t < d; ++t)
            s = s + (double)q[t] * (double)X[i * (int64_t)d + t];
        sc[c].s = s;
        sc[c].id = i;
    }
    qsort(sc, (size_t)ncand, sizeof(orc_scored), orc_cmp_scored);
    for (int32_t r = 0; r < k; ++r) {
        if (r < ncand) { out_ids[r] = sc[r].id; out_scores[r] = sc[r].s; }
        else { out_ids[r] = -1; out_scores[r] = -INFINITY; }
    }
    free(sc);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* D12: exact MIPS ground truth, Eq. (1): top k of q^T x  */
/* over all n items, (score desc, id asc).                              */
/* ------------------------------------------------------------------ */
int orc_exact_topk(const float *X, int64_t n, int32_t d, const float *q,
                   int32_t k, int64_t *out_ids, double *out_scores)
{
    int32_t *all = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (!all) return ORC_ENOMEM;
    for (int64_t i = 0; i < n; ++i) all[i] = (int32_t)i;
    int rc = orc_rerank(X, n, d, q, all, n, k, out_ids, out_scores);
    free(all);
    return rc;
}

/* ------------------------------------------------------------------ */
/* One whole query of the method (Alg. 2 merged with multi-probe):     */
/* query code -> candidates (T) -> exact re-rank -> top k.  Used for    */
/* the CPU baseline timing and end-to-end parity.                       */
/* ------------------------------------------------------------------ */
int orc_query(const float *X, int64_t n, int32_t d, const uint32_t *codes,
              const int32_t *part, const uint16_t *R, int32_t m,
              const float *A, int32_t L, const float *q, int64_t T,
              int32_t k, int64_t *out_ids, double *out_scores)
{
    uint32_t qcode[8];
    if (L > 256) return ORC_EINVAL;
    int rc = orc_query_codes(q, 1, d, A, L, qcode, NULL);
    if (rc) return rc;
    int64_t Tp = T < n ? T : n;
    int32_t *cid = (int32_t *)malloc(sizeof(int32_t) * (size_t)Tp);
    uint16_t *crk = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)Tp);
    if (!cid || !crk) { free(cid); free(crk); return ORC_ENOMEM; }
    int64_t got = orc_candidates(codes, part, n, L, qcode, R, m, T, cid, crk);
    if (got < 0) { free(cid); free(crk); return (int)got; }
    rc = orc_rerank(X, n, d, q, cid, got, k, out_ids, out_scores);
    free(cid);
    free(crk);
    return rc;
}

/* ================================================================== */
/* Per-sub-dataset projections (reading Q4).  */
/* Alg. 1 l.7 "Apply SIMPLE-LSH to build index I_j for S_j"           */
/* (PAPER:155), "building a hash index for each sub-dataset            */
/* independently": sub-index j draws its own projection A_j, */
/* from the documented generator with seed_j = seed XOR j (SPEC:453,   */
/* "seed (+) j"), so A_0 is the shared projection and m = 1 is plain   */
/* SIMPLE-LSH again.  The query is hashed once per sub-index            */
/* ("hash q once per sub-index"), and an item of S_j is      */
/* compared with the query's code under A_j.                           */
/* A_all: m blocks of (d+1) x L, block j = A_j.                         */
/* ================================================================== */
void orc_projection_pp(uint64_t seed, int32_t m, int32_t rows, int32_t L, float *A_all)
{
    for (int32_t j = 0; j < m; ++j)
        orc_projection(seed ^ (uint64_t)j, rows, L, A_all + (int64_t)j * rows * L);
}

/* D5 with A := A_{j(i)}: each item is hashed by its own sub-index.      */
int orc_item_codes_pp(const float *X, int64_t n, int32_t d,
                      const int32_t *part, const double *V, const double *norm2,
                      const float *A_all, int32_t L, uint32_t *codes, double *z)
{
    if (L < 1) return ORC_EINVAL;
    int32_t W = (L + 31) / 32;
    for (int64_t i = 0; i < n; ++i) {
        const float *Aj = A_all + (int64_t)part[i] * (d + 1) * L;
        int rc = orc_item_codes(X + i * (int64_t)d, 1, d, part + i, V, norm2 + i, Aj, L,
                                codes + i * W, z ? z + i * (int64_t)L : NULL);
        if (rc) return rc;
    }
    return ORC_OK;
}

/* D6 once per sub-index: qcodes [nq x m x W], z [nq x m x L].          */
int orc_query_codes_pp(const float *Q, int64_t nq, int32_t d, const float *A_all,
                       int32_t m, int32_t L, uint32_t *qcodes, double *z)
{
    if (L < 1 || m < 1) return ORC_EINVAL;
    int32_t W = (L + 31) / 32;
    for (int64_t i = 0; i < nq; ++i)
        for (int32_t j = 0; j < m; ++j) {
            int rc = orc_query_codes(Q + i * (int64_t)d, 1, d, A_all + (int64_t)j * (d + 1) * L, L,
                                     qcodes + (i * m + j) * W,
                                     z ? z + (i * m + j) * (int64_t)L : NULL);
            if (rc) return rc;
        }
    return ORC_OK;
}

/* D10 with per-sub-index query codes: qcodes [m x W]; item i is compared */
/* with the query's code of its own sub-dataset, qcodes[part[i]].         */
int64_t orc_candidates_pp(const uint32_t *codes, const int32_t *part, int64_t n,
                          int32_t L, const uint32_t *qcodes, const uint16_t *R,
                          int32_t m, int64_t T, int32_t *cand_ids,
                          uint16_t *cand_rank)
{
    if (L < 1 || T < 1) return ORC_EINVAL;
    int32_t W = (L + 31) / 32;
    int64_t nent = (int64_t)m * (L + 1);
    int64_t Tp = T < n ? T : n;
    int64_t *start = (int64_t *)calloc((size_t)nent + 1, sizeof(int64_t));
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)nent);
    int32_t *key = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t *items = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (!start || !fill || !key || !items) {
        free(start); free(fill); free(key); free(items);
        return ORC_ENOMEM;
    }
    for (int64_t i = 0; i < n; ++i) {
        int32_t h = orc_hamming(codes + i * W, qcodes + (int64_t)part[i] * W, W);
        key[i] = (int32_t)R[(int64_t)part[i] * (L + 1) + h];
        start[key[i] + 1] += 1;
    }
    for (int64_t p = 0; p < nent; ++p) start[p + 1] += start[p];
    for (int64_t p = 0; p < nent; ++p) fill[p] = start[p];
    for (int64_t i = 0; i < n; ++i) items[fill[key[i]]++] = (int32_t)i;
    int64_t taken = 0;
    for (int64_t p = 0; p < nent && taken < Tp; ++p) {
        for (int64_t e = start[p]; e < start[p + 1] && taken < Tp; ++e) {
            cand_ids[taken] = items[e];
            cand_rank[taken] = (uint16_t)p;
            ++taken;
        }
    }
    free(start); free(fill); free(key); free(items);
    return taken;
}

/* One whole query with per-sub-index projections.                       */
int orc_query_pp(const float *X, int64_t n, int32_t d, const uint32_t *codes,
                 const int32_t *part, const uint16_t *R, int32_t m,
                 const float *A_all, int32_t L, const float *q, int64_t T,
                 int32_t k, int64_t *out_ids, double *out_scores)
{
    if (L > 256 || m < 1) return ORC_EINVAL;
    int32_t W = (L + 31) / 32;
    uint32_t *qc = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)m * W);
    int64_t Tp = T < n ? T : n;
    int32_t *cid = (int32_t *)malloc(sizeof(int32_t) * (size_t)Tp);
    uint16_t *crk = (uint16_t *)malloc(sizeof(uint16_t) * (size_t)Tp);
    if (!qc || !cid || !crk) { free(qc); free(cid); free(crk); return ORC_ENOMEM; }
    int rc = orc_query_codes_pp(q, 1, d, A_all, m, L, qc, NULL);
    if (!rc) {
        int64_t got = orc_candidates_pp(codes, part, n, L, qc, R, m, T, cid, crk);
        rc = got < 0 ? (int)got : orc_rerank(X, n, d, q, cid, got, k, out_ids, out_scores);
    }
    free(qc);
    free(cid);
    free(crk);
    return rc;
}
