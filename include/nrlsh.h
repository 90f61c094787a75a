/*
 * nrlsh.h — C ABI of the B200-native norm-ranging LSH (RANGE-LSH) library
 * (libnrlsh.so, sm_100a).  Method: arXiv 1809.08782, /root/reference/PAPER.md
 * cited as PAPER:<line>.
 *
 * Conventions (all entry points):
 *  - Plain pointers and sizes only.  A pointer argument may be DEVICE memory or
 *    HOST memory (pageable or pinned); the library detects which with
 *    cudaPointerGetAttributes and stages host buffers through device memory
 *    itself (host<->device copies then happen inside the call).
 *  - Every entry point validates its arguments and returns an nrlsh_status;
 *    no C++ exception ever crosses the ABI.  On error, nrlsh_last_error()
 *    returns a thread-local message naming the offending argument or index
 *    (e.g. "zero-norm query at index 7").
 *  - Work is enqueued on `cuda_stream` (a cudaStream_t, or NULL for the legacy
 *    default stream).  nrlsh_build, nrlsh_query and nrlsh_exact_topk
 *    synchronise that stream before returning so that device-side validation
 *    (non-finite items, zero-norm queries) is reported in the return value.
 *  - Row-major fp32 matrices: items X [n x d], queries Q [nq x d].
 *  - Single GPU: the device current on the calling thread.
 */
#ifndef NRLSH_H
#define NRLSH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nrlsh_index nrlsh_index; /* opaque; owns its device buffers */

typedef enum {
    NRLSH_OK = 0,
    NRLSH_EINVAL = 1,     /* bad argument (sizes, k < 1, T < 1, m > n, bits) */
    NRLSH_ENONFINITE = 2, /* NaN/Inf in an item or query (index recorded)      */
    NRLSH_EZERONORM = 3,  /* zero-norm query (index recorded)                  */
    NRLSH_ENOMEM = 4,     /* device or host allocation failed                  */
    NRLSH_ECUDA = 5,      /* CUDA runtime error (message recorded)             */
    NRLSH_ENOTIMPL = 6    /* option not implemented                            */
} nrlsh_status;

enum { NRLSH_SCHEME_PERCENTILE = 0, /* Alg. 1 l.4             */
       NRLSH_SCHEME_UNIFORM = 1 };  /* equal-width norm ranges */

/* Hash functions of the sub-indexes ("Apply SIMPLE-LSH to build index I_j for S_j",
   Alg. 1 l.7).  SHARED: one projection A for every sub-dataset (one
   query code per query).  PER_PARTITION: sub-index j draws its own A_j with seed
   seed XOR j, so A_0 = A; the query is hashed once per sub-index and an
   item of S_j is compared with the query's code under A_j. */
enum { NRLSH_PROJ_SHARED = 0, NRLSH_PROJ_PER_PARTITION = 1 };

typedef struct nrlsh_options {
    double eps;            /* metric adjustment of PAPER:215, 0 <= eps < 1; default 0.01 */
    int32_t scheme;        /* NRLSH_SCHEME_*; default PERCENTILE                        */
    int32_t index_bits_in_budget; /* 1: code_bits counts ceil(log2 m) partition-index bits
                                     (PAPER:1075), so L_h = code_bits - ceil(log2 m);
                                     0 (default): all code_bits are SRP hash bits         */
    int32_t query_batch;   /* queries per internal sub-batch; 0 -> 1024                  */
    int32_t proj;          /* NRLSH_PROJ_*; default SHARED.  PER_PARTITION needs the
                              tensor-core code kernel's shapes (d <= 512, L_h <= 128,
                              ceil(L_h/32) != 3), else NRLSH_ENOTIMPL                  */
} nrlsh_options;

/* Fill *opt with the defaults above. */
void nrlsh_default_options(nrlsh_options *opt);

/*
 * nrlsh_build — index building, Alg. 1:
 *   rank items by 2-norm, split into `num_parts` sub-datasets at norm
 *   percentiles (ties by ascending id), normalise each by its own maximum
 *   norm U_j, apply the SIMPLE-LSH transform P(x) = [x/U_j; sqrt(1-||x/U_j||^2)]
 *   (Eq. (8)) and hash with sign random projections (Eq. (4),
 *   PAPER:55) into bit-packed codes; precompute the sorted (U_j, l) structure
 *   of PAPER:217.
 * items      fp32 [n x d] row-major.  DEVICE pointer: BORROWED, must outlive the
 *            index (re-rank reads it).  HOST pointer: copied into an owned
 *            device buffer.  Must be finite (else NRLSH_ENONFINITE, index of the
 *            first bad item recorded).  Zero-norm items are allowed.
 * n, d       1 <= n < 2^31, 1 <= d <= 4096.
 * code_bits  SRP hash bits L_h in [1, 64] or [97, 128] (the BASELINE configs use
 *            32, 64, 128); with index_bits_in_budget, the total code length, of
 *            which L_h = code_bits - ceil(log2 m) are hash bits.  Codes are stored
 *            in 1, 2 or 4 32-bit words.
 * num_parts  m, 1 <= m <= min(n, 256) (percentile) / 256 (uniform).
 * seed       seeds the projection matrix A [(d+1) x L_h] (one A shared by all
 *            sub-datasets, reading Q4; with opt->proj = PER_PARTITION
 *            sub-dataset j uses the same generator with seed XOR j): entry e = k*L_h + b is
 *            g = sqrt(-2 ln u1) cos(2 pi u2) with u1 = ((s(2e) >> 11) + 1) 2^-53,
 *            u2 = (s(2e+1) >> 11) 2^-53, s(c) = SplitMix64 output at counter c
 *            (z = seed + (c+1)*0x9E3779B97F4A7C15, then the standard mix), rounded
 *            to fp32 and then to the nearest-even TF32 value (11 significant bits).
 * out        receives the new index (free with nrlsh_free).
 * Errors: EINVAL (sizes, bits, m > n), ENONFINITE, ENOMEM, ECUDA.
 */
nrlsh_status nrlsh_build(const float *items, int64_t n, int32_t d, int32_t code_bits,
                         int32_t num_parts, uint64_t seed, nrlsh_index **out,
                         void *cuda_stream);
nrlsh_status nrlsh_build_ex(const float *items, int64_t n, int32_t d, int32_t code_bits,
                            int32_t num_parts, uint64_t seed, const nrlsh_options *opt,
                            nrlsh_index **out, void *cuda_stream);

/*
 * nrlsh_query — query processing, Alg. 2 merged with single-table multi-probe
 * (PAPER:160-171, 207-217): query SRP code of P(q) = [q; 0]; popcount Hamming
 * scan of every item code; buckets ranked across sub-datasets by the adjusted
 * metric s_hat = U_j cos[pi (1-eps) (1 - l/L)]; the first
 * min(T, n) items of that order (ties by ascending item id) are the probed
 * candidates; they are re-ranked by exact fp32 inner product and the top k
 * returned by (score desc, id asc).
 * queries     fp32 [nq x d] (device or host); need not be unit, must be finite and
 *             non-zero (NRLSH_ENONFINITE / NRLSH_EZERONORM with the index).
 * k           >= 1.  probe_budget T >= 1 (clamped to n).
 * out_ids     int64 [nq x k] (device or host, caller-allocated); -1 padding if T < k.
 * out_scores  fp32  [nq x k]; -inf padding.
 */
nrlsh_status nrlsh_query(const nrlsh_index *index, const float *queries, int64_t nq,
                         int32_t k, int64_t probe_budget, int64_t *out_ids,
                         float *out_scores, void *cuda_stream);

/*
 * nrlsh_exact_topk — exact brute-force MIPS, Eq. (1): for every
 * query the k items of largest q^T x, (score desc, id asc), fp32 scores.  Used as
 * the ground truth for recall.  Arguments as above; items need no index.
 */
nrlsh_status nrlsh_exact_topk(const float *items, int64_t n, int32_t d,
                              const float *queries, int64_t nq, int32_t k,
                              int64_t *out_ids, float *out_scores, void *cuda_stream);

void nrlsh_free(nrlsh_index *index);
const char *nrlsh_last_error(void);

/* Index geometry: n, d, L_h (hash bits), m, words per code (ceil(L_h/32)).
   (nrlsh_get_proj gives the projection mode.) */
nrlsh_status nrlsh_get_info(const nrlsh_index *index, int64_t *n, int32_t *d,
                            int32_t *hash_bits, int32_t *num_parts, int32_t *words);

/* Projection mode of the index: NRLSH_PROJ_SHARED or NRLSH_PROJ_PER_PARTITION. */
nrlsh_status nrlsh_get_proj(const nrlsh_index *index, int32_t *proj);

/* ---- parity / test hooks (copies; pointers may be host or device) ------- */
/* norm2 fp64 [n] (item-id order), perm int32 [n] (ids grouped by sub-dataset,
   ascending id within), offsets int64 [m+1], V fp64 [m] = U_j^2. Any may be NULL. */
nrlsh_status nrlsh_get_partition(const nrlsh_index *index, double *norm2, int32_t *perm,
                                 int64_t *offsets, double *V);
/* A fp32 [(d+1) x L_h] row-major; PER_PARTITION: m such blocks, block j = A_j. */
nrlsh_status nrlsh_get_projection(const nrlsh_index *index, float *A);
/* R uint16 [m x (L_h+1)]: position of (j, h) in the sorted structure. */
nrlsh_status nrlsh_get_rank_table(const nrlsh_index *index, uint16_t *R);
/* codes uint32 [n x words], PARTITION order (row p = item perm[p]); bits >= L_h are 0. */
nrlsh_status nrlsh_get_codes(const nrlsh_index *index, uint32_t *codes);
/* overwrite the codes (same layout) — lets tests inject the oracle's codes. */
nrlsh_status nrlsh_set_codes(nrlsh_index *index, const uint32_t *codes);
/* query codes uint32 [nq x words] of P(q) = [q; 0]; PER_PARTITION: [nq x m x words],
   the code of q under each sub-index's projection A_j. */
nrlsh_status nrlsh_query_codes(const nrlsh_index *index, const float *queries, int64_t nq,
                               uint32_t *qcodes, void *cuda_stream);
/* The probed candidates of each query (a prefix of the probing order, exactly
   min(T,n) per query, in unspecified order): cand_ids int32 [nq x T'] and their
   positions in the sorted structure cand_rank uint16 [nq x T'].  qcodes may be
   NULL (computed from queries) or injected (then queries may be NULL), laid out as
   nrlsh_query_codes returns them. */
nrlsh_status nrlsh_query_candidates(const nrlsh_index *index, const float *queries,
                                    const uint32_t *qcodes, int64_t nq, int64_t probe_budget,
                                    int32_t *cand_ids, uint16_t *cand_rank, void *cuda_stream);
/* Statistics of the last nrlsh_query / nrlsh_query_candidates on this thread:
   queries that took the exact fallback (pilot bound under/overflowed), kernels
   launched, (query, item) pairs the Hamming scan actually evaluated (pairs of
   sub-datasets whose radius delta_j(q) < 0 are skipped exactly), and candidate-
   buffer entries the top-T select read (8 bytes each). Any may be NULL. */
nrlsh_status nrlsh_last_query_stats(int64_t *fallback_queries, int64_t *kernel_launches,
                                    int64_t *scanned_pairs, int64_t *buffer_entries);

/* Of the last nrlsh_query's scanned pairs on this thread (codes of >= 64 bits): the
   pairs on which the scan first evaluated a lower bound of h — the pair bound
   h >= sum over word pairs of popcount((x_a ^ q_a) | (x_b ^ q_b)) (radii delta_j(q)
   up to 16 for 64-bit codes, 37 for 128-bit codes) or, at very small radii, the
   coarser bound described under nrlsh_last_scan_popc alone — and the pairs a bound
   decided alone (a warp's 256 items all above the radius: no exact distance needed,
   the same candidates as without it).  Either may be NULL. */
nrlsh_status nrlsh_last_scan_stats(int64_t *bound_pairs, int64_t *bound_decided_pairs);

/* POPC instructions (per thread, on existing items) the popcount scan of the last
   nrlsh_query on this thread issued for distances and lower bounds: W per exact
   distance, W/2 per pair bound, and for the coarser first bound at very small radii
   one per item (128-bit codes: popcount of the OR of the four XOR words) or one per
   two items (64-bit codes: popcount((a_u | b_u) & (a_v | b_v)) <= min(h_u, h_v)).
   This is the scan's algorithmic work on the POPC roofline (PAPER:209, PAPER:217:
   the Hamming ranking of every item of every probed sub-dataset).  0 if the
   tensor-core scan ran.  May be NULL. */
nrlsh_status nrlsh_last_scan_popc(int64_t *popc_ops);

/* Candidates of the last nrlsh_query on this thread that the re-rank rescored in
   fp32 after a certified bf16 pass (the others provably could not enter the
   top-k; the answer is the same as rescoring all of them): the tensor-core
   re-rank's survivor slots; 0 for the plain gather path. */
nrlsh_status nrlsh_last_rerank_stats(int64_t *rescored_fp32);

/* Which implementation re-ranked the last nrlsh_query on this thread (all return
   the same answer: the exact fp32 top-k of the probed candidates):
     NRLSH_RERANK_GATHER       per-candidate row gather + fp32 dot (default for
                               small budgets);
     NRLSH_RERANK_TENSOR       one bf16 tcgen05 pass over the items of the
                               sub-datasets holding candidates, with a certified
                               filter (|s~ - s_f| <= eps |q||x|) against a running
                               lower bound of the k-th best candidate score,
                               keeping survivors that pass the select's candidate
                               rule, then the same fp32 re-rank of the survivors
                               (default when probe_budget >= n / 300 and a
                               sub-batch's queries x probe_budget >= 1.28 n).
   overflow_redone: queries whose tensor-core survivor list overflowed and were
   re-ranked by the gather path instead; filter_pairs: (query, item) pairs the
   tensor-core filter multiplied (0 on the other paths).  Any pointer may be NULL. */
#define NRLSH_RERANK_GATHER 0
#define NRLSH_RERANK_TENSOR 1
nrlsh_status nrlsh_last_rerank_path(int32_t *path, int64_t *overflow_redone,
                                    int64_t *filter_pairs);

/* Exact top-k (as nrlsh_exact_topk) against the index's own items (device copy
   or borrowed pointer), so host-buffer callers do not re-stage the items. */
nrlsh_status nrlsh_index_exact_topk(const nrlsh_index *index, const float *queries, int64_t nq,
                                    int32_t k, int64_t *out_ids, float *out_scores,
                                    void *cuda_stream);

/*
 * Seeded variants: seed_ids int64 [nq x seed_k] (device or host; -1, out-of-range
 * and repeated ids are ignored), 1 <= seed_k <= 1024, are ANY item ids per query
 * — typically the answers of nrlsh_query.  Their exact scores are recomputed and
 * the k-th largest certified lower bound (fl(q.x) - 1.25 (d+2) 2^-24 |q||x|) starts
 * the tensor-core filter's threshold instead of -inf.  The result is identical
 * to the unseeded call (the threshold stays a lower bound of the true k-th best
 * score); only the number of filter survivors, hence the time, changes.
 * Errors as nrlsh_exact_topk, plus EINVAL for a NULL seed_ids or a bad seed_k.
 */
nrlsh_status nrlsh_exact_topk_seeded(const float *items, int64_t n, int32_t d,
                                     const float *queries, int64_t nq, int32_t k,
                                     const int64_t *seed_ids, int32_t seed_k, int64_t *out_ids,
                                     float *out_scores, void *cuda_stream);
nrlsh_status nrlsh_index_exact_topk_seeded(const nrlsh_index *index, const float *queries,
                                           int64_t nq, int32_t k, const int64_t *seed_ids,
                                           int32_t seed_k, int64_t *out_ids, float *out_scores,
                                           void *cuda_stream);

/* Statistics of the last exact top-k on this thread: the largest and the total
   number of filter survivors per query (re-scored exactly), the number of
   queries whose survivors overflowed the buffer (answered by a full exact scan),
   and the (query, item) pairs the tensor-core filter multiplied (nq * n without
   the index's tile pruning).  Any may be NULL. */
nrlsh_status nrlsh_last_exact_stats(int64_t *max_cand, int64_t *sum_cand, int64_t *overflow,
                                    int64_t *filter_pairs);

/* ---- tracing ------------------------------------------------------------
   With profiling on, every kernel class is bracketed by CUDA events recorded on
   the stream it is launched on; elapsed times are accumulated per class at the
   entry point's final synchronisation.  Process-wide. */
void nrlsh_profile_enable(int on);
/* Fill ms[i] (total milliseconds) and counts[i] (ranges) for slot i < nslots;
   returns the number of slots; reset != 0 clears the accumulators. */
int nrlsh_profile_read(double *ms, int64_t *counts, int32_t nslots, int reset);
const char *nrlsh_profile_slot_name(int32_t slot);
/* Kernels launched by this library since it was loaded (all threads). */
int64_t nrlsh_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* NRLSH_H */
