// internal.h — host-side structures and kernel launchers of libnrlsh.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/nrlsh.h"

struct nrlsh_index {
    int64_t n = 0;
    int32_t d = 0;
    int32_t L = 0;        // SRP hash bits L_h
    int32_t W = 0;        // 32-bit words per code = ceil(L/32)
    int32_t m = 0;        // sub-datasets
    int32_t code_bits = 0;
    uint64_t seed = 0;
    double eps = 0.01;
    int32_t scheme = NRLSH_SCHEME_PERCENTILE;
    int32_t proj = NRLSH_PROJ_SHARED;
    int32_t QM = 1;             // query codes per query: 1 (shared A) or m (per-sub-dataset A_j)
    int32_t query_batch = 1024;
    int device = 0;

    const float *X = nullptr;   // items, device, borrowed unless X_owned
    float *X_owned = nullptr;
    float *Xpad = nullptr;      // fp32 rows [n x dpad], dpad = d rounded up to 4 (16-byte rows),
    int32_t dpad = 0;           //   only when d % 4 != 0: the re-rank's gather source
    void *Xb = nullptr;         // bf16 rows [n x dpb], dpb = d rounded up to 8 (16-byte rows),
    int32_t dpb = 0;            //   PARTITION order: the tensor-core filter's B operand
    float *xnorm = nullptr;     // [n rounded up to 256] |x| rounded up (0 past n), item order
    float *xnorm_pos = nullptr; // the same in partition order (the filter's |x| tiles)
    float *tile_xmax = nullptr; // [ceil(n/128)] largest xnorm_pos of each 128-row tile
    float tile_xsplit = 0.f;    // xmax above which ~2% of those tiles lie (first filter pass)

    double *norm2 = nullptr;      // [n] item order
    int32_t *perm = nullptr;      // [n] position -> id
    int32_t *pos_of_id = nullptr; // [n] id -> position
    uint8_t *part_of_id = nullptr;  // [n rounded up to 256] (0 past n)
    uint8_t *part_of_pos = nullptr; // [n rounded up to 256] (0 past n)
    int64_t *offsets_d = nullptr;   // [m+1]
    double *V_d = nullptr;          // [m]
    uint32_t *codes = nullptr;      // [n x W], partition order
    int8_t *codes_pm = nullptr;     // [n x scan_kp(L)] +-1 int8 code rows, partition order
                                    //   (the opt-in tensor-core scan's B operand)
    float *A = nullptr;             // [QM x (d+1) x L] row-major (as generated; block j = A_j)
    float *Apad = nullptr;          // [QM x (d+1) x 32W], zero columns >= L
    int4 *ctiles_d = nullptr;       // per-sub-dataset projections: code-kernel tiles
    int32_t nctiles = 0;            //   (j, p0, p1): <= 128 positions of one sub-dataset
    uint16_t *R_d = nullptr;        // [m x (L+1)]
    int4 *chunks_d = nullptr;       // scan work units (j, pos0, pos1, 0)
    int32_t *order_d = nullptr;     // [m*(L+1)] structure position -> j*(L+1)+h
    int32_t nchunks = 0;
    uint32_t *samp_codes = nullptr; // pilot sample: codes of positions t * stride (compacted)
    uint8_t *samp_part = nullptr;
    int64_t nsamp = 0;

    std::vector<int64_t> offsets;
    std::vector<double> V, U;
    std::vector<float> A_h;
    std::vector<uint16_t> R_h;
};

namespace nrlsh {

// stream-ordered device allocation from the library's private per-device pool
cudaError_t dmalloc(void **p, size_t bytes, cudaStream_t s);

// ---------------------------------------------------------------- tracing
enum ProfSlot { SLOT_NORMS = 0, SLOT_PARTITION, SLOT_SCATTER, SLOT_CODES, SLOT_QCODES,
                SLOT_PILOT, SLOT_SCAN, SLOT_FALLBACK, SLOT_SELECT, SLOT_SCORE, SLOT_TOPK,
                SLOT_GT_NORMS, SLOT_GT_FILTER, SLOT_RERANK, SLOT_RERANK_TOPK, SLOT_OTHER,
                kNumSlots };
void note_launch(int k = 1);
long long launch_count();
void prof_collect();
// CUDA-event range on stream s around the kernels launched in its scope
struct ProfScope {
    ProfScope(int slot, cudaStream_t s);
    ~ProfScope();
    int slot_;
    cudaStream_t s_;
    void *a_;
};

// ---------------------------------------------------------------- build
// (Xb != nullptr: also writes bf16 rows [n x dpb] (zero-padded) and |x| rounded up)
// (returns true when it also wrote the keys' min / max bits into mm)
bool launch_norms(const float *X, int64_t n, int d, double *norm2, unsigned long long *bad,
                  void *Xb, int dpb, float *xnorm, cudaStream_t s, unsigned long long *mm = nullptr);
// K2 (percentile): fills part_of_id.  Host-orchestrated; may synchronise `s`.
int partition_percentile(const double *norm2, int64_t n, int m, uint8_t *part_of_id,
                         cudaStream_t s, std::string *err);
// level 0 + in-smem group sorts, decided on the device (no host sync); sets *large
// (device flag) when a boundary group exceeds the in-smem sort: then run the above
// mm: the keys' (smallest positive, largest) bits if the norms pass computed them
// (nullptr: computed here)
int partition_percentile_fast(const double *norm2, int64_t n, int m, uint8_t *part_of_id,
                              unsigned int *large, cudaStream_t s, std::string *err,
                              const unsigned long long *mm = nullptr);
// largest-|x| threshold of the filter's first pass: the r-th smallest of nt tile
// maxima (non-negative floats), radix-selected by one CTA into *out
void launch_select_kth_float(const float *v, int64_t nt, int64_t r, float *out, cudaStream_t s);
int partition_uniform(const double *norm2, int64_t n, int m, uint8_t *part_of_id,
                      cudaStream_t s, std::string *err);
// stable scatter by sub-dataset: perm, pos_of_id, part_of_pos, offsets, V
int partition_scatter(const double *norm2, const uint8_t *part_of_id, int64_t n, int m,
                      int32_t *perm, int32_t *pos_of_id, uint8_t *part_of_pos,
                      int64_t *offsets_d, double *V_d, cudaStream_t s, std::string *err);
// K3: SRP codes of P(x) in partition order
// (Xb != nullptr: also writes the bf16 rows [n x dpb]; xnorm is only touched by the
//  SIMT fallback, the norms pass writes it otherwise)
void launch_item_codes(const float *X, int64_t n, int d, const double *norm2,
                       const uint8_t *part_of_id, const double *V_d, const float *Apad,
                       int L, int W, const int32_t *pos_of_id, uint32_t *codes, void *Xb,
                       int dpb, float *xnorm, float *Xpad, int dpad, cudaStream_t s,
                       const int32_t *perm, int m);

// K3 on tcgen05 (codes_tc.cu); the SIMT kernel above covers the other shapes
bool codes_tc_supported(int d, int W);
// (ctiles != nullptr: per-sub-dataset projections — items are processed in partition
//  order, tile t = (j, p0, p1) uses A_j = Apad + j (d+1) 32W; perm maps positions to ids)
void launch_item_codes_tc(const float *X, int64_t n, int d, const double *norm2,
                          const uint8_t *part_of_id, const double *V_d, const float *Apad,
                          int L, int W, const int32_t *pos_of_id, uint32_t *codes, void *Xb,
                          int dpb, float *Xpad, int dpad, cudaStream_t s,
                          const int4 *ctiles = nullptr, int nctiles = 0,
                          const int32_t *perm = nullptr, int m = 0);

// ---------------------------------------------------------------- query

// qcodes [nq x QM x W]: QM = 1 (Apad = A) or m (Apad = [m x (d+1) x 32W], code j under A_j)
void launch_qcodes(const float *Q, int64_t nq, int d, const float *Apad, int L, int W,
                   uint32_t *qcodes, int *flags, int64_t q_index_base, cudaStream_t s,
                   int QM = 1);
int pilot_stride(int64_t n);
void launch_gather_sample(const nrlsh_index *ix, int stride, uint32_t *sc, uint8_t *sp,
                          cudaStream_t s);
// zero_word (nullable): zeroed by the pilot (the fallback's counter, fallback_counter())
void launch_pilot(const nrlsh_index *ix, const uint32_t *qcodes, int Qb, int64_t Tq,
                  int stride, int8_t *delta, uint32_t *cnt, cudaStream_t s, uint32_t *zero_word = nullptr);
// lbc (nullable): [0] pairs the one-POPC lower bound ran on, [1] pairs it decided alone
// units_ws: scan_units_ws_bytes() of scratch whose first 16 bytes are zero (the unit
// list of the sub-batch and its counters; the scan leaves them zero again)
size_t scan_units_ws_bytes(const nrlsh_index *ix, int Qmax);
void launch_scan(const nrlsh_index *ix, const uint32_t *qcodes, const int8_t *delta, int Qb,
                 unsigned long long *buf, uint32_t *cnt, int64_t C,
                 unsigned long long *pairs, cudaStream_t s, unsigned long long *lbc,
                 void *units_ws);
// cntv: the real entries of each query's buffer (the tensor-core scan pads its append
// runs with ~0 sentinels, counted in cnt); == cnt for the popcount scan
// ws: fallback_ws_bytes() of zeroed scratch for the all-SM re-do of failed queries
// (nullptr: one CTA per failed query only)
size_t fallback_ws_bytes(const nrlsh_index *ix);
uint32_t *fallback_counter(const nrlsh_index *ix, void *ws);
void launch_fallback(const nrlsh_index *ix, const uint32_t *qcodes, int Qb, int64_t Tq,
                     unsigned long long *buf, uint32_t *cnt, uint32_t *cntv, int64_t C,
                     int *flags, void *ws, cudaStream_t s);
// tensor-core Hamming scan (scan_tc.cu, NEXT-3, opt-in NRLSH_SCAN_TC=1): +-1 int8 item
// codes expanded at build
int scan_kp(int L);
void launch_expand_pm(const uint32_t *codes, int64_t rows, int W, int L, int8_t *out, cudaStream_t s);
bool scan_tc_supported(const nrlsh_index *ix);
size_t scan_tc_ws_bytes(const nrlsh_index *ix, int Qb);
int64_t scan_tc_slack(int Qmax);   // buffer slots per query the tensor-core scan may fill with sentinels
int launch_scan_tc(const nrlsh_index *ix, const uint32_t *qcodes, const int8_t *delta, int Qb,
                   void *ws, unsigned long long *buf, uint32_t *cnt, uint32_t *cntv, int64_t C,
                   unsigned long long *pairs, cudaStream_t s);
void launch_select(const nrlsh_index *ix, int Qb, int64_t Tq, const unsigned long long *buf,
                   const uint32_t *cnt, int64_t C, int32_t *cand, uint16_t *cand_rank,
                   cudaStream_t s);
// scores[q][t] = q . X[cand[q][t]] (fp32); if lb_eps > 0 writes fl(s) - lb_eps*|q|*|x|
// (a certified lower bound, for the ground-truth pilot).  cand == nullptr means the
// implicit list cand[q][t] = t * stride.
void launch_score(const float *X, int d, const float *Q, int Qb, const int32_t *cand,
                  int64_t ncand, int64_t cand_ld, const uint32_t *ncand_per_q, int stride,
                  const float *xnorm, const float *qnorm, float lb_eps, float *scores,
                  cudaStream_t s);
// top-k by (score desc, id asc) over scores[q][0..ncand_q)
void launch_topk(const float *scores, const int32_t *cand, int Qb, int64_t ncand,
                 int64_t cand_ld, const uint32_t *ncand_per_q, int stride, int k,
                 int64_t *out_ids, float *out_scores, float *kth_out, cudaStream_t s);

// fused exact re-rank + top-k (score desc, id asc) over cand[q][0..ncand_q); cand ==
// nullptr means cand[q][t] = t * stride.  `partial` needs rerank_partial_bytes().
size_t rerank_partial_bytes(int Qb, int64_t ncand, int k);
// X rows at stride ldx >= d (zeros past d).
void launch_rerank(const float *X, int d, int ldx, const float *Q, int Qb, const int32_t *cand,
                   int64_t ncand, int64_t cand_ld, const uint32_t *ncand_per_q, int stride,
                   int k, unsigned long long *partial, int64_t *out_ids, float *out_scores,
                   cudaStream_t s);


// row gather (dst row r = src row idx[r]) or scatter (dst row idx[r] = src row r);
// row_bytes a multiple of 4
void launch_move_rows(const void *src, const int64_t *idx, int nrows, size_t row_bytes, void *dst,
                      bool scatter, cudaStream_t s);
// dst[p] = src[idx[p]] for p < n
void launch_gather_f32(const float *src, const int32_t *idx, int64_t n, float *dst, cudaStream_t s);
// theta_glob[q] = max(theta_glob[q], orderable image of out_scores[q][k-1]) when that
// slot holds an item
void launch_restart_from_topk(const int64_t *ids, int Qb, int k, int32_t *cand, int64_t C,
                              uint32_t *cnt, cudaStream_t s);
// theta_glob[q] := (assign ? : max with) the order key of the k-th score (0 if none);
// zero_cnt, if given, is zeroed per query on the way (saves a memset node)
void launch_theta_from_topk(const int64_t *ids, const float *scores, int Qb, int k,
                            uint32_t *theta_glob, cudaStream_t s, bool assign = false,
                            uint32_t *zero_cnt = nullptr);
// *out += sum_q min(cnt[q], C)
void launch_sum_counts(const uint32_t *cnt, int Qb, int64_t C, unsigned long long *out,
                       cudaStream_t s);
// out[0] = max(out[0], max_q cnt[q]); out[1] += sum_q cnt[q]
void launch_count_stats(const uint32_t *cnt, int Qb, unsigned long long *out, cudaStream_t s);
// appends q0 + q to list (count at *n) for every q with cnt[q] > C
void launch_collect_overflow(const uint32_t *cnt, int Qb, int64_t C, int64_t q0, int64_t *list,
                             uint32_t *n, cudaStream_t s);
// select bound pass that also picks `ks` seed members per query: members in the
// best-ranked structure positions (int32 ids, -1 padded)
void launch_select_seeds(const nrlsh_index *ix, int Qb, int64_t Tq, const unsigned long long *buf,
                         const uint32_t *cnt, int64_t C, uint32_t *sel_B, uint32_t *sel_pk,
                         int32_t *seeds, int ks, cudaStream_t s);

// ---------------------------------------------------------------- ground truth
void launch_vec_norms(const float *X, int64_t n, int d, float *xnorm, cudaStream_t s);
void launch_gt_filter(const float *X, int64_t n, int d, const float *Q, int Qb,
                      const float *xnorm, const float *qnorm, const float *lb, float eps_rel,
                      int32_t *cand, uint32_t *cnt, int64_t C, cudaStream_t s);
int scan_chunk_items();
void launch_gt_seed_theta(const float *X, int64_t n, int d, const float *Q, int Qb,
                          const float *qnorm, const int64_t *seeds, int ks, int k, float eps_rel,
                          uint32_t *theta_glob, cudaStream_t s, uint32_t *zero_cnt = nullptr);
// tensor-core ground truth (tc_kernels.cu)
void launch_bf16_prep(const float *X, int64_t n, int d, int dp, void *Xb, float *xnorm,
                      cudaStream_t s, const int32_t *perm = nullptr);
bool gt_tc_supported(int d, int k);
size_t gt_heap_bytes(int k);
// Candidate membership for the tensor-core re-rank (the select's rule): item i is a
// candidate of query q iff r = R[part(i)][h(q,i)] < B_q or (r == B_q and pos(i) <= pk_q)
// (Xb rows are partition positions here; only the tiles of sub-datasets holding a
// candidate of a query pair are streamed for it)
struct GtMember {
    const uint32_t *codes;      // [npad x W] partition order
    const uint8_t *part;        // [npad] sub-dataset of each position
    const int64_t *offsets;     // [m+1] (device)
    int m;
    const uint16_t *R;          // [m x (L+1)]
    int L, W;
    const uint32_t *qcodes;     // [Qb x QM x W]
    int qm;                     // QM: 1, or m (a query's code under each A_j)
    const uint32_t *sel_B, *sel_pk;   // [Qb]
};
// Tile pruning for rows in partition order (the index's Xb): per query pair, only
// the NT-row tiles that can hold an answer are streamed — not the tiles whose
// largest |x| keeps |q||x| (1 + 2 eps) below every query's starting bound theta_q
// (Cauchy-Schwarz: such rows fail the filter's screen at that bound), and, in
// member mode, not the tiles of sub-datasets without a candidate of the pair.
struct GtTiles {
    const float *xmax128;       // [ceil(n/128)] largest |x| (rounded up) per 128-row tile
    int32_t *ws;                // gt_tile_ws_bytes(n, Qb) of scratch for the lists
    unsigned long long *pairs;  // optional: += (query, row) pairs multiplied
    float xsplit;               // > 0: two passes, tiles with xmax >= xsplit first
    int pass;                   // 0: both passes; 1 / 2: only that one
    const int32_t *qperm;       // optional: row r of the bf16 queries / qnorm is query
                                //   qperm[r] (queries sorted by theta/|q|: pairs of similar
                                //   bound prune alike); theta, lists and member data stay
                                //   in query order
};
// qperm[0..Qb) = the queries in descending theta_q / |q| (theta_glob orderable
// images, 0 = unset); one CTA, Qb <= 4096
void launch_sort_by_bound(const float *Q, int d, int Qb, const uint32_t *theta_glob,
                          int32_t *qperm, cudaStream_t s);
size_t gt_tile_ws_bytes(int64_t n, int Qb);
// qperm in: uint32 keys per query; out: queries in ascending (key, index) order (Qb <= 4096)
void launch_sort_keys(int Qb, int32_t *qperm, cudaStream_t s);
void launch_tile_xmax128(const float *xnorm_pos, int64_t n, float *out, cudaStream_t s);
// Xb / xnorm rows in any order: perm[row] = item id written to the survivor lists
// (nullptr: rows are ids)
int launch_gt_filter_tc(const void *Xb, int64_t n, int d, int dp, const void *Qb16, int Qb,
                        const float *xnorm, const float *qnorm, float eps_rel, int k,
                        uint32_t *theta_glob, float *heap, int32_t *cand, uint32_t *cnt,
                        int64_t C, cudaStream_t s, const int32_t *perm = nullptr,
                        const GtMember *member = nullptr, const GtTiles *tiles = nullptr);

}  // namespace nrlsh
