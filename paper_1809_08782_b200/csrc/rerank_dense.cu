// rerank_dense.cu — the exact re-rank (Alg. 2 l.6) for the sub-datasets
// in which a large share of the (query, item) pairs of a batch are candidates.
//
// The probe order of PAPER:209/217 concentrates the candidates in the sub-datasets of
// largest U_j (c4, 1% budget: ~50% of the pairs of the top sub-dataset, ~18% of the
// next).  Gathering one row per (query, candidate) there re-reads the same rows for
// every query; instead a CTA stages 64 rows once in shared memory (1-D TMA bulk
// copies) and evaluates the 64 x 64 (query, row) block with register-tiled fp32 FMAs.
// Membership is decided exactly as the select does: the pair's structure position
// r = R[j][popc(code ^ qcode)] and position p are a candidate iff r < B(q), or r = B(q)
// and p <= pk(q) (B, pk from the select's bound pass).  Candidate scores feed a
// per-query running top-k in shared memory; each CTA writes its partial top-k, which
// the merge kernel combines with the gather re-rank of the other sub-datasets.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "tc_sm100.cuh"

namespace nrlsh {

constexpr int DR_Q = 64;          // queries per CTA
constexpr int DR_R = 32;          // rows per tile
constexpr int DR_THREADS = 256;   // 16 x 16 threads, 4 x 4 (query, row) outputs each

struct DenseArgs {
    const float *X;            // rows [n x ld], ld % 4 == 0 (16-byte rows)
    int ld, dq;                // row length, query length (dq <= ld; rows zero past dq)
    const float *Q;            // [Qb x dq]
    const uint32_t *qcodes;    // [Qb x W]
    const uint32_t *sel_B, *sel_pk;
    const uint32_t *codes;     // [n x W] partition order
    const int32_t *perm;
    const uint16_t *R;
    int L, W, Qb, k, cap, S;
    const int32_t *dinfo;      // [0] = #dense sub-datasets nd, [1..nd] = j, then nd+1 row prefixes
    const int64_t *offsets;    // [m+1]
    unsigned long long *partial;   // [Qb][S][k]
};

__device__ __forceinline__ unsigned long long dr_key(float sc, uint32_t id) {
    return ((unsigned long long)(~float_order(sc)) << 32) | id;
}

__device__ __forceinline__ void dr_sort_warp(unsigned long long *a, int np2) {
    const int lane = threadIdx.x & 31;
    for (int size = 2; size <= np2; size <<= 1)
        for (int st = size >> 1; st > 0; st >>= 1) {
            for (int t = lane; t < np2; t += 32) {
                const int o = t ^ st;
                if (o > t) {
                    const bool up = (t & size) == 0;
                    const unsigned long long x = a[t], y = a[o];
                    if ((x > y) == up) { a[t] = y; a[o] = x; }
                }
            }
            __syncwarp();
        }
}

// Warp w owns queries [8w, 8w + 8) of the CTA's 64: its lanes compute 2 queries x 8
// rows of each 64-row tile (lane = query pair qp = lane / 8, row group rg = lane % 8,
// rows rg + 8y), push candidates into the owned queries' buffers and compact them,
// so no CTA-wide barrier sits in the tile loop: tiles are double-buffered with a
// full (TMA bytes) and an empty (8 warp arrivals) mbarrier per stage.  Warp 0's
// lane 0 also stages the next tile (row ids, codes, the R row, the bulk copies).
__global__ void __launch_bounds__(DR_THREADS, 2) k8_rerank_dense(DenseArgs a) {
    extern __shared__ __align__(16) uint8_t dsm[];
    const int LDX = ((a.ld / 4) % 2 == 0) ? a.ld + 4 : a.ld;   // LDX/4 odd: conflict-free LDS.128
    float *Qs = reinterpret_cast<float *>(dsm);                    // [64][LDX]
    float *Xs = Qs + DR_Q * LDX;                                   // [2][64][LDX]
    unsigned long long *kb = reinterpret_cast<unsigned long long *>(Xs + 2 * DR_R * LDX);   // [64][cap]
    uint32_t *scnt = reinterpret_cast<uint32_t *>(kb + DR_Q * a.cap);   // [64]
    uint32_t *sB = scnt + DR_Q, *spk = sB + DR_Q;                  // [64] each
    uint32_t *sqc = spk + DR_Q;                                    // [64][W]
    uint32_t *sc = sqc + DR_Q * a.W;                               // [2][64][W] row codes
    int32_t *sid = reinterpret_cast<int32_t *>(sc + 2 * DR_R * a.W);   // [2][64] row ids
    int32_t *spos = sid + 2 * DR_R;                                // [2][64] row positions
    int32_t *sj = spos + 2 * DR_R;                                 // [2] tile sub-dataset, [2..3] rows
    uint16_t *sRj = reinterpret_cast<uint16_t *>(sj + 4);          // [2][L+1] R row of the tile's j
    unsigned long long *sthr = reinterpret_cast<unsigned long long *>(
        (reinterpret_cast<uintptr_t>(sRj + 2 * (a.L + 1)) + 7) & ~(uintptr_t)7);   // [64]
    uint64_t *full = reinterpret_cast<uint64_t *>(sthr + DR_Q);     // [2]
    uint64_t *empty = full + 2;                                    // [2]
    __shared__ int s_nd;
    __shared__ int s_dj[kMaxParts];
    __shared__ int s_dpre[kMaxParts + 1];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ng = (a.Qb + DR_Q - 1) / DR_Q;
    const int g = blockIdx.x % ng, split = blockIdx.x / ng;
    const int q0 = g * DR_Q;
    const int nq = min(DR_Q, a.Qb - q0);
    if (tid == 0) {
        s_nd = a.dinfo[0];
        for (int st = 0; st < 2; ++st) {
            tc::mbar_init(&full[st], 1);
            tc::mbar_init(&empty[st], DR_THREADS / 32);
        }
        tc::fence_mbar_init();
    }
    __syncthreads();
    const int nd = s_nd;
    for (int i = tid; i < nd; i += DR_THREADS) s_dj[i] = a.dinfo[1 + i];
    for (int i = tid; i <= nd; i += DR_THREADS) s_dpre[i] = a.dinfo[1 + nd + i];
    for (int e = tid; e < DR_Q * LDX; e += DR_THREADS) {
        const int r = e / LDX, c = e - r * LDX;
        Qs[e] = (r < nq && c < a.dq) ? a.Q[(int64_t)(q0 + r) * a.dq + c] : 0.f;
    }
    for (int e = tid; e < DR_Q; e += DR_THREADS) {
        scnt[e] = 0;
        sthr[e] = ~0ull;   // the query's current k-th best key (after a compaction)
        sB[e] = e < nq ? a.sel_B[q0 + e] : 0u;
        spk[e] = e < nq ? a.sel_pk[q0 + e] : 0u;
    }
    for (int e = tid; e < DR_Q * a.W; e += DR_THREADS)
        sqc[e] = (e / a.W) < nq ? a.qcodes[(int64_t)q0 * a.W + e] : 0u;
    __syncthreads();
    const int ntile = s_dpre[nd];

    // tile t: dense sub-dataset i holds tiles [pre_i, pre_{i+1}) of <= 64 rows each,
    // aligned to its own first position (a tile never spans two sub-datasets)
    auto tile_rows = [&](int t, int &j, int &p0, int &rows) {
        int i = 0;
        while (i + 1 < nd && s_dpre[i + 1] <= t) ++i;
        j = s_dj[i];
        p0 = (int)a.offsets[j] + (t - s_dpre[i]) * DR_R;
        rows = min(DR_R, (int)a.offsets[j + 1] - p0);
    };
    // (warp 0 only) stage tile t into buffer st once every warp released it
    auto stage = [&](int t, int st, int use) {
        if (use > 0) tc::mbar_wait(&empty[st], (use - 1) & 1);
        int j, p0, rows;
        tile_rows(t, j, p0, rows);
        for (int r = lane; r < DR_R; r += 32) {
            const int pos = p0 + min(r, rows - 1);
            sid[st * DR_R + r] = r < rows ? a.perm[pos] : -1;
            spos[st * DR_R + r] = p0 + r;
            for (int w = 0; w < a.W; ++w) sc[(st * DR_R + r) * a.W + w] = a.codes[(int64_t)pos * a.W + w];
        }
        for (int h = lane; h <= a.L; h += 32) sRj[st * (a.L + 1) + h] = a.R[j * (a.L + 1) + h];
        if (lane == 0) sj[st] = j;
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_expect_tx(&full[st], (uint32_t)rows * a.ld * 4);
        __syncwarp();
        // every lane issues its rows' copies (a single issuing lane serialises them)
        for (int r = lane; r < rows; r += 32)
            tc::bulk_load(Xs + (st * DR_R + r) * LDX, a.X + (int64_t)sid[st * DR_R + r] * a.ld,
                          (uint32_t)a.ld * 4, &full[st]);
        __syncwarp();
    };

    const int qp = lane >> 3, rg = lane & 7;
    const int qa = warp * 8 + 2 * qp;            // the lane's two queries: qa, qa + 1
    int it = 0;
    if (warp == 0 && split < ntile) stage(split, 0, 0);
    for (int t = split; t < ntile; t += a.S, ++it) {
        const int st = it & 1;
        if (warp == 0 && t + a.S < ntile) stage(t + a.S, st ^ 1, (it + 1) >> 1);
        tc::mbar_wait(&full[st], (it >> 1) & 1);
        float acc[2][DR_R / 8];
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
            for (int y = 0; y < DR_R / 8; ++y) acc[x][y] = 0.f;
        const float *xb = Xs + st * DR_R * LDX;
        const float *qb0 = Qs + qa * LDX, *qb1 = qb0 + LDX;
#pragma unroll 2
        for (int kk = 0; kk < a.ld; kk += 4) {
            const float4 q0v = *reinterpret_cast<const float4 *>(qb0 + kk);
            const float4 q1v = *reinterpret_cast<const float4 *>(qb1 + kk);
#pragma unroll
            for (int y = 0; y < DR_R / 8; ++y) {
                const float4 xv = *reinterpret_cast<const float4 *>(xb + (rg + 8 * y) * LDX + kk);
                acc[0][y] = fmaf(q0v.x, xv.x, acc[0][y]);
                acc[0][y] = fmaf(q0v.y, xv.y, acc[0][y]);
                acc[0][y] = fmaf(q0v.z, xv.z, acc[0][y]);
                acc[0][y] = fmaf(q0v.w, xv.w, acc[0][y]);
                acc[1][y] = fmaf(q1v.x, xv.x, acc[1][y]);
                acc[1][y] = fmaf(q1v.y, xv.y, acc[1][y]);
                acc[1][y] = fmaf(q1v.z, xv.z, acc[1][y]);
                acc[1][y] = fmaf(q1v.w, xv.w, acc[1][y]);
            }
        }
        // membership (exactly the select's rule) and the owned queries' running top-k
        const int j = sj[st];
        const uint16_t *Rj = sRj + st * (a.L + 1);
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            const int qi = qa + x;
            if (qi >= nq) continue;
            const unsigned long long thr = sthr[qi];
            const uint32_t Bq = sB[qi], pkq = spk[qi];
#pragma unroll
            for (int y = 0; y < DR_R / 8; ++y) {
                const int ri = rg + 8 * y;
                const int id = sid[st * DR_R + ri];
                if (id < 0) continue;
                const unsigned long long key = dr_key(acc[x][y], (uint32_t)id);
                if (key >= thr) continue;   // cannot enter the query's top-k
                int h = 0;
                for (int w = 0; w < a.W; ++w)
                    h += __popc(sc[(st * DR_R + ri) * a.W + w] ^ sqc[qi * a.W + w]);
                const uint32_t r = Rj[h];
                const uint32_t pos = (uint32_t)spos[st * DR_R + ri];
                if (r < Bq || (r == Bq && pos <= pkq)) {
                    const uint32_t slot = atomicAdd(&scnt[qi], 1u);
                    kb[qi * a.cap + slot] = key;
                }
            }
        }
        __syncwarp();
        // this warp is done with the tile's rows
        if (lane == 0) tc::mbar_arrive(&empty[st]);
        // compact the owned buffers that could overflow on the next tile
        for (int qi = warp * 8; qi < min(nq, warp * 8 + 8); ++qi) {
            const uint32_t c = scnt[qi];
            if (c <= (uint32_t)(a.cap - DR_R)) continue;
            unsigned long long *b = kb + qi * a.cap;
            for (int e = (int)c + lane; e < a.cap; e += 32) b[e] = ~0ull;
            __syncwarp();
            dr_sort_warp(b, a.cap);
            if (lane == 0) {
                scnt[qi] = min(c, (uint32_t)a.k);
                if (c >= (uint32_t)a.k) sthr[qi] = b[a.k - 1];
            }
            __syncwarp();
        }
    }
    // partial top-k of this CTA's queries
    for (int qi = warp * 8; qi < min(nq, warp * 8 + 8); ++qi) {
        unsigned long long *b = kb + qi * a.cap;
        const uint32_t c = scnt[qi];
        for (int e = (int)c + lane; e < a.cap; e += 32) b[e] = ~0ull;
        __syncwarp();
        dr_sort_warp(b, a.cap);
        unsigned long long *pp = a.partial + ((int64_t)(q0 + qi) * a.S + split) * a.k;
        for (int e = lane; e < a.k; e += 32) pp[e] = e < (int)c ? b[e] : ~0ull;
        __syncwarp();
    }
    for (int qi = nq + warp; qi < DR_Q && 0; qi += 8) {}
}

// dense[j] = the batch's candidate pairs in sub-dataset j reach frac of all its pairs;
// dinfo = {nd, j_1..j_nd, 64-row tile prefix 0..nd}
__global__ void dense_decide(const uint32_t *__restrict__ cnt_part, const int64_t *__restrict__ offsets,
                             int m, int Qb, float frac, uint8_t *__restrict__ dense,
                             int32_t *__restrict__ dinfo) {
    if (threadIdx.x != 0) return;
    int nd = 0;
    int32_t js[kMaxParts];
    for (int j = 0; j < m; ++j) {
        const double pairs = (double)Qb * (double)(offsets[j + 1] - offsets[j]);
        const bool dj = pairs > 0 && (double)cnt_part[j] >= (double)frac * pairs;
        dense[j] = dj;
        if (dj) js[nd++] = j;
    }
    dinfo[0] = nd;
    int pre = 0;
    for (int i = 0; i < nd; ++i) {
        dinfo[1 + i] = js[i];
        dinfo[1 + nd + i] = pre;
        pre += (int)((offsets[js[i] + 1] - offsets[js[i]] + DR_R - 1) / DR_R);
    }
    dinfo[1 + 2 * nd] = pre;
}

// final top-k of each query from S dense partial lists and the gather's top-k
__global__ void __launch_bounds__(256) dense_merge(const unsigned long long *__restrict__ partial,
                                                   int S, int k, const int64_t *__restrict__ g_ids,
                                                   const float *__restrict__ g_sc, int np2,
                                                   int64_t *__restrict__ out_ids,
                                                   float *__restrict__ out_scores) {
    extern __shared__ unsigned long long mk2[];
    const int q = blockIdx.x;
    const int tot = (S + 1) * k;
    for (int e = threadIdx.x; e < np2; e += blockDim.x) {
        unsigned long long v = ~0ull;
        if (e < S * k) v = partial[(int64_t)q * S * k + e];
        else if (e < tot) {
            const int t = e - S * k;
            const int64_t id = g_ids[(int64_t)q * k + t];
            if (id >= 0) v = dr_key(g_sc[(int64_t)q * k + t], (uint32_t)id);
        }
        mk2[e] = v;
    }
    __syncthreads();
    for (int size = 2; size <= np2; size <<= 1)
        for (int st = size >> 1; st > 0; st >>= 1) {
            for (int t = threadIdx.x; t < np2; t += blockDim.x) {
                const int o = t ^ st;
                if (o > t) {
                    const bool up = (t & size) == 0;
                    const unsigned long long x = mk2[t], y = mk2[o];
                    if ((x > y) == up) { mk2[t] = y; mk2[o] = x; }
                }
            }
            __syncthreads();
        }
    for (int t = threadIdx.x; t < k; t += blockDim.x) {
        const unsigned long long v = mk2[t];
        out_ids[(int64_t)q * k + t] = v == ~0ull ? -1 : (int64_t)(uint32_t)v;
        out_scores[(int64_t)q * k + t] = v == ~0ull ? -INFINITY : float_unorder(~(uint32_t)(v >> 32));
    }
}

static int dr_pow2(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

int dense_splits(int Qb) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int ng = (Qb + DR_Q - 1) / DR_Q;
    return std::max(1, sms / ng);
}

static size_t dense_smem(int ld, int W, int cap) {
    const int LDX = ((ld / 4) % 2 == 0) ? ld + 4 : ld;
    return (size_t)(DR_Q + 2 * DR_R) * LDX * 4 + (size_t)DR_Q * cap * 8 + 3 * DR_Q * 4 +
           (size_t)(DR_Q + 2 * DR_R) * W * 4 + 4 * DR_R * 4 + 16 + 2 * 129 * 2 + 8 +
           DR_Q * 8 + 4 * 8 + 16;
}

// Opt-in (NRLSH_DENSE=1): exact and parity-tested, but not yet faster than the gather
// on c4 (dense 1.70 ms + cold gather 1.0 ms vs gather-only 1.64 ms per 1024 queries):
// the register-tiled loop reaches ~13% of the FFMA peak (8 warps per SM, LDS->FFMA
// latency, membership epilogue).  DESIGN.md "Dense re-rank" has the numbers.
bool dense_rerank_supported(int ld, int W, int k) {
    const int cap = dr_pow2(k + DR_R + 16);
    return ld % 4 == 0 && dense_smem(ld, W, cap) <= 227 * 1024 && getenv("NRLSH_DENSE") &&
           atoi(getenv("NRLSH_DENSE")) != 0 && !getenv("NRLSH_NO_DENSE");
}

void launch_dense_decide(const uint32_t *cnt_part, const int64_t *offsets, int m, int Qb,
                         float frac, uint8_t *dense, int32_t *dinfo, cudaStream_t s) {
    dense_decide<<<1, 32, 0, s>>>(cnt_part, offsets, m, Qb, frac, dense, dinfo);
    note_launch();
}

void launch_rerank_dense(const float *X, int ld, int dq, const float *Q, const uint32_t *qcodes,
                         const uint32_t *sel_B, const uint32_t *sel_pk, const nrlsh_index *ix,
                         int Qb, int k, const int32_t *dinfo, unsigned long long *partial, int S,
                         cudaStream_t s) {
    DenseArgs a;
    a.X = X;
    a.ld = ld;
    a.dq = dq;
    a.Q = Q;
    a.qcodes = qcodes;
    a.sel_B = sel_B;
    a.sel_pk = sel_pk;
    a.codes = ix->codes;
    a.perm = ix->perm;
    a.R = ix->R_d;
    a.L = ix->L;
    a.W = ix->W;
    a.Qb = Qb;
    a.k = k;
    a.cap = dr_pow2(k + DR_R + 16);
    a.S = S;
    a.dinfo = dinfo;
    a.offsets = ix->offsets_d;
    a.partial = partial;
    const size_t sm = dense_smem(ld, ix->W, a.cap);
    cudaFuncSetAttribute(k8_rerank_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int ng = (Qb + DR_Q - 1) / DR_Q;
    k8_rerank_dense<<<ng * S, DR_THREADS, sm, s>>>(a);
    note_launch();
}

void launch_dense_merge(const unsigned long long *partial, int S, int k, const int64_t *g_ids,
                        const float *g_sc, int Qb, int64_t *out_ids, float *out_scores,
                        cudaStream_t s) {
    const int np2 = dr_pow2((S + 1) * k);
    cudaFuncSetAttribute(dense_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, np2 * 8);
    dense_merge<<<Qb, 256, (size_t)np2 * 8, s>>>(partial, S, k, g_ids, g_sc, np2, out_ids, out_scores);
    note_launch();
}

}  // namespace nrlsh
