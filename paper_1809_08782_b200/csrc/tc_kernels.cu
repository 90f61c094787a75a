// tc_kernels.cu — tcgen05 / TMEM / TMA kernels (sm_100a).
//
// gt_filter_tc: the exact-MIPS ground truth (Eq. (1)) as a
// tensor-core GEMM with a fused, certified top-k filter.  Per CTA tile the
// tensor cores compute 128 queries x 256 items (bf16 operands, fp32 accumulate
// in TMEM); epilogue warps read their query row from TMEM and keep an item iff
//      s~ + e(q,x) >= theta_q,   e(q,x) = eps_rel |q| |x|  (bf16 + fp32 error bound)
// where theta_q is a running lower bound on the true k-th best score: the k-th
// largest s~ - e(q,x) over real items seen (a per-thread min-heap), shared
// across CTAs through a global atomicMax.  Every exact top-k item survives
// (its s >= theta, and s~ >= s - e), so the survivors re-scored exactly contain
// the answer.  Warp roles: 0 TMA producer, 1 MMA issuer, 2 TMEM allocator,
// 3 |x| tile loader, 4-7 epilogue (TMEM lane group = warp % 4).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>
#include <cstdio>

#include "common.cuh"
#include "internal.h"
#include "tc_sm100.cuh"

namespace nrlsh {

// ------------------------------------------------------------ operand prep
// fp32 rows -> bf16 rows padded to dp (multiple of 8) + fp32 |row| rounded up;
// with perm, output row i is input row perm[i].
__global__ void bf16_prep(const float *__restrict__ X, int64_t n, int d, int dp,
                          __nv_bfloat16 *__restrict__ Xb, float *__restrict__ xnorm,
                          const int32_t *__restrict__ perm) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const float *src = X + (perm ? (int64_t)perm[i] : i) * (int64_t)d;
        __nv_bfloat16 *dst = Xb + i * (int64_t)dp;
        double s = 0.0;
        for (int k = lane; k < dp; k += 32) {
            const float v = k < d ? __ldg(src + k) : 0.f;
            s += (double)v * (double)v;
            dst[k] = __float2bfloat16_rn(v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(NR_FULL, s, o);
        if (lane == 0 && xnorm) xnorm[i] = __double2float_ru(sqrt(s) * (1.0 + 0x1p-50));   // upper bound
    }
}

void launch_bf16_prep(const float *X, int64_t n, int d, int dp, void *Xb, float *xnorm,
                      cudaStream_t s, const int32_t *perm) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    launch_pdl(bf16_prep, dim3(grid_for(n * 32, 256, sms * 16)), dim3(256), 0, s, X, n, d, dp, (__nv_bfloat16 *)Xb,
                                                             xnorm, perm);
    note_launch();
}

// ------------------------------------------------------------ tensor maps
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

// 2-D row-major [rows x cols] of `esize`-byte elements, box {box_cols, box_rows},
// 128-byte (default), 64-byte or (0) no swizzle
bool make_tmap_2d(CUtensorMap *m, const void *base, CUtensorMapDataType dt, int esize,
                  uint64_t cols, uint64_t rows, uint32_t box_cols, uint32_t box_rows, int swizzle) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * (uint64_t)esize};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, dt, 2, const_cast<void *>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swizzle == 0 ? CU_TENSOR_MAP_SWIZZLE_NONE
                                 : (swizzle == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B),
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}
// 1-D tensor of n elements, box of `box` elements (any start element; out of range
// reads as zero)
bool make_tmap_1d(CUtensorMap *m, const void *base, CUtensorMapDataType dt, int esize, uint64_t n,
                  uint32_t box) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    (void)esize;
    cuuint64_t dims[1] = {n};
    cuuint64_t strides[1] = {0};
    cuuint32_t bx[1] = {box};
    cuuint32_t es[1] = {1};
    CUresult r = fn(m, dt, 1, const_cast<void *>(base), dims, strides, bx, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}
static bool make_tmap(CUtensorMap *m, const void *base, CUtensorMapDataType dt, int esize,
                      uint64_t cols, uint64_t rows, uint32_t box_cols, uint32_t box_rows) {
    return make_tmap_2d(m, base, dt, esize, cols, rows, box_cols, box_rows, 128);
}

// ------------------------------------------------------------ the kernel
// CTA unit = (pair of 128-query blocks, split of the items).  The two query blocks
// stay resident in smem (A operands, K-major, 128B-swizzled); every 256-item tile
// of X (B operand) is TMA-loaded once and multiplied into two TMEM accumulators
// (one per query block, M=128 x N=256 MMAs: the N that runs the tensor core at its
// full rate), so each X byte fetched from L2 feeds 256 query rows.
// TMEM: 2 query blocks x 256 fp32 columns = all 512 columns, single-buffered: a
// block's next tile waits for its epilogue warps to drain it (an M=128 x N=128 MMA
// runs at half rate, so halving N for double buffering costs more).  Rows longer
// than 192 bf16 leave no room for a 3-deep ring of 32 KB tiles: NT = 128 there,
// double-buffered.
constexpr int GT_M = 128;          // queries per block (TMEM lanes)
constexpr int GT_QB = 2;           // query blocks per CTA
constexpr int GT_KB = 64;          // bf16 per K block (128-byte swizzled rows)
constexpr int GT_MAX_STAGES = 8;
constexpr int GT_PREFETCH = 0;        // L2 prefetch distance (tiles): measured harmful
constexpr int GT_A_BLK = GT_M * 128;   // 16 KB
constexpr int GT_THREADS = 384;        // warps 0-3 control, 4-7 epilogue of block 0, 8-11 of block 1
constexpr int GT_MAX_KBLK = 5;         // d <= 320
constexpr int GT_MAX_K = 256;

struct GtArgs {
    int64_t n;
    int Qb;
    int d;                  // real K (the MMAs of the zero K tail are skipped)
    int kblocks;
    int k;
    float eps_rel;
    const float *xnorm;
    const float *qnorm;
    uint32_t *theta_glob;   // orderable fp32 images, 0 = unset
    float *heap;            // [grid x 256 x k] per-(CTA, query row) min-heaps (rare access)
    int32_t *cand;
    uint32_t *cnt;
    int64_t C;
    int nqp;                // query-block pairs
    int nsplit;
    int64_t split_items;    // multiple of GT_N
    int stages;             // B ring depth
    int heap_smem;          // 1: heaps in shared memory, 0: global scratch
    int dbg;                // profiling experiments only (NRLSH_GT_DBG): 1 = skip the
                            // epilogue arithmetic, 2 = skip the TMEM reads too,
                            // 3 = also skip the MMAs (TMA stream only)
    int prefetch;           // item tiles prefetched into L2 ahead of the ring
    // candidate-membership mode (the tensor-core re-rank): survivors must also be
    // candidates of their query; the running bound is over candidates only
    int member;
    const uint32_t *codes;  // [npad x W] in the row order of Xb (partition order)
    const uint8_t *part;    // [npad]
    const uint16_t *R;
    int L, W;
    const uint32_t *qcodes; // [Qb x qm x W]
    int qm;                 // 1, or m (per-sub-dataset projections: q's code under A_j)
    const uint32_t *sel_B, *sel_pk;
    const int32_t *perm;    // row -> item id of the survivors (nullptr: identity)
    const int32_t *qperm;   // query row -> original query index (nullptr: identity)
    // per query-pair tile lists (member mode: only tiles of sub-datasets holding a
    // candidate of the pair's queries); nullptr: every tile
    const int32_t *tlist;   // [nqp x tstride] tile indices
    const int32_t *tcount;  // [nqp]
    int64_t tstride;
    int64_t split_tiles;    // tiles per split without lists
    int64_t ntiles;
};

// Unit (query pair qp, split sp) takes every nsplit-th tile starting at sp: rows in
// partition order sort by norm, and the high-norm tiles (where the filter keeps the
// most) spread over all splits instead of loading the last few.  v = 0..count-1
// indexes the unit's tiles; the CTAs of the other pairs of a split read the same ones.
// With tile lists the nqp * nsplit units are shared out in proportion to the pairs'
// list lengths (each pair >= 1 unit), so a pair with many tiles gets more CTAs; every
// role derives the same map from tcount.  Units past the map are idle (count 0).
__device__ __forceinline__ void gt_unit_map(const GtArgs &a, int u, int &qp, int &sp, int &ns) {
    if (!a.tlist) {
        qp = u % a.nqp;
        sp = u / a.nqp;
        ns = a.nsplit;
        return;
    }
    const int U = a.nqp * a.nsplit;
    int64_t C = 0;
    for (int g = 0; g < a.nqp; ++g) C += a.tcount[g];
    int base = 0;
    for (int g = 0; g < a.nqp; ++g) {
        const int n_g = (int)((int64_t)(U - a.nqp) * a.tcount[g] / max(C, (int64_t)1)) + 1;
        if (u < base + n_g) { qp = g; sp = u - base; ns = n_g; return; }
        base += n_g;
    }
    qp = 0; sp = 0; ns = 0;   // idle
}
__device__ __forceinline__ int64_t gt_unit_count(const GtArgs &a, int qp, int sp, int ns) {
    if (ns == 0) return 0;
    const int64_t c = a.tlist ? (int64_t)a.tcount[qp] : a.ntiles;
    return c > sp ? (c - sp + ns - 1) / ns : 0;
}
__device__ __forceinline__ int64_t gt_tile_row0(const GtArgs &a, int qp, int sp, int ns, int64_t v, int nt) {
    const int64_t e = sp + v * ns;
    return (a.tlist ? (int64_t)__ldg(a.tlist + qp * a.tstride + e) : e) * nt;
}

__device__ __forceinline__ float fmax3f(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// Tiles of a unit's item range, in order (concurrent readers of one tile — the
// CTAs of the other query pairs of the same split — share its L2 fetch; rotating
// their start tiles was measured 20% slower).
// Per-(query row, column range) epilogue state of the certified filter: the
// running bound theta (k-th best lower bound s~ - e seen, or shared / warm-started),
// the survivor list cursor and (member mode) the query's code and select bound.
struct GtEpiRow {
    const GtArgs *a;
    int q;
    bool vq;
    float qe, theta, thr_adj, pub;
    int hs;
    float *hp;
    int32_t *cl;
    uint32_t sbase, sleft;
    uint32_t qcw[4], Bq, pkq;

    __device__ __forceinline__ void set_theta(float th) {
        // the hot-loop test uses a round-to-nearest FMA; thr_adj absorbs its rounding
        // (<= 2^-24 |result| near the threshold) so the filter stays certified
        theta = th;
        thr_adj = th - fabsf(th) * 2.384185791015625e-7f;   // 2^-22
    }
    // qrow: the query's row of the (possibly bound-sorted) bf16 query matrix and of
    // qnorm; everything else is indexed by the original query index q = qperm[qrow]
    __device__ __forceinline__ void begin(const GtArgs &args, int qrow, bool vq_, float *heap_) {
        a = &args;
        vq = vq_;
        q = vq && args.qperm ? __ldg(args.qperm + qrow) : qrow;
        qe = vq ? args.eps_rel * args.qnorm[qrow] : 0.f;
        theta = -INFINITY;
        thr_adj = -INFINITY;
        pub = -INFINITY;
        hs = 0;
        hp = heap_;
        // survivors go to 16-slot chunks of the query's list reserved with one
        // atomic each; unused slots of the last chunk are filled with -1
        cl = args.cand + (int64_t)(vq ? q : 0) * args.C;
        sbase = 0;
        sleft = 0;
        qcw[0] = qcw[1] = qcw[2] = qcw[3] = 0u;
        Bq = pkq = 0u;
        if (vq) {
            const uint32_t o = args.theta_glob[q];
            if (o) set_theta(float_unorder(o));
            if (args.member) {
#pragma unroll
                for (int w = 0; w < 4; ++w)
                    if (w < args.W) qcw[w] = args.qcodes[(int64_t)q * args.qm * args.W + w];
                Bq = args.sel_B[q];
                pkq = args.sel_pk[q];
            }
        }
    }
    __device__ __forceinline__ void end() {
        // publish the final bound (a later pass over the remaining tiles starts from it)
        if (vq && hs == a->k && hp[0] > pub) atomicMax(&a->theta_glob[q], float_order(hp[0]));
        for (; sleft > 0; --sleft)
            if (sbase + (16 - sleft) < a->C) cl[sbase + (16 - sleft)] = -1;
    }
    // share the bound across CTAs (called every few tiles; o_next was loaded earlier)
    __device__ __forceinline__ void share(uint32_t o_next) {
        if (hs == a->k && hp[0] > pub) {
            pub = hp[0];
            atomicMax(&a->theta_glob[q], float_order(pub));
        }
        if (o_next) {
            const float g = float_unorder(o_next);
            if (g > theta) set_theta(g);
        }
    }
    // 64 accumulator columns [c, c+64) of the row (r0: c..c+31, r1: c+32..c+63) of the
    // tile starting at item i0; xn = the tile's |x| (rounded up), xmax = its largest
    // over the chunk's columns; scode/spart = the tile's codes / sub-datasets.
    __device__ __forceinline__ void chunk(const uint32_t (&r0)[32], const uint32_t (&r1)[32], int c,
                                          const float *xn, float xmax, int64_t i0,
                                          const uint32_t *scode, const uint8_t *spart) {
        const float thr_tile = __fmaf_rd(-xmax, qe, thr_adj);
        // cheap screen: max of the 64 approximate scores against the threshold
        // loosened by the chunk's largest error term
        float m0 = __uint_as_float(r0[0]), m1 = __uint_as_float(r1[0]);
        float m2 = __uint_as_float(r0[1]), m3 = __uint_as_float(r1[1]);
#pragma unroll
        for (int j = 2; j < 32; j += 4) {   // 3-input max (FMNMX3)
            m0 = fmax3f(m0, __uint_as_float(r0[j]), __uint_as_float(r0[j + 1]));
            m1 = fmax3f(m1, __uint_as_float(r1[j]), __uint_as_float(r1[j + 1]));
            if (j + 3 < 32) {
                m2 = fmax3f(m2, __uint_as_float(r0[j + 2]), __uint_as_float(r0[j + 3]));
                m3 = fmax3f(m3, __uint_as_float(r1[j + 2]), __uint_as_float(r1[j + 3]));
            }
        }
        if (fmax3f(fmaxf(m0, m1), m2, m3) < thr_tile) return;
        const float4 *x4 = reinterpret_cast<const float4 *>(xn + c);
        unsigned hit = 0u, hit2 = 0u;
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
            const float4 xa = x4[j4];
            const float4 xb = x4[j4 + 8];
            hit |= (fmaf(xa.x, qe, __uint_as_float(r0[4 * j4 + 0])) >= thr_adj) << (4 * j4 + 0);
            hit |= (fmaf(xa.y, qe, __uint_as_float(r0[4 * j4 + 1])) >= thr_adj) << (4 * j4 + 1);
            hit |= (fmaf(xa.z, qe, __uint_as_float(r0[4 * j4 + 2])) >= thr_adj) << (4 * j4 + 2);
            hit |= (fmaf(xa.w, qe, __uint_as_float(r0[4 * j4 + 3])) >= thr_adj) << (4 * j4 + 3);
            hit2 |= (fmaf(xb.x, qe, __uint_as_float(r1[4 * j4 + 0])) >= thr_adj) << (4 * j4 + 0);
            hit2 |= (fmaf(xb.y, qe, __uint_as_float(r1[4 * j4 + 1])) >= thr_adj) << (4 * j4 + 1);
            hit2 |= (fmaf(xb.z, qe, __uint_as_float(r1[4 * j4 + 2])) >= thr_adj) << (4 * j4 + 2);
            hit2 |= (fmaf(xb.w, qe, __uint_as_float(r1[4 * j4 + 3])) >= thr_adj) << (4 * j4 + 3);
        }
        // rare path: survivors (pushed + fed to the running top-k bound)
        for (int hh = 0; hh < 2; ++hh) {
            unsigned m = hh ? hit2 : hit;
            while (m) {
                const int j = __ffs(m) - 1;
                m &= m - 1;
                const int col = c + 32 * hh + j;
                const int64_t i = i0 + col;   // row of Xb
                if (i >= a->n) continue;
                // (member mode: the candidate test first — most hits of a re-rank are
                // not candidates of q, and it needs no score)
                if (a->member) {   // candidate of q? (the select's rule; rows are positions)
                    const uint32_t *cw = scode + col * a->W;
                    int hq = 0;
                    if (a->qm > 1) {   // the query's code under the item's sub-index A_j
                        const uint32_t *qj = a->qcodes + ((int64_t)q * a->qm + spart[col]) * a->W;
#pragma unroll
                        for (int w = 0; w < 4; ++w)
                            if (w < a->W) hq += __popc(cw[w] ^ __ldg(qj + w));
                    } else {
#pragma unroll
                        for (int w = 0; w < 4; ++w)
                            if (w < a->W) hq += __popc(cw[w] ^ qcw[w]);
                    }
                    const uint32_t r = __ldg(a->R + spart[col] * (a->L + 1) + hq);
                    if (!(r < Bq || (r == Bq && (uint32_t)i <= pkq))) continue;
                }
                float s_j = 0.f;
#pragma unroll
                for (int jj = 0; jj < 32; ++jj)
                    if (jj == j) s_j = __uint_as_float(hh ? r1[jj] : r0[jj]);
                const float x = xn[col];
                if (__fmaf_ru(x, qe, s_j) < theta) continue;   // exact re-test
                if (sleft == 0) { sbase = atomicAdd(&a->cnt[q], 16u); sleft = 16; }
                if (sbase + (16 - sleft) < a->C)
                    cl[sbase + (16 - sleft)] = a->perm ? __ldg(a->perm + i) : (int32_t)i;
                --sleft;
                const float lb = __fmaf_rd(-x, qe, s_j);
                const int k = a->k;
                if (hs < k) {            // min-heap push
                    int p = hs++;
                    while (p > 0) {
                        const int par = (p - 1) >> 1;
                        if (hp[par] <= lb) break;
                        hp[p] = hp[par];
                        p = par;
                    }
                    hp[p] = lb;
                    if (hs == k && hp[0] > theta) set_theta(hp[0]);
                } else if (lb > hp[0]) { // replace the minimum
                    int p = 0;
                    while (true) {
                        int ch = 2 * p + 1;
                        if (ch >= k) break;
                        if (ch + 1 < k && hp[ch + 1] < hp[ch]) ++ch;
                        if (hp[ch] >= lb) break;
                        hp[p] = hp[ch];
                        p = ch;
                    }
                    hp[p] = lb;
                    if (hp[0] > theta) set_theta(hp[0]);
                }
            }
        }
    }
};

// largest |x| over 128 consecutive entries (one warp, 4 per lane)
__device__ __forceinline__ float warp_max128(const float *xn, int lane) {
    const float4 xv = reinterpret_cast<const float4 *>(xn)[lane];
    float m = fmaxf(fmaxf(xv.x, xv.y), fmaxf(xv.z, xv.w));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(NR_FULL, m, o));
    return m;
}

template <int NT>
__global__ void __launch_bounds__(GT_THREADS, 1)
    gt_filter_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmX,
                 GtArgs a) {
    constexpr int GT_N = NT;                     // items per tile
    constexpr int GT_B_BLK = NT * 128;           // one K block of a tile
    constexpr int NBUF = 512 / (GT_QB * NT);     // TMEM accumulator buffers per block
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *sA = smem;                                        // QB x kblocks x 16 KB
    uint8_t *sB = sA + GT_QB * a.kblocks * GT_A_BLK;           // stages x 32 KB
    float *sxn = (float *)(sB + a.stages * GT_B_BLK);          // [2][GT_N] |x| tiles
    uint32_t *scode = (uint32_t *)(sxn + 2 * GT_N);            // [2][GT_N x W<=4] (member mode)
    uint8_t *spart = (uint8_t *)(scode + 2 * GT_N * 4);        // [2][GT_N]        (member mode)
    uint64_t *bars = (uint64_t *)(spart + 2 * GT_N);
    uint64_t *full = bars, *empty = bars + GT_MAX_STAGES;
    uint64_t *a_full = bars + 2 * GT_MAX_STAGES, *a_empty = a_full + 1;
    uint64_t *tfull = a_empty + 1, *tempty = tfull + 4;        // [NBUF][GT_QB]
    uint64_t *xfull = tempty + 4, *xempty = xfull + 2;         // per |x| tile buffer
    uint32_t *tmem_slot = (uint32_t *)(xempty + 2);
    float *sheap = reinterpret_cast<float *>(tmem_slot + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
        tc::mbar_init(a_full, 1);
        tc::mbar_init(a_empty, 1);
        for (int h = 0; h < NBUF * GT_QB; ++h) {
            tc::mbar_init(&tfull[h], 1);
            tc::mbar_init(&tempty[h], 4);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&xfull[b], 1);
            tc::mbar_init(&xempty[b], 8);
        }
        tc::fence_mbar_init();
    }
    if (warp == 2) tc::tmem_alloc(tmem_slot, 512);
    if (warp == 0 && lane == 0) { tc::tma_prefetch(&tmQ); tc::tma_prefetch(&tmX); }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();   // (the prologue above overlaps the previous kernel's tail)
    const int nunits = a.nqp * a.nsplit;

    if (warp == 0 && lane == 0) {
        // ================= TMA producer
        uint32_t g = 0, ul = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++ul) {
            int qp, sp, ns;
            gt_unit_map(a, u, qp, sp, ns);
            const int64_t v0 = 0, v1 = gt_unit_count(a, qp, sp, ns);
            // query blocks of this pair that hold any query (a block wholly past Qb
            // is neither loaded nor multiplied)
            const int nh = min(GT_QB, (a.Qb - qp * GT_QB * GT_M + GT_M - 1) / GT_M);
            if (ul > 0) tc::mbar_wait(a_empty, (ul - 1) & 1);
            tc::mbar_arrive_expect_tx(a_full, nh * a.kblocks * GT_A_BLK);
            for (int h = 0; h < nh; ++h)
                for (int kb = 0; kb < a.kblocks; ++kb)
                    tc::tma_load_2d(sA + (h * a.kblocks + kb) * GT_A_BLK, &tmQ, a_full, kb * GT_KB,
                                    (qp * GT_QB + h) * GT_M);
            for (int64_t v = v0; v < v1; ++v) {
                const int64_t i0 = gt_tile_row0(a, qp, sp, ns, v, GT_N);
                if (a.prefetch > 0 && v + a.prefetch < v1) {
                    const int64_t ip = gt_tile_row0(a, qp, sp, ns, v + a.prefetch, GT_N);
                    for (int kb = 0; kb < a.kblocks; ++kb) tc::tma_prefetch_2d(&tmX, kb * GT_KB, (int)ip);
                }
                for (int kb = 0; kb < a.kblocks; ++kb, ++g) {
                    const uint32_t s = g % a.stages, r = g / a.stages;
                    tc::mbar_wait(&empty[s], (r & 1) ^ 1);
                    tc::mbar_arrive_expect_tx(&full[s], GT_B_BLK);
                    tc::tma_load_2d(sB + s * GT_B_BLK, &tmX, &full[s], kb * GT_KB, (int)i0);
                }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer (warp-uniform loop, one elected lane issues)
        constexpr uint32_t idesc = tc::umma_idesc(1, GT_M, GT_N);
        uint32_t g = 0, t = 0, ul = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++ul) {
            int qp, sp, ns;
            gt_unit_map(a, u, qp, sp, ns);
            const int nh = min(GT_QB, (a.Qb - qp * GT_QB * GT_M + GT_M - 1) / GT_M);
            const int64_t v0 = 0, v1 = gt_unit_count(a, qp, sp, ns);
            tc::mbar_wait(a_full, ul & 1);
            tc::tc_fence_after();
            for (int64_t v = v0; v < v1; ++v, ++t) {
                const uint32_t buf = t % NBUF, tr = t / NBUF;
                for (int kb = 0; kb < a.kblocks; ++kb, ++g) {
                    const uint32_t s = g % a.stages, r = g / a.stages;
                    tc::mbar_wait(&full[s], r & 1);
                    tc::tc_fence_after();
                    const uint32_t bbase = tc::smem_u32(sB + s * GT_B_BLK);
                    const int nk = min(GT_KB / 16, (a.d - kb * GT_KB + 15) / 16);   // K = 16 per MMA
                    // (every block's barriers advance once per tile, holding queries or
                    // not, so their phases stay in step across units)
                    for (int h = 0; h < GT_QB; ++h) {
                        if (kb == 0) {   // the block's accumulator drained by its epilogue
                            tc::mbar_wait(&tempty[buf * GT_QB + h], (tr & 1) ^ 1);
                            tc::tc_fence_after();
                        }
                        if (h >= nh) continue;
                        const uint32_t abase = tc::smem_u32(sA + (h * a.kblocks + kb) * GT_A_BLK);
                        const uint32_t dt = tmem_base + (buf * GT_QB + h) * GT_N;
                        for (int kk = 0; kk < (a.dbg == 3 ? 0 : nk); ++kk)
                            tc::mma_f16_warp(dt, tc::umma_desc_sw128(abase + kk * 32),
                                             tc::umma_desc_sw128(bbase + kk * 32), idesc, (kb | kk) != 0);
                    }
                    tc::mma_commit_warp(&empty[s]);
                }
                for (int h = 0; h < GT_QB; ++h) tc::mma_commit_warp(&tfull[buf * GT_QB + h]);
            }
            tc::mma_commit_warp(a_empty);
        }
    } else if (warp == 3 && lane == 0) {
        // ================= |x| (and member-mode code / sub-dataset) tile loader: bulk
        // copies into the tile's buffer once both epilogue groups released it
        uint32_t t = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            int qp, sp, ns;
            gt_unit_map(a, u, qp, sp, ns);
            const int64_t v0 = 0, v1 = gt_unit_count(a, qp, sp, ns);
            for (int64_t v = v0; v < v1; ++v, ++t) {
                const int64_t i0 = gt_tile_row0(a, qp, sp, ns, v, GT_N);
                const uint32_t b = t & 1, tr = t >> 1;
                tc::mbar_wait(&xempty[b], (tr & 1) ^ 1);
                tc::mbar_arrive_expect_tx(&xfull[b], GT_N * 4 + (a.member ? GT_N * (a.W * 4 + 1) : 0));
                tc::bulk_load(sxn + b * GT_N, a.xnorm + i0, GT_N * 4, &xfull[b]);
                if (a.member) {   // the tile's codes and sub-datasets
                    tc::bulk_load(scode + b * GT_N * 4, a.codes + i0 * a.W, GT_N * a.W * 4, &xfull[b]);
                    tc::bulk_load(spart + b * GT_N, a.part + i0, GT_N, &xfull[b]);
                }
            }
        }
    } else if (warp >= 4) {
        // ================= epilogue: warps 4-7 drain query block 0, warps 8-11 block 1;
        // thread <-> query row (TMEM lane quadrant = warp % 4), all NT columns
        const int grp = warp & 3;
        const int h = (warp - 4) >> 2;
        const int row = grp * 32 + lane;
        uint32_t t = 0;
        GtEpiRow er;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            int qp, sp, ns;
            gt_unit_map(a, u, qp, sp, ns);
            const int nh = min(GT_QB, (a.Qb - qp * GT_QB * GT_M + GT_M - 1) / GT_M);
            const bool hact = h < nh;   // this group's block holds queries in this unit
            const int64_t v0 = 0, v1 = gt_unit_count(a, qp, sp, ns);
            const int q = (qp * GT_QB + h) * GT_M + row;
            // heap of this CTA's query row (CTAs of other item splits keep their own)
            er.begin(a, q, hact && q < a.Qb,
                     a.heap_smem ? sheap + (h * GT_M + row) * a.k
                                 : a.heap + ((int64_t)(blockIdx.x * 2 + h) * GT_M + row) * a.k);
            for (int64_t v = v0; v < v1; ++v, ++t) {
                const int64_t i0 = gt_tile_row0(a, qp, sp, ns, v, GT_N);
                const uint32_t b = t & 1;
                const float *xn = sxn + b * GT_N;
                uint32_t o_next = 0;
                const bool share = er.vq && ((t & 3) == 0);
                if (share) o_next = *((volatile uint32_t *)&a.theta_glob[er.q]);   // consumed below
                tc::mbar_wait(&xfull[b], (t >> 1) & 1);
                const uint32_t buf = t % NBUF, tr = t / NBUF;
                tc::mbar_wait(&tfull[buf * GT_QB + h], tr & 1);
                tc::tc_fence_after();
                if (hact) {
                    const uint32_t taddr = tmem_base + ((uint32_t)(grp * 32) << 16) + (buf * GT_QB + h) * GT_N;
                    // largest |x| of each 128-column part: s~ + qe |x| >= thr_adj
                    // implies s~ >= thr_adj - qe xmax
                    const float xm0 = warp_max128(xn, lane);
                    const float xm1 = GT_N == 256 ? warp_max128(xn + 128, lane) : 0.f;
#pragma unroll 1
                    for (int c = 0; c < GT_N; c += 64) {
                        if (a.dbg >= 2) break;
                        uint32_t r0[32], r1[32];
                        tc::tmem_ld_32x32b_x32(taddr + c, r0);
                        tc::tmem_ld_32x32b_x32(taddr + c + 32, r1);
                        tc::tmem_ld_wait();
                        if (!er.vq || a.dbg) continue;
                        er.chunk(r0, r1, c, xn, c < 128 ? xm0 : xm1, i0, scode + b * GT_N * 4,
                                 spart + b * GT_N);
                    }
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    tc::mbar_arrive(&tempty[buf * GT_QB + h]);
                    tc::mbar_arrive(&xempty[b]);
                }
                if (share) er.share(o_next);
            }
            er.end();
        }
    }
    __syncthreads();
    if (warp == 2) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, 512);
    }
}


static size_t gt_tc_smem_bytes(int nt, int kblocks, int stages, int heap_k) {
    return 1024 + (size_t)GT_QB * kblocks * GT_A_BLK + (size_t)stages * nt * 128 + 2 * nt * 4 +
           2 * nt * 16 + 2 * nt + (2 * GT_MAX_STAGES + 2 + 8 + 4) * 8 + 16 +
           (size_t)GT_QB * GT_M * heap_k * 4;
}

size_t gt_heap_bytes(int k) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    return (size_t)sms * 2 * GT_M * k * 4;
}

// Tile lists (rows in partition order): for query pair g, the NT-row tiles that can
// hold an answer of one of its queries.  A tile is skipped if its largest |x| is
// below tau_g = min_q theta_q / (|q| (1 + eps2)) (every row then has
// s~ + eps|q||x| <= |q||x|(1 + 2 eps) < theta_q <= the in-kernel bound, so the
// filter's screen drops it anyway; tau = 0 while some theta_q is unset), and in
// member mode if it overlaps no sub-dataset j with R[j][0] <= B_q for some q of the
// pair (j holds candidates of q only then: R[j][h] grows with h).
// (grid: x = chunks of 1024 tiles, y = query pairs; list order is arbitrary — the
// filter's splits interleave the list anyway; count[] must be zeroed beforehand)
constexpr int kTlChunk = 256;   // tiles per list-building CTA (one per thread)

__global__ void __launch_bounds__(256) gt_tile_lists(const uint16_t *__restrict__ R, int L, int m,
                                                     const uint8_t *__restrict__ part, int64_t n,
                                                     const uint32_t *__restrict__ sel_B, int Qb, int nt,
                                                     const float *__restrict__ xmax128,
                                                     const uint32_t *__restrict__ theta_glob,
                                                     const float *__restrict__ qnorm, double eps2,
                                                     float xsplit, int phase,
                                                     int32_t *__restrict__ list, int64_t stride,
                                                     int32_t *__restrict__ count,
                                                     unsigned long long *__restrict__ pairs,
                                                     const int32_t *__restrict__ qperm) {
    pdl_wait();
    __shared__ uint32_t act[257];
    __shared__ uint32_t sB[2 * GT_M];
    __shared__ float s_tau;
    __shared__ uint32_t s_found;
    const int g = blockIdx.y;
    const int q0 = g * 2 * GT_M, q1 = min(Qb, q0 + 2 * GT_M);
    // tau_g: min over the pair's queries (a thread per query; warp + smem min)
    float tq = INFINITY;
    for (int q = q0 + threadIdx.x; q < q1; q += blockDim.x) {   // q: query row
        const int qo = qperm ? qperm[q] : q;
        const uint32_t o = theta_glob[qo];
        const float th = o ? float_unorder(o) : -INFINITY;
        // rounded down in double: tau never exceeds the exact threshold
        const double t = th > 0.f ? (double)th / ((double)qnorm[q] * (1.0 + eps2) * (1.0 + 0x1p-20)) : 0.0;
        tq = fminf(tq, __double2float_rd(t));
        if (R) sB[q - q0] = sel_B[qo];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tq = fminf(tq, __shfl_xor_sync(NR_FULL, tq, o));
    if (threadIdx.x == 0) { s_tau = INFINITY; s_found = 0; }
    __syncthreads();
    if ((threadIdx.x & 31) == 0) atomicMin((int *)&s_tau, __float_as_int(fmaxf(tq, 0.f)));   // (>= 0: int order)
    if (R) {
        for (int j = threadIdx.x; j < m; j += blockDim.x) {
            const uint32_t r0 = R[j * (L + 1)];
            uint32_t on = 0;
            for (int i = 0; i < q1 - q0 && !on; ++i) on = r0 <= sB[i];
            act[j] = on;
        }
        __syncthreads();
        if (threadIdx.x == 0) {   // exclusive prefix count, act[j+1] - act[j0] = #active in [j0, j]
            uint32_t c = 0;
            for (int j = 0; j < m; ++j) { const uint32_t v = act[j]; act[j] = c; c += v; }
            act[m] = c;
        }
    }
    __syncthreads();
    const float tau = s_tau;
    const int64_t ntiles = (n + nt - 1) / nt;
    const int64_t n128 = (n + 127) / 128;
    const int lane = threadIdx.x & 31;
    for (int64_t t = (int64_t)blockIdx.x * kTlChunk + threadIdx.x; t < min(ntiles, (int64_t)(blockIdx.x + 1) * kTlChunk);
         t += blockDim.x) {
        const int64_t a0 = t * (nt / 128);
        float xm = xmax128[a0];
        if (nt == 256 && a0 + 1 < n128) xm = fmaxf(xm, xmax128[a0 + 1]);
        bool on = xm >= tau && (phase == 0 || (phase == 1) == (xm >= xsplit));
        if (R && on) {
            const int j0 = part[t * nt], j1 = part[min(n - 1, t * nt + nt - 1)];
            on = act[j1 + 1] - act[j0] > 0;
        }
        const unsigned bal = __ballot_sync(__activemask(), on);
        int base = 0;
        if (lane == __ffs(__activemask()) - 1 && bal) base = atomicAdd(&count[g], __popc(bal));
        base = __shfl_sync(__activemask(), base, __ffs(__activemask()) - 1);
        if (on) list[g * stride + base + __popc(bal & lanemask_lt())] = (int32_t)t;
        if (lane == 0) atomicAdd(&s_found, (uint32_t)__popc(bal));
    }
    __syncthreads();
    // (query, item) pairs the filter multiplies for this pair's real queries
    if (threadIdx.x == 0 && pairs && s_found)
        atomicAdd(pairs, (unsigned long long)s_found * nt * (unsigned long long)(q1 - q0));
}

// queries in descending theta_q / |q| (unset theta last): grouping queries of similar
// bound into the filter's 256-query pairs makes each pair's pruning bound (its
// minimum) tight for all but the last pair
// sort key of each query, theta_q / |q| descending (a warp per query row, all SMs;
// the key only orders the pairs, so any |q| rounding is fine), written over qperm
__global__ void __launch_bounds__(256) bound_keys(const float *__restrict__ Q, int d, int Qb,
                                                  const uint32_t *__restrict__ theta,
                                                  uint32_t *__restrict__ key_out) {
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= Qb) return;
    float ss = 0.f;
    for (int e = lane; e < d; e += 32) ss = fmaf(Q[(int64_t)i * d + e], Q[(int64_t)i * d + e], ss);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if (lane == 0) {
        const uint32_t o = theta[i];
        const float th = o ? float_unorder(o) : 0.f;
        const float kf = (th > 0.f && ss > 0.f) ? th / sqrtf(ss) : 0.f;
        key_out[i] = ~float_order(kf);
    }
}

__global__ void __launch_bounds__(1024) sort_by_bound(int Qb, int32_t *__restrict__ qperm) {
    pdl_wait();
    extern __shared__ unsigned long long keys[];
    int np2 = 2;
    while (np2 < Qb) np2 <<= 1;
    for (int i = threadIdx.x; i < np2; i += blockDim.x)
        keys[i] = i < Qb ? ((unsigned long long)(uint32_t)qperm[i] << 32) | (uint32_t)i : ~0ull;
    __syncthreads();
    if (np2 <= (int)blockDim.x) {
        // one key per thread (blockDim.x, a power of two, keys padded): the stages
        // with partner distance < 32 exchange through shuffles, the rest through smem
        const int P = blockDim.x, i = threadIdx.x;
        unsigned long long v = i < np2 ? keys[i] : ~0ull;
        __syncthreads();
        for (int size = 2; size <= P; size <<= 1)
            for (int st = size >> 1; st > 0; st >>= 1) {
                unsigned long long o;
                if (st < 32) {
                    o = __shfl_xor_sync(0xffffffffu, v, st);
                } else {
                    keys[i] = v;
                    __syncthreads();
                    o = keys[i ^ st];
                    __syncthreads();
                }
                const bool up = (i & size) == 0, lower = (i & st) == 0;
                v = (lower == up) ? (v < o ? v : o) : (v < o ? o : v);
            }
        if (i < Qb) qperm[i] = (int32_t)(uint32_t)v;
        return;
    }
    for (int size = 2; size <= np2; size <<= 1)
        for (int st = size >> 1; st > 0; st >>= 1) {
            for (int t = threadIdx.x; t < np2; t += blockDim.x) {
                const int o = t ^ st;
                if (o > t) {
                    const bool up = (t & size) == 0;
                    const unsigned long long x = keys[t], y = keys[o];
                    if ((x > y) == up) { keys[t] = y; keys[o] = x; }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < Qb; i += blockDim.x) qperm[i] = (int32_t)(uint32_t)keys[i];
}

// qperm in: uint32 keys per query; out: the queries in ascending (key, index) order
void launch_sort_keys(int Qb, int32_t *qperm, cudaStream_t s) {
    int np2 = 2;
    while (np2 < Qb) np2 <<= 1;
    launch_pdl(sort_by_bound, dim3(1), dim3(1024), (size_t)std::max(np2, 1024) * 8, s, Qb, qperm);
    note_launch();
}

void launch_sort_by_bound(const float *Q, int d, int Qb, const uint32_t *theta_glob,
                          int32_t *qperm, cudaStream_t s) {
    int np2 = 2;
    while (np2 < Qb) np2 <<= 1;
    launch_pdl(bound_keys, dim3((Qb + 7) / 8), dim3(256), 0, s, Q, d, Qb, theta_glob, reinterpret_cast<uint32_t *>(qperm));
    note_launch();
    launch_pdl(sort_by_bound, dim3(1), dim3(1024), (size_t)std::max(np2, 1024) * 8, s, Qb, qperm);
    note_launch();
}

__global__ void tile_xmax128(const float *__restrict__ xn, int64_t n, float *__restrict__ out) {
    const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t * 128 >= n) return;
    float m = 0.f;
    for (int e = lane; e < 128; e += 32) {
        const int64_t i = t * 128 + e;
        if (i < n) m = fmaxf(m, xn[i]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(NR_FULL, m, o));
    if (lane == 0) out[t] = m;
}

void launch_tile_xmax128(const float *xnorm_pos, int64_t n, float *out, cudaStream_t s) {
    const int64_t nt = (n + 127) / 128;
    tile_xmax128<<<(unsigned)((nt * 32 + 255) / 256), 256, 0, s>>>(xnorm_pos, n, out);
    note_launch();
}

size_t gt_tile_ws_bytes(int64_t n, int Qb) {
    const int64_t ng = (Qb + 2 * GT_M - 1) / (2 * GT_M);
    return (size_t)(ng * (1 + (n + 127) / 128) + 4) * 4;
}

static int gt_pick_nt(int kb) {
    if (getenv("NRLSH_GT_NT") && atoi(getenv("NRLSH_GT_NT")) == 128) return 128;
    return gt_tc_smem_bytes(256, kb, 3, 0) <= 227 * 1024 ? 256 : 128;
}

bool gt_tc_supported(int d, int k) {
    const int dp = (d + 7) / 8 * 8;
    const int kb = (dp + GT_KB - 1) / GT_KB;
    return encode_fn() != nullptr && kb <= GT_MAX_KBLK && k <= GT_MAX_K &&
           gt_tc_smem_bytes(128, kb, 3, 0) <= 227 * 1024;
}

int launch_gt_filter_tc(const void *Xb, int64_t n, int d, int dp, const void *Qb16, int Qb,
                        const float *xnorm, const float *qnorm, float eps_rel, int k,
                        uint32_t *theta_glob, float *heap, int32_t *cand, uint32_t *cnt, int64_t C,
                        cudaStream_t s, const int32_t *perm, const GtMember *mb,
                        const GtTiles *tl) {
    const int kblocks = (dp + GT_KB - 1) / GT_KB;
    const int NT = gt_pick_nt(kblocks);
    CUtensorMap tq, tx;
    if (!make_tmap(&tq, Qb16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dp, Qb, GT_KB, GT_M) ||
        !make_tmap(&tx, Xb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dp, n, GT_KB, NT))
        return -1;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    GtArgs a;

    a.n = n;
    a.Qb = Qb;
    a.d = d;
    a.kblocks = kblocks;
    a.k = k;
    a.eps_rel = eps_rel;
    a.xnorm = xnorm;
    a.qnorm = qnorm;
    a.theta_glob = theta_glob;
    a.heap = heap;
    a.cand = cand;
    a.cnt = cnt;
    a.C = C;
    a.dbg = getenv("NRLSH_GT_DBG") ? atoi(getenv("NRLSH_GT_DBG")) : 0;
    a.prefetch = getenv("NRLSH_GT_PREFETCH") ? atoi(getenv("NRLSH_GT_PREFETCH")) : GT_PREFETCH;
    a.member = mb != nullptr;
    a.codes = mb ? mb->codes : nullptr;
    a.part = mb ? mb->part : nullptr;
    a.R = mb ? mb->R : nullptr;
    a.perm = perm;
    a.qperm = tl ? tl->qperm : nullptr;
    a.tlist = nullptr;
    a.tcount = nullptr;
    a.tstride = 0;
    a.L = mb ? mb->L : 0;
    a.W = mb ? mb->W : 1;
    a.qcodes = mb ? mb->qcodes : nullptr;
    a.qm = mb ? mb->qm : 1;
    a.sel_B = mb ? mb->sel_B : nullptr;
    a.sel_pk = mb ? mb->sel_pk : nullptr;
    if (mb && (mb->W < 1 || mb->W > 4)) return -1;
    a.nqp = (Qb + GT_QB * GT_M - 1) / (GT_QB * GT_M);
    const int64_t ntiles = (n + NT - 1) / NT;
    int nsplit = std::max(1, sms / a.nqp);     // one unit per CTA: no tail wave
    nsplit = (int)std::min<int64_t>(nsplit, ntiles);
    a.split_tiles = (ntiles + nsplit - 1) / nsplit;
    a.split_items = a.split_tiles * NT;
    a.nsplit = (int)((n + a.split_items - 1) / a.split_items);
    a.ntiles = ntiles;
    const bool lists = tl && tl->ws && !getenv("NRLSH_GT_ALLTILES");
    // two passes when the rows are norm-sorted tiles: the tiles of largest |x| first
    // (their scores lift theta close to its final value), then the rest, pruned
    // against the lifted theta
    const bool two = lists && tl->xsplit > 0.f && !getenv("NRLSH_GT_ONEPASS");
    // tl->pass: 0 = both passes here, 1 / 2 = only that pass (the caller re-ranks the
    // first pass's survivors in between, lifting theta to an exact k-th best)
    const int p_lo = two ? (tl->pass == 2 ? 1 : 0) : 0;
    const int p_hi = two ? (tl->pass == 1 ? 1 : 2) : 1;
    if (!two && tl && tl->pass == 2) return 0;   // single pass already done
    if (lists) {
        a.tcount = tl->ws;
        a.tstride = ntiles;
        a.tlist = tl->ws + a.nqp + 4;
        a.nsplit = nsplit;
    }
    // deepest ring that fits, with the heaps in smem if they fit too
    const int smax = NT == 256 ? 6 : GT_MAX_STAGES;
    a.stages = 3;
    a.heap_smem = 0;
    for (int st = smax; st >= 3; --st)
        if (gt_tc_smem_bytes(NT, kblocks, st, k) <= 227 * 1024) { a.stages = st; a.heap_smem = 1; break; }
    if (!a.heap_smem || (NT == 128 && a.stages < 6))
        for (int st = smax; st > (a.heap_smem ? a.stages : 2); --st)
            if (gt_tc_smem_bytes(NT, kblocks, st, 0) <= 227 * 1024) { a.stages = st; a.heap_smem = 0; break; }
    if (getenv("NRLSH_GT_STAGES")) {   // experiments: force a ring depth (heaps to global)
        a.stages = std::max(2, std::min(smax, atoi(getenv("NRLSH_GT_STAGES"))));
        a.heap_smem = gt_tc_smem_bytes(NT, kblocks, a.stages, k) <= 227 * 1024;
        if (gt_tc_smem_bytes(NT, kblocks, a.stages, 0) > 227 * 1024) return -1;
    }
    const size_t sm = gt_tc_smem_bytes(NT, kblocks, a.stages, a.heap_smem ? k : 0);
    const int grid = std::min(sms, a.nqp * a.nsplit);
    for (int pass = p_lo; pass < p_hi; ++pass) {
        if (lists) {   // per query pair, only the tiles that can hold an answer (GtTiles)
            cudaMemsetAsync(const_cast<int32_t *>(a.tcount), 0, (size_t)a.nqp * 4, s);
            launch_pdl(gt_tile_lists, dim3(dim3((unsigned)((ntiles + kTlChunk - 1) / kTlChunk), a.nqp)), dim3(256), 0, s, mb ? mb->R : nullptr, mb ? mb->L : 0, mb ? mb->m : 0,
                                                mb ? mb->part : nullptr, n, mb ? mb->sel_B : nullptr,
                                                Qb, NT, tl->xmax128, theta_glob, qnorm, 2.0 * eps_rel,
                                                tl->xsplit, two ? pass + 1 : 0,
                                                const_cast<int32_t *>(a.tlist), a.tstride,
                                                const_cast<int32_t *>(a.tcount), tl->pairs, a.qperm);
            note_launch();
        }
        if (lists && getenv("NRLSH_GT_TILESTATS")) {   // development: tiles kept per pair
            std::vector<int32_t> hc(a.nqp);
            cudaMemcpyAsync(hc.data(), a.tcount, (size_t)a.nqp * 4, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            fprintf(stderr, "gt tiles (%s, pass %d, of %lld):", mb ? "member" : "gt", pass,
                    (long long)ntiles);
            for (int g = 0; g < a.nqp; ++g) fprintf(stderr, " %d", hc[g]);
            fprintf(stderr, "\n");
        }
        if (NT == 256) {
            cudaFuncSetAttribute(gt_filter_tc<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            launch_pdl(gt_filter_tc<256>, dim3(grid), dim3(GT_THREADS), sm, s, tq, tx, a);
        } else {
            cudaFuncSetAttribute(gt_filter_tc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            launch_pdl(gt_filter_tc<128>, dim3(grid), dim3(GT_THREADS), sm, s, tq, tx, a);
        }
        note_launch();
    }
    return 0;
}

}  // namespace nrlsh
