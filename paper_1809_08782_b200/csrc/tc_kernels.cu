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

#include "common.cuh"
#include "internal.h"
#include "tc_sm100.cuh"

namespace nrlsh {

// ------------------------------------------------------------ operand prep
// fp32 rows -> bf16 rows padded to dp (multiple of 8) + fp32 |row| rounded up.
__global__ void bf16_prep(const float *__restrict__ X, int64_t n, int d, int dp,
                          __nv_bfloat16 *__restrict__ Xb, float *__restrict__ xnorm) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const float *src = X + i * (int64_t)d;
        __nv_bfloat16 *dst = Xb + i * (int64_t)dp;
        double s = 0.0;
        for (int k = lane; k < dp; k += 32) {
            const float v = k < d ? __ldg(src + k) : 0.f;
            s += (double)v * (double)v;
            dst[k] = __float2bfloat16_rn(v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(NR_FULL, s, o);
        if (lane == 0) xnorm[i] = __double2float_ru(sqrt(s) * (1.0 + 0x1p-50));   // upper bound
    }
}

void launch_bf16_prep(const float *X, int64_t n, int d, int dp, void *Xb, float *xnorm,
                      cudaStream_t s) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    bf16_prep<<<grid_for(n * 32, 256, sms * 16), 256, 0, s>>>(X, n, d, dp, (__nv_bfloat16 *)Xb,
                                                             xnorm);
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

// 2-D row-major [rows x cols] of `esize`-byte elements, box {64 B*2 ... } with 128B swizzle
static bool make_tmap(CUtensorMap *m, const void *base, CUtensorMapDataType dt, int esize,
                      uint64_t cols, uint64_t rows, uint32_t box_cols, uint32_t box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * (uint64_t)esize};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, dt, 2, const_cast<void *>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// ------------------------------------------------------------ the kernel
// CTA unit = (pair of 128-query blocks, split of the items).  The two query blocks
// stay resident in smem (A operands, K-major, 128B-swizzled); every 128-item tile
// of X (B operand) is TMA-loaded once and multiplied into two TMEM accumulators
// (one per query block), so each X byte fetched from L2 feeds 256 query rows.
// TMEM: 2 buffers x 2 query blocks x 128 fp32 columns = 512 columns.
constexpr int GT_M = 128;          // queries per block (TMEM lanes)
constexpr int GT_QB = 2;           // query blocks per CTA (1 or 2)
constexpr int GT_N = 128;          // items per tile (fp32 TMEM columns per accumulator)
constexpr int GT_EPI_SUB = 2 / GT_QB;   // epilogue warps per TMEM lane quadrant and query block
constexpr int GT_EPI_COLS = GT_N / GT_EPI_SUB;
static_assert(GT_EPI_COLS == 128, "epilogue thread = one 128-column slice of a query row");
constexpr int GT_KB = 64;          // bf16 per K block (128-byte swizzled rows)
constexpr int GT_MAX_STAGES = 8;
constexpr int GT_PREFETCH = 6;        // item tiles prefetched into L2 ahead of the ring
constexpr int GT_A_BLK = GT_M * 128;   // 16 KB
constexpr int GT_B_BLK = GT_N * 128;   // 16 KB
constexpr int GT_THREADS = 384;        // warps 0-3 control, 4-11 epilogue
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
    int stages;             // B ring depth (3 or 4)
    int heap_smem;          // 1: heaps in shared memory, 0: global scratch
    int dbg;                // profiling experiments only (NRLSH_GT_DBG): 1 = skip the
                            // epilogue arithmetic, 2 = skip the TMEM reads too,
                            // 3 = also skip the MMAs (TMA stream only)
};

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}


// Tiles of a unit's item range in a rotated order: the CTAs of the different query
// blocks that share an item split start at different tiles, so they do not all
// request the same L2 lines at the same time.
__device__ __forceinline__ int64_t gt_tile_at(int64_t ib, int64_t ie, int qp, int nqp, int64_t jt) {
    const int64_t nt = (ie - ib + GT_N - 1) / GT_N;
    const int64_t rot = 0;   // measured: concurrent readers of one tile share its L2
                             // fetch; rotating the start (nt * qp / nqp) was 20% slower
    int64_t j = jt + rot;
    if (j >= nt) j -= nt;
    return ib + j * GT_N;
}

__global__ void __launch_bounds__(GT_THREADS, 1)
    gt_filter_tc(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmX,
                 GtArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *sA = smem;                                        // QB x kblocks x 16 KB
    uint8_t *sB = sA + GT_QB * a.kblocks * GT_A_BLK;           // stages x 16 KB
    float *sxn = (float *)(sB + a.stages * GT_B_BLK);          // [2][GT_N]
    uint64_t *bars = (uint64_t *)(sxn + 2 * GT_N);
    uint64_t *full = bars, *empty = bars + GT_MAX_STAGES;
    uint64_t *a_full = bars + 2 * GT_MAX_STAGES, *a_empty = a_full + 1;
    uint64_t *tfull = a_empty + 1, *tempty = tfull + 2;
    uint64_t *xfull = tempty + 2;                              // xnorm tile landed
    uint32_t *tmem_slot = (uint32_t *)(xfull + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
        tc::mbar_init(a_full, 1);
        tc::mbar_init(a_empty, 1);
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&tfull[s], 1);
            tc::mbar_init(&tempty[s], 8);
            tc::mbar_init(&xfull[s], 1);
        }
        tc::fence_mbar_init();
    }
    if (warp == 2) tc::tmem_alloc(tmem_slot, 512);
    if (warp == 0 && lane == 0) { tc::tma_prefetch(&tmQ); tc::tma_prefetch(&tmX); }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int nunits = a.nqp * a.nsplit;

    if (warp == 0 && lane == 0) {
        // ================= TMA producer
        uint32_t g = 0, ul = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++ul) {
            const int qp = u % a.nqp, sp = u / a.nqp;
            const int64_t ib = (int64_t)sp * a.split_items;
            const int64_t ie = min(a.n, ib + a.split_items);
            // query blocks of this pair that hold any query (a block wholly past Qb
            // is neither loaded nor multiplied)
            const int nh = min(GT_QB, (a.Qb - qp * GT_QB * GT_M + GT_M - 1) / GT_M);
            if (ul > 0) tc::mbar_wait(a_empty, (ul - 1) & 1);
            tc::mbar_arrive_expect_tx(a_full, nh * a.kblocks * GT_A_BLK);
            for (int h = 0; h < nh; ++h)
                for (int kb = 0; kb < a.kblocks; ++kb)
                    tc::tma_load_2d(sA + (h * a.kblocks + kb) * GT_A_BLK, &tmQ, a_full, kb * GT_KB,
                                    (qp * GT_QB + h) * GT_M);
            const int64_t ntu = (ie - ib + GT_N - 1) / GT_N;
            for (int64_t jt = 0; jt < ntu; ++jt) {
                const int64_t i0 = gt_tile_at(ib, ie, qp, a.nqp, jt);
                if (jt + GT_PREFETCH < ntu) {
                    const int64_t ip = gt_tile_at(ib, ie, qp, a.nqp, jt + GT_PREFETCH);
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
            const int qp = u % a.nqp, sp = u / a.nqp;
            const int nh = min(GT_QB, (a.Qb - qp * GT_QB * GT_M + GT_M - 1) / GT_M);
            const int64_t ib = (int64_t)sp * a.split_items;
            const int64_t ie = min(a.n, ib + a.split_items);
            tc::mbar_wait(a_full, ul & 1);
            tc::tc_fence_after();
            for (int64_t i0 = ib; i0 < ie; i0 += GT_N, ++t) {   // (order irrelevant here)
                const uint32_t acc = t & 1, tr = t >> 1;
                tc::mbar_wait(&tempty[acc], (tr & 1) ^ 1);
                tc::tc_fence_after();
                for (int kb = 0; kb < a.kblocks; ++kb, ++g) {
                    const uint32_t s = g % a.stages, r = g / a.stages;
                    tc::mbar_wait(&full[s], r & 1);
                    tc::tc_fence_after();
                    const uint32_t bbase = tc::smem_u32(sB + s * GT_B_BLK);
                    const int nk = min(GT_KB / 16, (a.d - kb * GT_KB + 15) / 16);   // K = 16 per MMA
                    for (int h = 0; h < nh; ++h) {
                        const uint32_t abase = tc::smem_u32(sA + (h * a.kblocks + kb) * GT_A_BLK);
                        const uint32_t dt = tmem_base + (acc * GT_QB + h) * GT_N;
                        for (int kk = 0; kk < (a.dbg == 3 ? 0 : nk); ++kk)
                            tc::mma_f16_warp(dt, tc::umma_desc_sw128(abase + kk * 32),
                                        tc::umma_desc_sw128(bbase + kk * 32), idesc, (kb | kk) != 0);
                    }
                    tc::mma_commit_warp(&empty[s]);
                }
                tc::mma_commit_warp(&tfull[acc]);
            }
            tc::mma_commit_warp(a_empty);
        }
    } else if (warp == 3 && lane == 0) {
        // ================= |x| tile loader: bulk copy per tile into the buffer of its
        // TMEM stage, once the epilogue released that stage
        uint32_t t = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            const int sp = u / a.nqp;
            const int64_t ib = (int64_t)sp * a.split_items;
            const int64_t ie = min(a.n, ib + a.split_items);
            const int qp = u % a.nqp;
            const int64_t ntu = (ie - ib + GT_N - 1) / GT_N;
            for (int64_t jt = 0; jt < ntu; ++jt, ++t) {
                const int64_t i0 = gt_tile_at(ib, ie, qp, a.nqp, jt);
                const uint32_t acc = t & 1, tr = t >> 1;
                tc::mbar_wait(&tempty[acc], (tr & 1) ^ 1);
                tc::mbar_arrive_expect_tx(&xfull[acc], GT_N * 4);
                tc::bulk_load(sxn + acc * GT_N, a.xnorm + i0, GT_N * 4, &xfull[acc]);
            }
        }
    } else if (warp >= 4) {
        // ================= epilogue: thread <-> query row (TMEM lane); warps 4-7 own
        // query block 0 of the pair, warps 8-11 block 1
        // warps 4-11: lane quadrant = warp % 4; with two query blocks per CTA the
        // upper four own block 1, with one block they own the upper half of the columns
        const int grp = warp & 3;
        const int esub = (warp - 4) >> 2;
        const int h = GT_QB == 2 ? esub : 0;
        const int c_lo = GT_QB == 2 ? 0 : esub * GT_EPI_COLS;
        const int row = grp * 32 + lane;
        uint32_t t = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            const int qp = u % a.nqp, sp = u / a.nqp;
            const int64_t ib = (int64_t)sp * a.split_items;
            const int64_t ie = min(a.n, ib + a.split_items);
            const int q = (qp * GT_QB + h) * GT_M + row;
            const bool vq = q < a.Qb;
            const float qe = vq ? a.eps_rel * a.qnorm[q] : 0.f;
            // heap of this CTA's query row (CTAs of other item splits keep their own)
            float *hp = a.heap_smem
                            ? reinterpret_cast<float *>(tmem_slot + 4) + (esub * GT_M + row) * a.k
                            : a.heap + ((int64_t)(blockIdx.x * 2 + esub) * GT_M + row) * a.k;
            // survivors go to 16-slot chunks of the query's list reserved with one
            // atomic each; unused slots of the last chunk are filled with -1
            int32_t *cl = a.cand + (int64_t)(vq ? q : 0) * a.C;
            uint32_t sbase = 0, sleft = 0;
            float theta = -INFINITY, pub = -INFINITY;
            int hs = 0;
            if (vq) {
                const uint32_t o = a.theta_glob[q];
                if (o) theta = float_unorder(o);
            }
            // the hot-loop test uses a round-to-nearest FMA; thr_adj absorbs its rounding
            // (<= 2^-24 |result| near the threshold) so the filter stays certified
            float thr_adj = -INFINITY;
            auto set_theta = [&](float th) {
                theta = th;
                thr_adj = th - fabsf(th) * 2.384185791015625e-7f;   // 2^-22
            };
            if (theta > -INFINITY) set_theta(theta);
            const int64_t ntu = (ie - ib + GT_N - 1) / GT_N;
            for (int64_t jt = 0; jt < ntu; ++jt, ++t) {
                const int64_t i0 = gt_tile_at(ib, ie, qp, a.nqp, jt);
                const uint32_t acc = t & 1, tr = t >> 1;
                const float *xn = sxn + acc * GT_N;
                uint32_t o_next = 0;
                const bool share = vq && ((t & 3) == 0);
                if (share) o_next = *((volatile uint32_t *)&a.theta_glob[q]);   // consumed below
                tc::mbar_wait(&xfull[acc], tr & 1);
                tc::mbar_wait(&tfull[acc], tr & 1);
                tc::tc_fence_after();
                const uint32_t taddr = tmem_base + ((uint32_t)(grp * 32) << 16) + (acc * GT_QB + h) * GT_N;
                // largest |x| of the tile (the loader's buffer): s~ + qe |x| >= thr_adj
                // implies s~ >= thr_adj - qe xmax
                float xmax = 0.f;
                {
                    const float4 xv = reinterpret_cast<const float4 *>(xn + c_lo)[lane];
                    xmax = fmaxf(fmaxf(xv.x, xv.y), fmaxf(xv.z, xv.w));
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) xmax = fmaxf(xmax, __shfl_xor_sync(NR_FULL, xmax, o));
                }
                const float thr_tile = __fmaf_rd(-xmax, qe, thr_adj);
#pragma unroll 1
                for (int c = c_lo; c < c_lo + GT_EPI_COLS; c += 64) {
                    if (a.dbg >= 2) break;
                    uint32_t r0[32], r1[32];
                    tc::tmem_ld_32x32b_x32(taddr + c, r0);
                    tc::tmem_ld_32x32b_x32(taddr + c + 32, r1);
                    tc::tmem_ld_wait();
                    if (!vq || a.dbg) continue;
                    // cheap screen: max of the 64 approximate scores against the
                    // threshold loosened by the tile's largest error term
                    float m0 = __uint_as_float(r0[0]), m1 = __uint_as_float(r1[0]);
#pragma unroll
                    for (int j = 1; j < 32; ++j) {
                        m0 = fmaxf(m0, __uint_as_float(r0[j]));
                        m1 = fmaxf(m1, __uint_as_float(r1[j]));
                    }
                    if (fmaxf(m0, m1) < thr_tile) continue;
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
                            float s_j = 0.f;
#pragma unroll
                            for (int jj = 0; jj < 32; ++jj)
                                if (jj == j) s_j = __uint_as_float(hh ? r1[jj] : r0[jj]);
                            const float x = xn[col];
                            if (__fmaf_ru(x, qe, s_j) < theta) continue;   // exact re-test
                            const int64_t i = i0 + col;
                            if (i >= a.n) continue;
                            if (sleft == 0) { sbase = atomicAdd(&a.cnt[q], 16u); sleft = 16; }
                            if (sbase + (16 - sleft) < a.C) cl[sbase + (16 - sleft)] = (int32_t)i;
                            --sleft;
                            const float lb = __fmaf_rd(-x, qe, s_j);
                            if (hs < a.k) {          // min-heap push
                                int p = hs++;
                                while (p > 0) {
                                    const int par = (p - 1) >> 1;
                                    if (hp[par] <= lb) break;
                                    hp[p] = hp[par];
                                    p = par;
                                }
                                hp[p] = lb;
                                if (hs == a.k && hp[0] > theta) set_theta(hp[0]);
                            } else if (lb > hp[0]) { // replace the minimum
                                int p = 0;
                                while (true) {
                                    int ch = 2 * p + 1;
                                    if (ch >= a.k) break;
                                    if (ch + 1 < a.k && hp[ch + 1] < hp[ch]) ++ch;
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
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&tempty[acc]);
                if (share) {   // share the bound across CTAs (every 4 tiles)
                    if (hs == a.k && hp[0] > pub) {
                        pub = hp[0];
                        atomicMax(&a.theta_glob[q], float_order(pub));
                    }
                    if (o_next) {
                        const float g = float_unorder(o_next);
                        if (g > theta) set_theta(g);
                    }
                }
            }
            for (; sleft > 0; --sleft)
                if (sbase + (16 - sleft) < a.C) cl[sbase + (16 - sleft)] = -1;
        }
    }
    __syncthreads();
    if (warp == 2) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, 512);
    }
}

static size_t gt_tc_smem_bytes(int kblocks, int stages, int heap_k) {
    return 1024 + (size_t)GT_QB * kblocks * GT_A_BLK + (size_t)stages * GT_B_BLK + 2 * GT_N * 4 +
           (2 * GT_MAX_STAGES + 8) * 8 + 16 + (size_t)2 * GT_M * heap_k * 4;
}

size_t gt_heap_bytes(int k) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    return (size_t)sms * 2 * GT_M * k * 4;
}

bool gt_tc_supported(int d, int k) {
    const int dp = (d + 7) / 8 * 8;
    const int kb = (dp + GT_KB - 1) / GT_KB;
    return encode_fn() != nullptr && kb <= GT_MAX_KBLK && k <= GT_MAX_K &&
           gt_tc_smem_bytes(kb, 3, 0) <= 227 * 1024;
}

int launch_gt_filter_tc(const void *Xb, int64_t n, int d, int dp, const void *Qb16, int Qb,
                        const float *xnorm, const float *qnorm, float eps_rel, int k,
                        uint32_t *theta_glob, float *heap, int32_t *cand, uint32_t *cnt, int64_t C,
                        cudaStream_t s) {
    CUtensorMap tq, tx;
    if (!make_tmap(&tq, Qb16, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dp, Qb, GT_KB, GT_M) ||
        !make_tmap(&tx, Xb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dp, n, GT_KB, GT_N))
        return -1;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    GtArgs a;
    a.n = n;
    a.Qb = Qb;
    a.d = d;
    a.kblocks = (dp + GT_KB - 1) / GT_KB;
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
    a.nqp = (Qb + GT_QB * GT_M - 1) / (GT_QB * GT_M);
    const int64_t ntiles = (n + GT_N - 1) / GT_N;
    int nsplit = std::max(1, sms / a.nqp);     // one unit per CTA: no tail wave
    nsplit = (int)std::min<int64_t>(nsplit, ntiles);
    a.split_items = ((ntiles + nsplit - 1) / nsplit) * GT_N;
    a.nsplit = (int)((n + a.split_items - 1) / a.split_items);
    // deepest ring that fits, with the heaps in smem if they fit too
    a.stages = 3;
    a.heap_smem = 0;
    for (int st = GT_MAX_STAGES; st >= 3; --st)
        if (gt_tc_smem_bytes(a.kblocks, st, k) <= 227 * 1024) { a.stages = st; a.heap_smem = 1; break; }
    if (a.stages < 6)
        for (int st = GT_MAX_STAGES; st > a.stages; --st)
            if (gt_tc_smem_bytes(a.kblocks, st, 0) <= 227 * 1024) { a.stages = st; a.heap_smem = 0; break; }
    const size_t sm = gt_tc_smem_bytes(a.kblocks, a.stages, a.heap_smem ? k : 0);
    cudaFuncSetAttribute(gt_filter_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    const int grid = std::min(sms, a.nqp * a.nsplit);
    gt_filter_tc<<<grid, GT_THREADS, sm, s>>>(tq, tx, a);
    note_launch();
    return 0;
}

}  // namespace nrlsh
