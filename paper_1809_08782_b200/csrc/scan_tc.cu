// scan_tc.cu — K6 on the tensor cores (sm_100a): the batched Hamming scan as an
// int8 GEMM whose epilogue only extracts sign bits.
//
// A code bit b becomes s_b = +1 (bit 1) or -1 (bit 0), bits b >= L_h become 0,
// so for a query code q and an item code x
//     sum_b s_b(q) s_b(x) = (L - h) - h = L - 2h,   h = popc(q ^ x)      (exact)
// and the single-table multi-probe test of PAPER:209 / PAPER:217 — item i of
// sub-dataset j is probed for query q iff R[j][h] <= B(q), i.e. h <= delta_j(q)
// (the pilot's per-(query, sub-dataset) radius) — becomes
//     D'(i, q) = dot(i, q) - (L - 2 delta_j(q)) >= 0.
// The threshold is folded into the MMA: one more K = 32 step multiplies a constant
// item-side block [1, 1, 0, ...] by a query-side block [a_q, b_q, 0, ...] with
// a_q + b_q = 2 delta_j(q) - L (or -(L + 1) when delta_j(q) < 0: D' < 0 for every
// item), rewritten per tile because the tile's sub-dataset j changes it.  So the
// epilogue reads D' and needs only its sign: bit = 1 - (D' >>> 31).
//
// Layout (transposed against the other filters): M = 128 ITEMS of one sub-dataset
// (TMEM lanes; the index's sub-dataset-aligned tiles of <= 128 positions) x N = 256
// QUERIES (TMEM columns).  An epilogue warp owns 32 items x 128 queries; per 32-query
// chunk it loads D' (tcgen05.ld 32x32b.x32: its item's 32 values), packs the 32 sign
// bits with funnel shifts (one instruction per pair), and transposes the warp's 32x32
// bit matrix with five shuffle rounds, so lane c holds query c's pass mask over the
// warp's 32 items.  Chunks whose 32 queries all have delta_j(q) < 0 are skipped
// before the TMEM read.  Passing pairs are appended as ((j, h) << 32 | position) —
// h from popc(code ^ qcode) of the tile's packed codes — into an 8-entry shared-
// memory stage per (item quarter, query), flushed to the query's candidate buffer
// with one global reservation per 8 entries (the buffer format, counts and overflow
// rule are the popcount scan's, so the fallback and the select are shared).
//
// Warp roles (persistent CTA, one per SM; unit = (256-query block, split of the
// block's tile list)):
//   warp 0     TMA producer: the block's +-1 query rows once per unit, one item tile
//              (+-1 rows) per ring stage
//   warp 1     MMA issuer: ceil(L/32) K = 32 steps + the threshold step per tile,
//              TMEM double-buffered (2 x 256 columns)
//   warp 2     TMEM allocator
//   (warp 3    idle)
//   warps 4-19 epilogue: item quarter = warp % 4, query slice of 64 = (warp - 4) / 4
// Every per-tile operand arrives by TMA on the stage's barrier: the +-1 item rows,
// the threshold block of (the tile's sub-dataset, the query block) — built per
// sub-batch in the layout the MMA reads, [m][Qb'][64 B] — and the tile's packed
// codes; a stage is released once the MMA and the epilogue are both done with it.
#include <cuda.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "internal.h"
#include "tc_sm100.cuh"

namespace nrlsh {

bool make_tmap_2d(CUtensorMap *m, const void *base, CUtensorMapDataType dt, int esize,
                  uint64_t cols, uint64_t rows, uint32_t box_cols, uint32_t box_rows, int swizzle);
bool make_tmap_1d(CUtensorMap *m, const void *base, CUtensorMapDataType dt, int esize, uint64_t n,
                  uint32_t box);

constexpr int SM_M = 128;                 // items per tile (TMEM lanes)
constexpr int SM_N = 256;                 // queries per block (TMEM columns per buffer)
constexpr int SM_MAX_STAGES = 8;
constexpr int SM_EPI = 16;                // epilogue warps: 4 item quarters x 4 query slices
constexpr int SM_CPW = 8 * 4 / SM_EPI;    // 32-query chunks per epilogue warp
constexpr int SM_THREADS = 32 * (4 + SM_EPI);   // warps 0-3 control, then the epilogue
constexpr int SM_RUN = 32;                // slots per reservation run (lane-owned)
constexpr int SM_EXT = 64;                // bytes per row of the threshold blocks (sw64)

struct ScanMmaArgs {
    const int4 *tiles;        // (j, p0, p1, 0), sub-dataset aligned, <= 128 positions
    const int4 *tlist;        // [nqb x tstride] tile descriptors per query block
    const int32_t *tcount;    // [nqb]
    int64_t tstride;
    const int8_t *delta;      // [Qb x m]
    const uint32_t *codes;    // [n x W] packed, partition order
    const uint32_t *qcodes;   // [Qb x W]
    int64_t n;
    int Qb, m, L, W, Kp, nqb, nsplit, stages;
    int qbpad;                // rows per sub-dataset of the threshold table (Qb rounded up)
    const int16_t *thr;       // [m x qbpad]: 2 delta_j(q) - L, or -(L + 1) (delta_j(q) < 0)
    const int32_t *qperm;     // row of the sorted query order -> query (nullptr: identity)
    unsigned long long *buf;  // [Qb x C]
    uint32_t *cnt;            // slots used per query (entries + sentinels)
    uint32_t *cntv;           // real entries per query
    int64_t C;
    unsigned long long *pairs;
    int dbg;                  // NRLSH_SCAN_DBG: 1 = no codes TMA, 2 = no threshold TMA/MMA
    unsigned int *dbgout;     // first timed-out wait: (tag << 16) | (warp << 8) | blockIdx low bits
};

// bounded wait that reports instead of trapping (debug builds of the protocol); with
// NRLSH_SCAN_DBG & 16 the cycles spent waiting are accumulated per tag (dbgout[16 + tag])
__device__ unsigned long long g_sc_waitcyc[32];
__device__ __forceinline__ bool sc_wait(uint64_t *bar, uint32_t parity, int tag, unsigned int *dbgout) {
    const uint32_t ad = tc::smem_u32(bar);
    const long long t0 = dbgout ? clock64() : 0;
    for (long long it = 0; it < (1ll << 26); ++it) {
        uint32_t done;
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done) : "r"(ad), "r"(parity) : "memory");
        if (done) {
            if (dbgout && (threadIdx.x & 31) == 0) atomicAdd(&g_sc_waitcyc[tag], (unsigned long long)(clock64() - t0));
            return true;
        }
    }
    if (dbgout) atomicCAS(dbgout, 0u, ((unsigned)tag << 16) | ((threadIdx.x >> 5) << 8) | (blockIdx.x & 255) | 0x80000000u);
    return false;
}

// 4 code bits -> 4 int8 (+1 for a 1 bit, -1 for a 0 bit): spread bit i to byte i
// (nibble * 0x204081 puts bit i at bit 8i), then 0xFF ^ (byte * 0xFE).
__device__ __forceinline__ uint32_t expand4(uint32_t nib) {
    const uint32_t y = (nib * 0x00204081u) & 0x01010101u;
    return 0xFFFFFFFFu ^ (y * 0xFEu);
}

// codes [rows x W] -> +-1 int8 rows [rows x Kp] (bytes of bits >= L are 0)
__global__ void expand_pm(const uint32_t *__restrict__ codes, int64_t rows, int W, int L, int Kp,
                          int8_t *__restrict__ out, const int32_t *__restrict__ rowmap) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        uint32_t *dst = reinterpret_cast<uint32_t *>(out + r * Kp);
        const int64_t sr = rowmap ? rowmap[r] : r;   // (source row: the sorted order's query)
        for (int b0 = 0; b0 < Kp; b0 += 4) {
            uint32_t v = 0u;
            if (b0 < L) {
                v = expand4((codes[sr * W + (b0 >> 5)] >> (b0 & 31)) & 0xFu);
                if (b0 + 4 > L) v &= (1u << (8 * (L - b0))) - 1u;
            }
            dst[b0 >> 2] = v;
        }
    }
}

int scan_kp(int L) { return L <= 64 ? 64 : 128; }

void launch_expand_pm(const uint32_t *codes, int64_t rows, int W, int L, int8_t *out, cudaStream_t s) {
    expand_pm<<<grid_for(rows, 256, 4096), 256, 0, s>>>(codes, rows, W, L, scan_kp(L), out, nullptr);
    note_launch();
}

// per query block: the sub-dataset tiles in which some query of the block has
// delta_j(q) >= 0 (grid: x = chunks of 1024 tiles, y = blocks; count zeroed before)
__global__ void __launch_bounds__(256) scan_tile_lists(const int8_t *__restrict__ delta, int Qb, int m,
                                                       const int4 *__restrict__ tiles, int ntiles,
                                                       int4 *__restrict__ list, int64_t stride,
                                                       int32_t *__restrict__ count,
                                                       const int32_t *__restrict__ qperm) {
    __shared__ uint8_t act[256];
    const int qb = blockIdx.y;
    const int q0 = qb * SM_N, q1 = min(Qb, q0 + SM_N);
    for (int j = threadIdx.x; j < m; j += blockDim.x) act[j] = 0;
    __syncthreads();
    const int nv = (q1 - q0) * m;   // the block's delta rows
    for (int e = threadIdx.x; e < nv; e += blockDim.x) {
        const int r = q0 + e / m, j = e % m;
        if (radius_of(delta[(int64_t)(qperm ? qperm[r] : r) * m + j]) >= 0) act[j] = 1;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int t = blockIdx.x * 1024 + threadIdx.x; t < min(ntiles, (int)(blockIdx.x + 1) * 1024);
         t += blockDim.x) {
        const int4 tt = tiles[t];
        const bool on = act[tt.x] != 0;
        const unsigned am = __activemask();
        const unsigned bal = __ballot_sync(am, on);
        const int leader = __ffs(am) - 1;
        int base = 0;
        if (lane == leader && bal) base = atomicAdd(&count[qb], __popc(bal));
        base = __shfl_sync(am, base, leader);
        if (on) list[qb * stride + base + __popc(bal & lanemask_lt())] = tt;
    }
}

// 32 x 32 bit-matrix transpose across a warp: in, lane i holds row i (bit c = entry
// (i, c)); out, lane c holds column c (bit i = entry (i, c)).  Block swaps of size
// 16, 8, 4, 2, 1 (each swaps the off-diagonal blocks of every 2k x 2k block).
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
    for (int k = 16, i = 0; k > 0; k >>= 1, ++i) {
        const uint32_t lo = i == 0 ? 0x0000FFFFu
                          : i == 1 ? 0x00FF00FFu
                          : i == 2 ? 0x0F0F0F0Fu
                          : i == 3 ? 0x33333333u : 0x55555555u;   // bits c with (c & k) == 0
        const uint32_t y = __shfl_xor_sync(NR_FULL, x, k);
        x = (lane & k) ? ((x & ~lo) | ((y & ~lo) >> k)) : ((x & lo) | ((y & lo) << k));
    }
    return x;
}

// position of the k-th (0-based) set bit of m (k < popc(m))
__device__ __forceinline__ int nth_bit(uint32_t m, int k) {
    int pos = 0, c;
    c = __popc(m & 0xFFFFu); if (k >= c) { k -= c; m >>= 16; pos += 16; }
    c = __popc(m & 0xFFu);   if (k >= c) { k -= c; m >>= 8;  pos += 8; }
    c = __popc(m & 0xFu);    if (k >= c) { k -= c; m >>= 4;  pos += 4; }
    c = __popc(m & 0x3u);    if (k >= c) { k -= c; m >>= 2;  pos += 2; }
    if (k >= (int)(m & 1u)) pos += 1;
    return pos;
}

// physical byte offset of logical (row, byte b) in a 64-byte-swizzled K-major block
__device__ __forceinline__ uint32_t sw64_off(int row, int b) {
    return (uint32_t)(row * 64 + ((((b >> 4) ^ ((row >> 1) & 3)) & 3) << 4) + (b & 15));
}

template <int KP, int W>
__global__ void __launch_bounds__(SM_THREADS, 1)
    k6_scan_mma(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmX,
                ScanMmaArgs a) {
    constexpr int Q_BYTES = SM_N * KP;
    constexpr int X_BYTES = SM_M * KP;
    constexpr int T_BYTES = SM_N * 2;                            // threshold row (int16)
    constexpr int C_BYTES = SM_M * W * 4;                        // packed codes
    constexpr int D_OFF = X_BYTES + T_BYTES + ((C_BYTES + 16 + 15) & ~15);   // the tile's descriptor
    constexpr int S_BYTES = X_BYTES + ((T_BYTES + C_BYTES + 16 + 16 + 1023) & ~1023);
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *sQ = smem;                                          // queries (B operand)
    uint8_t *sAone = sQ + Q_BYTES;                               // [128 x 64] ones block
    uint8_t *sBext = sAone + SM_M * SM_EXT;                      // [2][256 x 64] thresholds
    uint8_t *ring = sBext + 2 * SM_N * SM_EXT;                   // stages x (X | thr | codes)
    uint64_t *bars = reinterpret_cast<uint64_t *>(ring + a.stages * S_BYTES);
    uint64_t *full = bars, *empty = bars + SM_MAX_STAGES;
    uint64_t *q_full = bars + 2 * SM_MAX_STAGES, *q_empty = q_full + 1;
    uint64_t *tfull = q_empty + 1, *tempty = tfull + 2;
    uint64_t *xfull = tempty + 2, *xempty = xfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(xempty + 2);   // (then the producer's ring)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long k_t0 = clock64();
    // constant item-side threshold block, zeroed query-side blocks (only bytes 0-1 of
    // their rows are ever written)
    for (int e = threadIdx.x; e < (SM_M + 2 * SM_N) * SM_EXT / 4; e += blockDim.x)
        reinterpret_cast<uint32_t *>(sAone)[e] = 0u;
    __syncthreads();
    for (int r = threadIdx.x; r < SM_M; r += blockDim.x) {
        sAone[sw64_off(r, 0)] = 1;
        sAone[sw64_off(r, 1)] = 1;
    }
    tc::fence_async_shared();
    if (threadIdx.x == 0) {
        // a stage is free once its MMAs completed (commit) and the epilogue warps
        // are done with its thresholds and codes
        for (int s = 0; s < a.stages; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1 + SM_EPI); }
        tc::mbar_init(q_full, 1);
        tc::mbar_init(q_empty, 1);
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&tfull[b], 1);
            tc::mbar_init(&tempty[b], SM_EPI);
            tc::mbar_init(&xfull[b], 1);
            tc::mbar_init(&xempty[b], 1);
        }
        tc::fence_mbar_init();
    }
    if (warp == 2) tc::tmem_alloc(tmem_slot, 512);
    if (warp == 0 && lane == 0) {
        tc::tma_prefetch(&tmQ);
        tc::tma_prefetch(&tmX);
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    pdl_wait();
    // unit = (query block qb, split sp): every nsplit-th listed tile of qb from sp on;
    // the units of one split run concurrently and share each tile's L2 fetch
    const int nunits = a.nqb * a.nsplit;
    auto unit_count = [&](int qb, int sp) -> int {
        const int c = a.tcount[qb];
        return c > sp ? (c - sp + a.nsplit - 1) / a.nsplit : 0;
    };
    auto unit_tile_ptr = [&](int qb, int sp, int v) -> const int4 * {
        return a.tlist + qb * a.tstride + sp + (int64_t)v * a.nsplit;
    };

    if (warp == 0) {
        if (lane == 0) {
            // ================= TMA producer.  Tile descriptors are prefetched PF tiles
            // ahead with cp.async into a ring (a dependent global load per tile would
            // bound the loop by its latency); each stage carries its tile's descriptor
            constexpr int PF = 32;
            int4 *ring_d = reinterpret_cast<int4 *>(bars + 2 * SM_MAX_STAGES + 12);   // (past tmem_slot)
            uint32_t g = 0, ul = 0;
            for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++ul) {
                const int qb = u % a.nqb, sp = u / a.nqb;
                const int nt = unit_count(qb, sp);
                for (int v = 0; v < PF; ++v) {
                    if (v < nt)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(tc::smem_u32(ring_d + v)),
                                     "l"(unit_tile_ptr(qb, sp, v)) : "memory");
                    asm volatile("cp.async.commit_group;" ::: "memory");
                }
                if (ul > 0) sc_wait(q_empty, (ul - 1) & 1, 1, a.dbgout);
                tc::mbar_arrive_expect_tx(q_full, Q_BYTES);
                tc::tma_load_2d(sQ, &tmQ, q_full, 0, qb * SM_N);
                for (int v = 0; v < nt; ++v, ++g) {
                    asm volatile("cp.async.wait_group %0;" ::"n"(PF - 1) : "memory");
                    const int4 tl = ring_d[v % PF];
                    if (v + PF < nt)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(tc::smem_u32(ring_d + v % PF)),
                                     "l"(unit_tile_ptr(qb, sp, v + PF)) : "memory");
                    asm volatile("cp.async.commit_group;" ::: "memory");
                    const uint32_t s = g % a.stages, r = g / a.stages;
                    sc_wait(&empty[s], (r & 1) ^ 1, 2, a.dbgout);
                    uint8_t *st = ring + s * S_BYTES;
                    *reinterpret_cast<int4 *>(st + D_OFF) = tl;   // (published by the arrive below)
                    tc::mbar_arrive_expect_tx(&full[s], X_BYTES + T_BYTES + C_BYTES + 16);
                    tc::tma_load_2d(st, &tmX, &full[s], 0, tl.y);
                    // the thresholds of (the tile's sub-dataset, this query block)
                    tc::bulk_load(st + X_BYTES, a.thr + ((int64_t)tl.x * a.qbpad + qb * SM_N), T_BYTES, &full[s]);
                    // the tile's packed codes: a 16-byte-aligned superset
                    const uint32_t *src = a.codes + (int64_t)tl.y * W;
                    const uint32_t *al = reinterpret_cast<const uint32_t *>(
                        reinterpret_cast<uintptr_t>(src) & ~(uintptr_t)15);
                    tc::bulk_load(st + X_BYTES + T_BYTES, al, C_BYTES + 16, &full[s]);
                }
                asm volatile("cp.async.wait_all;" ::: "memory");
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer (warp-uniform loop, one elected lane issues)
        const uint32_t idesc = tc::umma_idesc_i8(SM_M, SM_N);
        const int nk = (a.L + 31) / 32;
        uint32_t g = 0, t = 0, ul = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++ul) {
            const int qb = u % a.nqb, sp = u / a.nqb;
            sc_wait(q_full, ul & 1, 3, a.dbgout);
            tc::tc_fence_after();
            const uint32_t qbase = tc::smem_u32(sQ);
            const int nt = unit_count(qb, sp);
            for (int v = 0; v < nt; ++v, ++g, ++t) {
                const uint32_t buf = t & 1, tr = t >> 1;
                sc_wait(&tempty[buf], (tr & 1) ^ 1, 4, a.dbgout);
                const uint32_t s = g % a.stages, r = g / a.stages;
                sc_wait(&full[s], r & 1, 5, a.dbgout);
                sc_wait(&xfull[buf], tr & 1, 8, a.dbgout);
                tc::tc_fence_after();
                const uint32_t xbase = tc::smem_u32(ring + s * S_BYTES);
                const uint32_t dt = tmem_base + buf * SM_N;
#pragma unroll
                for (int kk = 0; kk < KP / 32; ++kk) {
                    if (kk >= nk) break;   // K bytes past L are zero
                    const uint64_t da = KP == 64 ? tc::umma_desc_sw64(xbase + kk * 32)
                                                 : tc::umma_desc_sw128(xbase + kk * 32);
                    const uint64_t db = KP == 64 ? tc::umma_desc_sw64(qbase + kk * 32)
                                                 : tc::umma_desc_sw128(qbase + kk * 32);
                    tc::mma_i8_warp(dt, da, db, idesc, kk != 0);
                }
                // D' = dot - (L - 2 delta_j(q)): the threshold step
                tc::mma_i8_warp(dt, tc::umma_desc_sw64(tc::smem_u32(sAone)),
                                tc::umma_desc_sw64(tc::smem_u32(sBext + buf * SM_N * SM_EXT)), idesc, 1);
                tc::mma_commit_warp(&empty[s]);
                tc::mma_commit_warp(&xempty[buf]);
                tc::mma_commit_warp(&tfull[buf]);
            }
            tc::mma_commit_warp(q_empty);
        }
    } else if (warp == 3) {
        // ================= the MMA's threshold block of each tile, from the stage's row
        uint32_t t = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            const int qb = u % a.nqb, sp = u / a.nqb;
            const int nt = unit_count(qb, sp);
            for (int v = 0; v < nt; ++v, ++t) {
                const uint32_t e = t & 1, s = t % a.stages;
                sc_wait(&xempty[e], ((t >> 1) & 1) ^ 1, 9, a.dbgout);
                sc_wait(&full[s], (t / a.stages) & 1, 10, a.dbgout);
                const uint4 v8 = *reinterpret_cast<const uint4 *>(ring + s * S_BYTES + X_BYTES + lane * 16);
                uint8_t *ext = sBext + e * SM_N * SM_EXT;
                const uint32_t w4[4] = {v8.x, v8.y, v8.z, v8.w};
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int val = (int)(int16_t)(uint16_t)(w4[k >> 1] >> (16 * (k & 1)));
                    const int lo = val >> 1, hi = val - lo;
                    const int row = lane * 8 + k;
                    *reinterpret_cast<uint16_t *>(ext + sw64_off(row, 0)) =
                        (uint16_t)((uint32_t)(uint8_t)(int8_t)lo | ((uint32_t)(uint8_t)(int8_t)hi << 8));
                }
                tc::fence_async_shared();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&xfull[e]);
            }
        }
    } else if (warp >= 4) {
        // ================= epilogue: item quarter g (TMEM lanes 32g..32g+31), query half hh
        const int g = warp & 3;
        const int hh = (warp - 4) >> 2;
        uint32_t t = 0, g2 = 0;
        unsigned long long npairs = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            const int qb = u % a.nqb, sp = u / a.nqb;
            // this lane's 4 queries (one per 32-column chunk) and their codes
            uint32_t qcw[SM_CPW][W];
            uint32_t rbase[SM_CPW], rleft[SM_CPW], rvalid[SM_CPW];   // this lane's open run per query
            int qrow[SM_CPW];                         // the query of each of its rows
#pragma unroll
            for (int cc = 0; cc < SM_CPW; ++cc) {
                rbase[cc] = 0u;
                rleft[cc] = 0u;
                rvalid[cc] = 0u;
                const int row = qb * SM_N + hh * SM_CPW * 32 + cc * 32 + lane;
                const int q = row < a.Qb ? (a.qperm ? __ldg(a.qperm + row) : row) : 0;
                qrow[cc] = q;
#pragma unroll
                for (int w = 0; w < W; ++w) qcw[cc][w] = row < a.Qb ? __ldg(a.qcodes + (int64_t)q * W + w) : 0u;
            }
            const int nt = unit_count(qb, sp);
            for (int v = 0; v < nt; ++v, ++t, ++g2) {
                const uint32_t b = t & 1, tr = t >> 1;
                const uint32_t s = g2 % a.stages, rs = g2 / a.stages;
                sc_wait(&tfull[b], tr & 1, 6, a.dbgout);
                sc_wait(&full[s], rs & 1, 7, a.dbgout);   // (the stage's thresholds and codes)
                tc::tc_fence_after();
                const int4 tl = *reinterpret_cast<const int4 *>(ring + s * S_BYTES + D_OFF);
                const int16_t *thr = reinterpret_cast<const int16_t *>(ring + s * S_BYTES + X_BYTES);
                const int myrows = min(32, max(0, tl.z - tl.y - 32 * g));
                const uint32_t fj = (uint32_t)(tl.x * (a.L + 1));
                // (the codes were copied from the 16-byte boundary at or below the tile's first)
                const uint32_t *sc = reinterpret_cast<const uint32_t *>(ring + s * S_BYTES + X_BYTES + T_BYTES) +
                                     ((tl.y * W) & 3) + g * 32 * W;
                const int inact = -(a.L + 1);
#pragma unroll
                for (int cc = 0; cc < SM_CPW; ++cc) {
                    __syncwarp();   // (reconverge: tcgen05.ld and the shuffles are warp-collective)
                    const int col0 = hh * SM_CPW * 32 + cc * 32;
                    const unsigned act = __ballot_sync(NR_FULL, thr[col0 + lane] != inact);
                    if (a.dbgout && lane == 0) atomicAdd(&g_sc_waitcyc[28], 1ull);   // chunk-tasks
                    if (!act || myrows == 0 || (a.dbg & 8)) continue;
                    if (a.dbgout && lane == 0) atomicAdd(&g_sc_waitcyc[29], 1ull);   // active chunk-tasks
                    npairs += (unsigned long long)__popc(act) * (unsigned)myrows;
                    uint32_t r[32];
                    tc::tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(g * 32) << 16) + b * SM_N + col0, r);
                    tc::tmem_ld_wait();
                    uint32_t fail = 0u;   // bit e: D'(item, query col0 + e) < 0
#pragma unroll
                    for (int e = 31; e >= 0; --e) fail = __funnelshift_l(r[e], fail, 1);
                    const uint32_t p = lane < myrows ? ~fail : 0u;
                    if (!__any_sync(NR_FULL, p != 0u)) continue;
                    if (a.dbgout && lane == 0) atomicAdd(&g_sc_waitcyc[30], 1ull);   // chunk-tasks with a pass
                    uint32_t mask = transpose32(p, lane);   // items passing query col0 + lane
                    if (!mask || (a.dbg & 4)) continue;
                    // Lane c appends query col0 + c's entries into runs of SM_RUN slots it owns,
                    // reserved with one global atomic (the unused tail of a run becomes ~0
                    // sentinels the select skips; cntv counts the real entries), so atomics on
                    // a query's counter stay rare
                    const int q = qrow[cc];
                    const uint32_t n = __popc(mask);
                    if (rleft[cc] < n) {   // close the run (sentinels), open one of >= n
                        for (uint32_t k = 0; k < rleft[cc]; ++k)
                            if (rbase[cc] + k < a.C) a.buf[(int64_t)q * a.C + rbase[cc] + k] = ~0ull;
                        const uint32_t len = max(n, (uint32_t)SM_RUN);
                        rbase[cc] = atomicAdd(&a.cnt[q], len);
                        rleft[cc] = len;
                    }
                    unsigned long long *dst = a.buf + (int64_t)q * a.C;
                    uint32_t slot = rbase[cc];
                    rbase[cc] += n;
                    rleft[cc] -= n;
                    rvalid[cc] += n;
                    const uint32_t pos0 = (uint32_t)(tl.y + 32 * g);
                    do {
                        const int i = __ffs(mask) - 1;
                        mask &= mask - 1;
                        int h = 0;
#pragma unroll
                        for (int w = 0; w < W; ++w) h += __popc(sc[i * W + w] ^ qcw[cc][w]);
                        if (slot < a.C) dst[slot] = ((unsigned long long)(fj + (uint32_t)h) << 32) | (pos0 + i);
                        ++slot;
                    } while (mask);
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    tc::mbar_arrive(&tempty[b]);
                    tc::mbar_arrive(&empty[s]);
                }
            }
            // close this lane's runs: sentinels in the unused slots, real entries counted
#pragma unroll
            for (int cc = 0; cc < SM_CPW; ++cc) {
                const int q = qrow[cc];
                for (uint32_t k = 0; k < rleft[cc]; ++k)
                    if (rbase[cc] + k < a.C) a.buf[(int64_t)q * a.C + rbase[cc] + k] = ~0ull;
                if (rvalid[cc]) atomicAdd(&a.cntv[q], rvalid[cc]);
            }
        }
        if (lane == 0 && npairs && a.pairs) atomicAdd(a.pairs, npairs);
    }
    if (a.dbgout && lane == 0) atomicAdd(&g_sc_waitcyc[20 + min(warp, 5)], (unsigned long long)(clock64() - k_t0));
    __syncthreads();
    if (warp == 2) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, 512);
    }
}

static size_t scan_mma_smem(int kp, int W, int stages) {
    const size_t stage_b = (size_t)SM_M * kp + (((size_t)SM_N * 2 + (size_t)SM_M * W * 4 + 32 + 1023) & ~(size_t)1023);
    return 1024 + (size_t)SM_N * kp + (size_t)SM_M * SM_EXT + 2 * (size_t)SM_N * SM_EXT +
           (size_t)stages * stage_b + (2 * SM_MAX_STAGES + 12) * 8 + 32 * 16 + 64;
}

// per (sub-dataset j, query q) of a sub-batch: 2 delta_j(q) - L, or -(L + 1) when
// delta_j(q) < 0 (no item can pass) and for the padding rows past Qb
// sort key of a query: sum_j (delta_j(q) + 1), monotone in its pilot bound B(q) —
// the active sub-datasets {j : delta_j(q) >= 0} of two queries are nested, so a block
// of neighbours in this order has nearly the active set of its least selective query
__global__ void scan_keys(const int8_t *__restrict__ delta, int Qb, int m, uint32_t *__restrict__ keys) {
    const int q = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (q >= Qb) return;
    uint32_t k = 0;
    for (int j = lane; j < m; j += 32) k += (uint32_t)(radius_of(delta[(int64_t)q * m + j]) + 1);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(NR_FULL, k, o);
    if (lane == 0) keys[q] = ~k;   // descending activity
}

__global__ void scan_thresholds(const int8_t *__restrict__ delta, int Qb, int qbpad, int m, int L,
                                int16_t *__restrict__ out, const int32_t *__restrict__ qperm) {
    const int64_t rows = (int64_t)m * qbpad;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int j = (int)(r / qbpad), q = (int)(r % qbpad);
        const int dl = q < Qb ? radius_of(delta[(int64_t)(qperm ? qperm[q] : q) * m + j]) : -1;
        out[r] = (int16_t)(dl >= 0 ? 2 * dl - L : -(L + 1));
    }
}

// Opt-in (NRLSH_SCAN_TC=1 at build and query; shared projection only): exact and
// parity-tested, but measured slower than the popcount scan on c4 (0.88-1.05 vs 0.58
// ms per 1024 queries): the epilogue issues at
// ~0.1 IPC per SMSP — per active 32 x 32 chunk a TMEM load, 32 funnel shifts and a
// 5-shuffle transpose, and ~73 passing pairs whose appends (per-lane runs, scattered
// 8-byte stores) cost ~18 SMSP-cycles each — while the base pipeline (TMA + MMA +
// threshold blocks) alone takes 0.3 ms.
bool scan_tc_supported(const nrlsh_index *ix) {
    if (!ix->codes_pm || !ix->ctiles_d || ix->L > 128 || ix->QM != 1) return false;
    const char *e = getenv("NRLSH_SCAN_TC");
    return e && atoi(e) != 0;
}

// buffer slots a query can lose to sentinels: one open run per (item quarter, unit)
int64_t scan_tc_slack(int Qmax) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int nqb = (Qmax + SM_N - 1) / SM_N;
    return 4ll * std::max(1, sms / nqb) * SM_RUN;
}

size_t scan_tc_ws_bytes(const nrlsh_index *ix, int Qb) {
    const int64_t nqb = (Qb + SM_N - 1) / SM_N;
    return (size_t)(nqb + 8) * 4 + (size_t)nqb * ix->nctiles * 16 + (size_t)Qb * scan_kp(ix->L) +
           (size_t)ix->m * nqb * SM_N * 2 + (size_t)std::max<int64_t>(Qb, 1024) * 4 + 8192;
}

int launch_scan_tc(const nrlsh_index *ix, const uint32_t *qcodes, const int8_t *delta, int Qb,
                   void *ws, unsigned long long *buf, uint32_t *cnt, uint32_t *cntv, int64_t C,
                   unsigned long long *pairs, cudaStream_t s) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int Kp = scan_kp(ix->L);
    ScanMmaArgs a;
    a.nqb = (Qb + SM_N - 1) / SM_N;
    int32_t *tcount = reinterpret_cast<int32_t *>(ws);
    int4 *tlist = reinterpret_cast<int4 *>(
        (reinterpret_cast<uintptr_t>(tcount + a.nqb + 4) + 15) & ~(uintptr_t)15);
    int8_t *qpm = reinterpret_cast<int8_t *>(
        (reinterpret_cast<uintptr_t>(tlist + (int64_t)a.nqb * ix->nctiles) + 1023) & ~(uintptr_t)1023);
    const int qbpad = a.nqb * SM_N;
    int16_t *thr = reinterpret_cast<int16_t *>(
        (reinterpret_cast<uintptr_t>(qpm + (size_t)Qb * Kp) + 1023) & ~(uintptr_t)1023);
    int32_t *qperm = reinterpret_cast<int32_t *>(thr + (size_t)ix->m * qbpad);
    // queries in descending activity (nested active sets: 256-query blocks of similar
    // queries list fewer tiles), their +-1 rows, the thresholds, the per-block tile lists
    const bool sorted = Qb > SM_N && Qb <= 4096 && !getenv("NRLSH_SCAN_NOSORT");
    if (sorted) {
        scan_keys<<<(Qb + 7) / 8, 256, 0, s>>>(delta, Qb, ix->m, reinterpret_cast<uint32_t *>(qperm));
        note_launch();
        launch_sort_keys(Qb, qperm, s);
    }
    expand_pm<<<grid_for(Qb, 256, 4096), 256, 0, s>>>(qcodes, Qb, ix->W, ix->L, Kp, qpm,
                                                      sorted ? qperm : nullptr);
    note_launch();
    scan_thresholds<<<grid_for((int64_t)ix->m * qbpad, 256, 4096), 256, 0, s>>>(
        delta, Qb, qbpad, ix->m, ix->L, thr, sorted ? qperm : nullptr);
    note_launch();
    cudaMemsetAsync(tcount, 0, (size_t)a.nqb * 4, s);
    scan_tile_lists<<<dim3((unsigned)((ix->nctiles + 1023) / 1024), a.nqb), 256, 0, s>>>(
        delta, Qb, ix->m, ix->ctiles_d, ix->nctiles, tlist, ix->nctiles, tcount, sorted ? qperm : nullptr);
    note_launch();
    CUtensorMap tq, tx;
    const int swz = Kp == 64 ? 64 : 128;
    if (!make_tmap_2d(&tq, qpm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, Kp, Qb, Kp, SM_N, swz) ||
        !make_tmap_2d(&tx, ix->codes_pm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, Kp, ix->n, Kp, SM_M, swz))
        return -1;
    a.thr = thr;
    a.qperm = sorted ? qperm : nullptr;
    a.qbpad = qbpad;
    a.tiles = ix->ctiles_d;
    a.tlist = tlist;
    a.tcount = tcount;
    a.tstride = ix->nctiles;
    a.delta = delta;
    a.codes = ix->codes;
    a.qcodes = qcodes;
    a.n = ix->n;
    a.Qb = Qb;
    a.m = ix->m;
    a.L = ix->L;
    a.W = ix->W;
    a.Kp = Kp;
    a.nsplit = std::max(1, sms / a.nqb);
    a.buf = buf;
    a.cnt = cnt;
    a.cntv = cntv;
    a.C = C;
    a.pairs = pairs;
    a.dbg = getenv("NRLSH_SCAN_DBG") ? atoi(getenv("NRLSH_SCAN_DBG")) : 0;
    static unsigned int *dbgbuf = nullptr;
    if (a.dbg && !dbgbuf) { cudaMalloc(&dbgbuf, 4); cudaMemset(dbgbuf, 0, 4); }
    a.dbgout = a.dbg ? dbgbuf : nullptr;
    a.stages = 2;
    for (int st = SM_MAX_STAGES; st > 2; --st)
        if (scan_mma_smem(Kp, ix->W, st) <= 227 * 1024) { a.stages = st; break; }
    const size_t sm = scan_mma_smem(Kp, ix->W, a.stages);
    const int grid = std::min(sms, a.nqb * a.nsplit);
#define NR_SC(KP_, W_)                                                                               \
    cudaFuncSetAttribute(k6_scan_mma<KP_, W_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    launch_pdl(k6_scan_mma<KP_, W_>, dim3(grid), dim3(SM_THREADS), sm, s, tq, tx, a)
    if (ix->W == 1) { NR_SC(64, 1); }
    else if (ix->W == 2) { NR_SC(64, 2); }
    else { NR_SC(128, 4); }
#undef NR_SC
    note_launch();
    if (a.dbg & 16) {
        unsigned long long w[32];
        cudaStreamSynchronize(s);
        cudaMemcpyFromSymbol(w, g_sc_waitcyc, sizeof(w));
        fprintf(stderr, "scan_tc waits (Mcycles summed over warps): prod q_empty %.1f empty %.1f | mma q_full %.1f "
                        "tempty %.1f full %.1f xfull %.1f | w3 xempty %.1f full %.1f | epi tfull %.1f full %.1f | "
                        "busy w0 %.1f w1 %.1f w2 %.1f w3 %.1f w4 %.1f w5+ %.1f (grid %d) chunk-tasks %llu active %llu "
                        "with-pass %llu\n",
                w[1] / 1e6, w[2] / 1e6, w[3] / 1e6, w[4] / 1e6, w[5] / 1e6, w[8] / 1e6, w[9] / 1e6, w[10] / 1e6,
                w[6] / 1e6, w[7] / 1e6, w[20] / 1e6, w[21] / 1e6, w[22] / 1e6, w[23] / 1e6, w[24] / 1e6,
                w[25] / 1e6, grid, w[28], w[29], w[30]);
        unsigned long long z[32] = {0};
        cudaMemcpyToSymbol(g_sc_waitcyc, z, sizeof(z));
    }
    if (a.dbg & 3) {
        unsigned int h = 0;
        cudaStreamSynchronize(s);
        cudaMemcpy(&h, dbgbuf, 4, cudaMemcpyDeviceToHost);
        fprintf(stderr, "scan_tc dbg=%d: stages=%d smem=%zu grid=%d nqb=%d first timeout=%08x (%s)\n", a.dbg,
                a.stages, sm, grid, a.nqb, h, cudaGetErrorString(cudaGetLastError()));
        cudaMemset(dbgbuf, 0, 4);
    }
    return 0;
}

}  // namespace nrlsh
