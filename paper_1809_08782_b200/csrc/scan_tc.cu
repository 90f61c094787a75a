// scan_tc.cu — K6 on the tensor cores (sm_100a): the batched Hamming scan as an
// int8 GEMM.
//
// A code bit b becomes s_b = +1 (bit 1) or -1 (bit 0), and bits b >= L_h become 0,
// so for a query code q and an item code x
//     sum_b s_b(q) s_b(x) = (L - h) - h = L - 2h,   h = popc(q ^ x)      (exact)
// and the single-table multi-probe test of PAPER:209 / PAPER:217 — item i of
// sub-dataset j is probed for query q iff R[j][h] <= B(q), i.e. h <= delta_j(q)
// (the pilot's per-(query, sub-dataset) radius) — becomes  dot >= L - 2 delta_j(q).
// Passing pairs are appended to the query's candidate buffer as ((j,h) << 32 | pos),
// exactly as the popcount scan (query_kernels.cu) appends them, so the fallback and
// select stages are shared.
//
// The +-1 item codes are expanded once, at index build, into an int8 matrix in
// partition order ([n x Kp], Kp = 64 or 128 bytes, 64/128-byte swizzled rows), so the
// kernel is a plain TMA -> tcgen05 kind::i8 -> TMEM pipeline (no converter warps):
//   warp 0     TMA producer: the block's 128 queries once per unit, then one
//              256-row tile per ring stage
//   warp 1     MMA issuer (warp-uniform, elected lane): M = 128 queries, N = 256
//              items, K = 32 per instruction, ceil(L/32) per tile, TMEM double-buffered
//   warp 2     TMEM allocator
//   warps 4-11 epilogue: thread = (query row, 128-column half); tcgen05.ld 32
//              columns, pass mask, the dots of a passing group staged in shared
//              memory, one append per passing pair into 64-slot chunks reserved per
//              thread
// Tiles are the index's sub-dataset-aligned runs of <= 256 positions, so a query has
// one threshold per tile; per query block only the tiles of sub-datasets with some
// delta_j(q) >= 0 are listed (exact: no pair elsewhere can pass).
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

constexpr int SM_M = 128;                 // queries per block (TMEM lanes)
constexpr int SM_N = 256;                 // items per tile (TMEM columns per buffer)
constexpr int SM_MAX_STAGES = 8;
constexpr int SM_THREADS = 384;           // warps 0-3 control, 4-11 epilogue
constexpr int SM_CH = 64;                 // append chunk (slots reserved per atomic)
constexpr int SM_DOT_LD = 36;             // staged dots per thread (16-byte aligned rows)

struct ScanMmaArgs {
    const int4 *tiles;        // (j, p0, p1, 0), sub-dataset aligned
    const int32_t *tlist;     // [nqb x tstride] tile indices per query block
    const int32_t *tcount;    // [nqb]
    int64_t tstride;
    const int8_t *delta;      // [Qb x m]
    int Qb, m, L, Kp, nqb, nsplit, stages;
    unsigned long long *buf;  // [Qb x C]
    uint32_t *cnt;            // slots used per query (entries incl. sentinels)
    uint32_t *cntv;           // valid entries per query
    int64_t C;
    unsigned long long *pairs;
};

// 4 code bits -> 4 int8 (+1 for a 1 bit, -1 for a 0 bit): spread bit i to byte i
// (nibble * 0x204081 puts bit i at bit 8i), then 0xFF ^ (byte * 0xFE).
__device__ __forceinline__ uint32_t expand4(uint32_t nib) {
    const uint32_t y = (nib * 0x00204081u) & 0x01010101u;
    return 0xFFFFFFFFu ^ (y * 0xFEu);
}

// codes [rows x W] -> +-1 int8 rows [rows x Kp] (bytes of bits >= L are 0)
__global__ void expand_pm(const uint32_t *__restrict__ codes, int64_t rows, int W, int L, int Kp,
                          int8_t *__restrict__ out) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        uint32_t *dst = reinterpret_cast<uint32_t *>(out + r * Kp);
        for (int b0 = 0; b0 < Kp; b0 += 4) {
            uint32_t v = 0u;
            if (b0 < L) {
                v = expand4((codes[r * W + (b0 >> 5)] >> (b0 & 31)) & 0xFu);
                if (b0 + 4 > L) v &= (1u << (8 * (L - b0))) - 1u;
            }
            dst[b0 >> 2] = v;
        }
    }
}

int scan_kp(int L) { return L <= 64 ? 64 : 128; }

void launch_expand_pm(const uint32_t *codes, int64_t rows, int W, int L, int8_t *out, cudaStream_t s) {
    expand_pm<<<grid_for(rows, 256, 4096), 256, 0, s>>>(codes, rows, W, L, scan_kp(L), out);
    note_launch();
}

// per query block: the sub-dataset tiles in which some query of the block has
// delta_j(q) >= 0 (grid: x = chunks of 1024 tiles, y = blocks; count zeroed before)
__global__ void __launch_bounds__(256) scan_tile_lists(const int8_t *__restrict__ delta, int Qb, int m,
                                                       const int4 *__restrict__ tiles, int ntiles,
                                                       int32_t *__restrict__ list, int64_t stride,
                                                       int32_t *__restrict__ count) {
    __shared__ uint8_t act[256];
    const int qb = blockIdx.y;
    const int q0 = qb * SM_M, q1 = min(Qb, q0 + SM_M);
    for (int j = threadIdx.x; j < m; j += blockDim.x) act[j] = 0;
    __syncthreads();
    const int nv = (q1 - q0) * m;   // the block's delta rows, read coalesced
    for (int e = threadIdx.x; e < nv; e += blockDim.x)
        if (delta[(int64_t)q0 * m + e] >= 0) act[e % m] = 1;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    for (int t = blockIdx.x * 1024 + threadIdx.x; t < min(ntiles, (int)(blockIdx.x + 1) * 1024);
         t += blockDim.x) {
        const bool on = act[tiles[t].x] != 0;
        const unsigned am = __activemask();
        const unsigned bal = __ballot_sync(am, on);
        const int leader = __ffs(am) - 1;
        int base = 0;
        if (lane == leader && bal) base = atomicAdd(&count[qb], __popc(bal));
        base = __shfl_sync(am, base, leader);
        if (on) list[qb * stride + base + __popc(bal & lanemask_lt())] = t;
    }
}

template <int KP>
__global__ void __launch_bounds__(SM_THREADS, 1)
    k6_scan_mma(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmX,
                ScanMmaArgs a) {
    constexpr int A_BYTES = SM_M * KP;
    constexpr int B_BYTES = SM_N * KP;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *sA = smem;
    uint8_t *ring = sA + A_BYTES;
    int *sdot = reinterpret_cast<int *>(ring + a.stages * B_BYTES);          // [256][SM_DOT_LD]
    uint64_t *bars = reinterpret_cast<uint64_t *>(sdot + 256 * SM_DOT_LD);
    uint64_t *full = bars, *empty = bars + SM_MAX_STAGES;
    uint64_t *a_full = bars + 2 * SM_MAX_STAGES, *a_empty = a_full + 1;
    uint64_t *tfull = a_empty + 1, *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
        tc::mbar_init(a_full, 1);
        tc::mbar_init(a_empty, 1);
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&tfull[b], 1);
            tc::mbar_init(&tempty[b], 8);
        }
        tc::fence_mbar_init();
    }
    if (warp == 2) tc::tmem_alloc(tmem_slot, 512);
    if (warp == 0 && lane == 0) { tc::tma_prefetch(&tmQ); tc::tma_prefetch(&tmX); }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // unit = (query block qb, split sp): every nsplit-th listed tile of qb from sp on;
    // the units of one split run concurrently and share each tile's L2 fetch
    const int nunits = a.nqb * a.nsplit;
    auto unit_count = [&](int qb, int sp) -> int {
        const int c = a.tcount[qb];
        return c > sp ? (c - sp + a.nsplit - 1) / a.nsplit : 0;
    };
    auto unit_tile = [&](int qb, int sp, int v) -> int4 {
        return a.tiles[__ldg(a.tlist + qb * a.tstride + sp + (int64_t)v * a.nsplit)];
    };

    if (warp == 0 && lane == 0) {
        // ================= TMA producer
        uint32_t g = 0, ul = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++ul) {
            const int qb = u % a.nqb, sp = u / a.nqb;
            if (ul > 0) tc::mbar_wait(a_empty, (ul - 1) & 1);
            tc::mbar_arrive_expect_tx(a_full, A_BYTES);
            tc::tma_load_2d(sA, &tmQ, a_full, 0, qb * SM_M);
            const int nt = unit_count(qb, sp);
            for (int v = 0; v < nt; ++v, ++g) {
                const int4 tl = unit_tile(qb, sp, v);
                const uint32_t s = g % a.stages, r = g / a.stages;
                tc::mbar_wait(&empty[s], (r & 1) ^ 1);
                tc::mbar_arrive_expect_tx(&full[s], B_BYTES);
                tc::tma_load_2d(ring + s * B_BYTES, &tmX, &full[s], 0, tl.y);
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer
        const uint32_t idesc = tc::umma_idesc_i8(SM_M, SM_N);
        uint32_t g = 0, t = 0, ul = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x, ++ul) {
            const int qb = u % a.nqb, sp = u / a.nqb;
            tc::mbar_wait(a_full, ul & 1);
            tc::tc_fence_after();
            const uint32_t abase = tc::smem_u32(sA);
            const int nt = unit_count(qb, sp);
            for (int v = 0; v < nt; ++v, ++g, ++t) {
                const uint32_t buf = t & 1, tr = t >> 1;
                tc::mbar_wait(&tempty[buf], (tr & 1) ^ 1);
                tc::tc_fence_after();
                const uint32_t s = g % a.stages, r = g / a.stages;
                tc::mbar_wait(&full[s], r & 1);
                tc::tc_fence_after();
                const uint32_t bbase = tc::smem_u32(ring + s * B_BYTES);
                const uint32_t dt = tmem_base + buf * SM_N;
#pragma unroll
                for (int kk = 0; kk < KP / 32; ++kk) {
                    if (kk * 32 >= a.L) break;   // K bytes past L are zero
                    const uint64_t da = KP == 64 ? tc::umma_desc_sw64(abase + kk * 32)
                                                 : tc::umma_desc_sw128(abase + kk * 32);
                    const uint64_t db = KP == 64 ? tc::umma_desc_sw64(bbase + kk * 32)
                                                 : tc::umma_desc_sw128(bbase + kk * 32);
                    tc::mma_i8_warp(dt, da, db, idesc, kk != 0);
                }
                tc::mma_commit_warp(&empty[s]);
                tc::mma_commit_warp(&tfull[buf]);
            }
            tc::mma_commit_warp(a_empty);
        }
    } else if (warp >= 4) {
        // ================= epilogue: thread <-> (query row = TMEM lane, 128-column half)
        const int grp = warp & 3;
        const int half = (warp - 4) >> 2;
        const int row = grp * 32 + lane;
        int *my = sdot + (threadIdx.x - 128) * SM_DOT_LD;
        uint32_t t = 0;
        for (int u = blockIdx.x; u < nunits; u += gridDim.x) {
            const int qb = u % a.nqb, sp = u / a.nqb;
            const int q = qb * SM_M + row;
            const bool vq = q < a.Qb;
            unsigned long long *bq = a.buf + (int64_t)(vq ? q : 0) * a.C;
            uint32_t cb = 0, cl = 0, nvalid = 0;
            unsigned long long npairs = 0;
            const int nt = unit_count(qb, sp);
            for (int v = 0; v < nt; ++v, ++t) {
                const int4 tl = unit_tile(qb, sp, v);
                const int rows = tl.z - tl.y;
                const int dl = vq ? (int)a.delta[(int64_t)q * a.m + tl.x] : -1;
                const int thr = dl >= 0 ? a.L - 2 * dl : INT_MAX;
                const uint32_t fj = (uint32_t)(tl.x * (a.L + 1));
                if (dl >= 0 && half == 0) npairs += rows;
                const uint32_t buf = t & 1, tr = t >> 1;
                tc::mbar_wait(&tfull[buf], tr & 1);
                tc::tc_fence_after();
                if (__any_sync(NR_FULL, dl >= 0)) {
                    const uint32_t taddr = tmem_base + ((uint32_t)(grp * 32) << 16) + buf * SM_N + half * 128;
#pragma unroll 1
                    for (int gcol = 0; gcol < 128; gcol += 32) {
                        uint32_t r[32];
                        tc::tmem_ld_32x32b_x32(taddr + gcol, r);
                        tc::tmem_ld_wait();
                        const int c0 = half * 128 + gcol;
                        uint32_t mask = 0;
#pragma unroll
                        for (int e = 0; e < 32; ++e) mask |= (uint32_t)((int)r[e] >= thr) << e;
                        const int vc = rows - c0;   // columns past the tile's rows
                        if (vc < 32) mask &= vc <= 0 ? 0u : ((1u << vc) - 1u);
                        if (!mask) continue;
#pragma unroll
                        for (int e = 0; e < 32; e += 4)
                            *reinterpret_cast<int4 *>(my + e) =
                                make_int4((int)r[e], (int)r[e + 1], (int)r[e + 2], (int)r[e + 3]);
                        nvalid += __popc(mask);
                        const uint32_t pos0 = (uint32_t)(tl.y + c0);
                        while (mask) {
                            const int e = __ffs(mask) - 1;
                            mask &= mask - 1;
                            const uint32_t h = (uint32_t)((a.L - my[e]) >> 1);
                            if (cl == 0) { cb = atomicAdd(&a.cnt[q], (uint32_t)SM_CH); cl = SM_CH; }
                            const uint32_t slot = cb + (SM_CH - cl);
                            if (slot < a.C) bq[slot] = ((unsigned long long)(fj + h) << 32) | (pos0 + e);
                            --cl;
                        }
                    }
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&tempty[buf]);
            }
            // unused slots of the last chunk: sentinel (skipped by select; the fallback
            // test counts real entries, cntv)
            for (; cl > 0; --cl)
                if (cb + (SM_CH - cl) < a.C) bq[cb + (SM_CH - cl)] = ~0ull;
            if (vq && nvalid) atomicAdd(&a.cntv[q], nvalid);
            if (vq && npairs && a.pairs) atomicAdd(a.pairs, npairs);
        }
    }
    __syncthreads();
    if (warp == 2) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, 512);
    }
}

static size_t scan_mma_smem(int kp, int stages) {
    return 1024 + (size_t)SM_M * kp + (size_t)stages * SM_N * kp + 256 * SM_DOT_LD * 4 +
           (2 * SM_MAX_STAGES + 6) * 8 + 16;
}

// Opt-in (NRLSH_SCAN_TC=1): exact and parity-tested, but measured slower than the
// popcount scan on c4 (0.93 vs 0.58 ms per 1024 queries): the tensor pipe is ~4%
// busy; the epilogue's per-pair appends (divergent loops over the pass bits, chunk
// reservations) bound it.  DESIGN.md "Tensor-core scan" has the numbers.
bool scan_tc_supported(const nrlsh_index *ix) {
    if (!ix->codes_pm || !ix->tiles_d || ix->L > 128) return false;
    const char *e = getenv("NRLSH_SCAN_TC");
    return e && atoi(e) != 0;
}

size_t scan_tc_ws_bytes(const nrlsh_index *ix, int Qb) {
    const int64_t nqb = (Qb + SM_M - 1) / SM_M;
    return (size_t)(nqb * (1 + ix->ntiles) + 4) * 4 + (size_t)Qb * scan_kp(ix->L) + 2048;
}

int launch_scan_tc(const nrlsh_index *ix, const uint32_t *qcodes, const int8_t *delta, int Qb,
                   void *ws, unsigned long long *buf, uint32_t *cnt, uint32_t *cntv, int64_t C,
                   unsigned long long *pairs, cudaStream_t s) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int Kp = scan_kp(ix->L);
    ScanMmaArgs a;
    a.nqb = (Qb + SM_M - 1) / SM_M;
    int32_t *tcount = reinterpret_cast<int32_t *>(ws);
    int32_t *tlist = tcount + a.nqb + 4;
    int8_t *qpm = reinterpret_cast<int8_t *>(
        (reinterpret_cast<uintptr_t>(tlist + (int64_t)a.nqb * ix->ntiles) + 1023) & ~(uintptr_t)1023);
    // the queries' +-1 rows, the per-block tile lists
    launch_expand_pm(qcodes, Qb, ix->W, ix->L, qpm, s);
    cudaMemsetAsync(tcount, 0, (size_t)a.nqb * 4, s);
    scan_tile_lists<<<dim3((unsigned)((ix->ntiles + 1023) / 1024), a.nqb), 256, 0, s>>>(
        delta, Qb, ix->m, ix->tiles_d, ix->ntiles, tlist, ix->ntiles, tcount);
    note_launch();
    CUtensorMap tq, tx;
    if (!make_tmap_2d(&tq, qpm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, Kp, Qb, Kp, SM_M, Kp) ||
        !make_tmap_2d(&tx, ix->codes_pm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, Kp, ix->n, Kp, SM_N, Kp))
        return -1;
    a.tiles = ix->tiles_d;
    a.tlist = tlist;
    a.tcount = tcount;
    a.tstride = ix->ntiles;
    a.delta = delta;
    a.Qb = Qb;
    a.m = ix->m;
    a.L = ix->L;
    a.Kp = Kp;
    a.nsplit = std::max(1, sms / a.nqb);
    a.buf = buf;
    a.cnt = cnt;
    a.cntv = cntv;
    a.C = C;
    a.pairs = pairs;
    a.stages = 2;
    for (int st = SM_MAX_STAGES; st > 2; --st)
        if (scan_mma_smem(Kp, st) <= 227 * 1024) { a.stages = st; break; }
    const size_t sm = scan_mma_smem(Kp, a.stages);
    const int grid = std::min(sms, a.nqb * a.nsplit);
    if (Kp == 64) {
        cudaFuncSetAttribute(k6_scan_mma<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k6_scan_mma<64><<<grid, SM_THREADS, sm, s>>>(tq, tx, a);
    } else {
        cudaFuncSetAttribute(k6_scan_mma<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k6_scan_mma<128><<<grid, SM_THREADS, sm, s>>>(tq, tx, a);
    }
    note_launch();
    return 0;
}

}  // namespace nrlsh
