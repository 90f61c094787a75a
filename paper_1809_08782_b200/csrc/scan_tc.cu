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
// select stages are shared (see the epilogue for how appends are reserved).
//
// CTA unit = (block of 128 queries, range of item tiles).  An item tile holds <= 256
// consecutive positions of ONE sub-dataset (tile list built at index build), so a
// query has one threshold per tile.
//   warps 0-3  expand packed codes into +-1 int8, K-major, 128B-swizzled smem tiles
//              (the block's 128 queries once per unit; 256 items per ring stage)
//   warp  4    TMEM allocator + warp-uniform tcgen05.mma kind::i8 issue (M = 128
//              queries, N = 256 items, K = 32 per instruction, ceil(L/32) per tile)
//   warps 8-23 epilogue: thread = query row, 64 columns each; tcgen05.ld, a max
//              screen per 32 columns, the exact test, the append
// Tiles of sub-datasets in which no query of the block has delta_j(q) >= 0 are
// skipped by every role (exact: no pair there can pass).
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

constexpr int ST_M = 128;                 // queries per block (TMEM lanes)
constexpr int ST_N = 256;                 // items per tile (TMEM columns)
constexpr int ST_ROWB = 128;              // bytes per swizzled K-major row (K <= 128 int8)
constexpr int ST_A = ST_M * ST_ROWB;      // 16 KB
constexpr int ST_B = ST_N * ST_ROWB;      // 32 KB per stage
constexpr int ST_STAGES = 4;             // max ring depth (runtime: a.stages)
constexpr int ST_THREADS = 24 * 32;        // 0-3 convert, 4 MMA, 8-23 epilogue
constexpr int ST_CONV = 128;              // converter threads (warps 0-3)
constexpr int ST_CH = 64;                 // append chunk (slots reserved per atomic)

struct ScanTcArgs {
    const uint32_t *codes;    // [n x W] partition order
    const uint32_t *qcodes;   // [Qb x W]
    const int8_t *delta;      // [Qb x m]
    const uint8_t *blk_act;   // [nqb x m]: any query of the block has delta_j >= 0
    const int4 *tiles;        // (j, p0, p1, 0)
    int ntiles;
    int Qb, m, L, W;
    int nqb, nsplit, tiles_per_split, stages;
    unsigned long long *clk;   // profiling experiments only (NRLSH_SCAN_CLK): per-CTA phase cycles
    int dbg;   // profiling experiments only (NRLSH_SCAN_DBG): 1 = epilogue reads TMEM only,
               // 2 = epilogue idle, 3 = converters store nothing
    unsigned long long *buf;  // [Qb x C]
    uint32_t *cnt;            // slots used per query (entries incl. sentinels)
    uint32_t *cntv;           // valid entries per query
    int64_t C;
    unsigned long long *pairs;
};

__device__ __forceinline__ uint32_t st_swz(int row, int kbyte) {
    return (uint32_t)(row * ST_ROWB + ((((kbyte >> 4) ^ (row & 7))) << 4) + (kbyte & 15));
}

// 4 code bits -> 4 int8 (+1 for a 1 bit, -1 for a 0 bit): spread bit i to byte i
// (nibble * 0x204081 puts bit i at bit 8i), then 0xFF ^ (byte * 0xFE).
__device__ __forceinline__ uint32_t expand4(uint32_t nib) {
    const uint32_t y = (nib * 0x00204081u) & 0x01010101u;
    return 0xFFFFFFFFu ^ (y * 0xFEu);
}

// one 32-bit code word (bits 32w .. 32w+31) -> two 16-byte chunks of the swizzled row
// (bytes for bits >= L are 0)
__device__ __forceinline__ void expand_word(uint32_t word, int w, int L, int row, uint8_t *tile) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int b0 = 32 * w + 16 * h + 4 * i;
            uint32_t x = expand4((word >> (16 * h + 4 * i)) & 0xFu);
            if (b0 + 4 > L) {   // partial nibble / past L: zero the bytes of bits >= L
                const int keep = max(0, min(4, L - b0));
                x &= keep >= 4 ? 0xFFFFFFFFu : ((1u << (8 * keep)) - 1u);
            }
            v[i] = x;
        }
        *reinterpret_cast<uint4 *>(tile + st_swz(row, 32 * w + 16 * h)) = make_uint4(v[0], v[1], v[2], v[3]);
    }
}

// Codes of rows [first, first + rows) -> registers (the loads of a whole tile are
// issued before any use); thread `tid` of `nthreads` owns rows tid, tid + nthreads, ...
template <int W, int RPT>
__device__ __forceinline__ void tile_load(const uint32_t *__restrict__ src, int64_t first, int rows,
                                          int tid, uint32_t (&c)[RPT][W]) {
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const int r = tid + k * ST_CONV;
        const int64_t p = first + min(r, max(rows - 1, 0));
        if (W == 4) {
            const uint4 v = __ldg(reinterpret_cast<const uint4 *>(src) + p);
            c[k][0] = v.x; c[k][1] = v.y; c[k][2] = v.z; c[k][3] = v.w;
        } else if (W == 2) {
            const uint2 v = __ldg(reinterpret_cast<const uint2 *>(src) + p);
            c[k][0] = v.x; c[k][1] = v.y;
        } else {
            c[k][0] = __ldg(src + p);
        }
    }
}

template <int W, int RPT>
__device__ __forceinline__ void tile_store(const uint32_t (&c)[RPT][W], int rows, int L, int tid,
                                           uint8_t *tile) {
#pragma unroll
    for (int k = 0; k < RPT; ++k) {
        const int r = tid + k * ST_CONV;
#pragma unroll
        for (int w = 0; w < W; ++w) expand_word(r < rows ? c[k][w] : 0u, w, r < rows ? L : 0, r, tile);
    }
}

template <int W>
__global__ void __launch_bounds__(ST_THREADS, 1) k6_scan_tc(ScanTcArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *sA = smem;                                   // 16 KB
    uint8_t *ring = sA + ST_A;                            // ST_STAGES x 32 KB
    int8_t *sdelta = reinterpret_cast<int8_t *>(ring + a.stages * ST_B);     // [128 x m]
    int4 *stile = reinterpret_cast<int4 *>(sdelta + ((ST_M * a.m + 15) & ~15)); // [tiles_per_split]
    uint64_t *bars = reinterpret_cast<uint64_t *>(stile + a.tiles_per_split);
    uint64_t *full = bars, *empty = bars + ST_STAGES;
    uint64_t *a_full = bars + 2 * ST_STAGES;
    uint64_t *tfull = a_full + 1, *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
    __shared__ int s_ntl;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // one unit per CTA: (query block, item split)
    const int qb = blockIdx.x % a.nqb, sp = blockIdx.x / a.nqb;
    const int t0 = sp * a.tiles_per_split, t1 = min(a.ntiles, t0 + a.tiles_per_split);
    const int q0 = qb * ST_M;
    const int nq = min(ST_M, a.Qb - q0);
    for (int e = threadIdx.x; e < ST_M * a.m; e += blockDim.x) {
        const int r = e / a.m;
        sdelta[e] = r < nq ? a.delta[(int64_t)(q0 + r) * a.m + (e % a.m)] : (int8_t)-1;
    }
    if (warp == 5) {   // compacted list of this unit's tiles in sub-datasets the block probes
        const uint8_t *act = a.blk_act + (int64_t)qb * a.m;
        int n = 0;
        for (int t = t0 + lane; t - lane < t1; t += 32) {
            int4 tl = make_int4(0, 0, 0, 0);
            const bool ok = t < t1 && act[(tl = a.tiles[t]).x];
            const unsigned bal = __ballot_sync(NR_FULL, ok);
            if (ok) stile[n + __popc(bal & lanemask_lt())] = tl;
            n += __popc(bal);
        }
        if (lane == 0) s_ntl = n;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            tc::mbar_init(&full[s], ST_CONV / 32);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(a_full, ST_CONV / 32);
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&tfull[s], 1);
            tc::mbar_init(&tempty[s], 16);
        }
        tc::fence_mbar_init();
    }
    if (warp == 4) tc::tmem_alloc(tmem_slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int ntl = s_ntl;
    const int ksteps = (a.L + 31) / 32;   // K = 32 int8 per MMA
    constexpr int RPT = ST_N / ST_CONV;   // item rows per converter thread

    if (warp < 4) {
        // ================= converters: queries once, then the tiles (loads of tile
        // t+1 in flight while tile t is expanded)
        {
            uint32_t c[ST_M / ST_CONV][W];
            tile_load<W, ST_M / ST_CONV>(a.qcodes, q0, nq, threadIdx.x, c);
            tile_store<W, ST_M / ST_CONV>(c, nq, a.L, threadIdx.x, sA);
            tc::fence_async_shared();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(a_full);
        }
        uint32_t cur[RPT][W];
        if (ntl > 0) tile_load<W, RPT>(a.codes, stile[0].y, stile[0].z - stile[0].y, threadIdx.x, cur);
        for (int t = 0; t < ntl; ++t) {
            const int4 tl = stile[t];
            uint32_t nxt[RPT][W];
            if (t + 1 < ntl)
                tile_load<W, RPT>(a.codes, stile[t + 1].y, stile[t + 1].z - stile[t + 1].y,
                                  threadIdx.x, nxt);
            const uint32_t s = t % a.stages, ph = (t / a.stages) & 1;
            const long long c0 = clock64();
            tc::mbar_wait(&empty[s], ph ^ 1);
            const long long c1 = clock64();
            if (a.dbg != 3) tile_store<W, RPT>(cur, tl.z - tl.y, a.L, threadIdx.x, ring + s * ST_B);
            if (a.clk && threadIdx.x == 0) {
                a.clk[blockIdx.x * 8 + 0] += c1 - c0;
                a.clk[blockIdx.x * 8 + 1] += clock64() - c1;
            }
            tc::fence_async_shared();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&full[s]);
#pragma unroll
            for (int k = 0; k < RPT; ++k)
#pragma unroll
                for (int w = 0; w < W; ++w) cur[k][w] = nxt[k][w];
        }
    } else if (warp == 4) {
        // ================= MMA issuer (warp-uniform, one elected lane issues)
        const uint32_t idesc = tc::umma_idesc_i8(ST_M, ST_N);
        tc::mbar_wait(a_full, 0);
        tc::tc_fence_after();
        const uint32_t abase = tc::smem_u32(sA);
        for (int t = 0; t < ntl; ++t) {
            const uint32_t acc = t & 1, tr = t >> 1;
            const long long c0 = clock64();
            tc::mbar_wait(&tempty[acc], (tr & 1) ^ 1);
            tc::tc_fence_after();
            const long long c1 = clock64();
            const uint32_t s = t % a.stages, ph = (t / a.stages) & 1;
            tc::mbar_wait(&full[s], ph);
            tc::tc_fence_after();
            if (a.clk && lane == 0) {
                a.clk[blockIdx.x * 8 + 2] += c1 - c0;
                a.clk[blockIdx.x * 8 + 3] += clock64() - c1;
            }
            const uint32_t bbase = tc::smem_u32(ring + s * ST_B);
            const uint32_t dt = tmem_base + acc * ST_N;
            for (int kk = 0; kk < ksteps; ++kk)
                tc::mma_i8_warp(dt, tc::umma_desc_sw128(abase + kk * 32),
                                tc::umma_desc_sw128(bbase + kk * 32), idesc, kk != 0);
            tc::mma_commit_warp(&empty[s]);
            tc::mma_commit_warp(&tfull[acc]);
        }
    } else if (warp >= 8) {
        // ================= epilogue: 16 warps; thread <-> query row (TMEM lane),
        // 64 columns each.  Appends fill 64-slot chunks of the query's buffer; the
        // next chunk is reserved one chunk ahead and only read when a group spills
        // into it, so the reservation atomic never stalls the common path.  Unused
        // reserved slots get the sentinel ~0 (skipped by select; the fallback test
        // counts real entries, cntv).
        const int grp = warp & 3;
        const int sub = (warp - 8) >> 2;            // 64-column slice of the tile
        const int row = grp * 32 + lane;
        const int q = q0 + row;
        const bool vq = row < nq;
        unsigned long long *bq = a.buf + (int64_t)(vq ? q : 0) * a.C;
        uint32_t nvalid = 0;
        uint32_t cb = 0, cl = 0, nb = 0;           // current chunk base / slots left; next chunk
        bool have = false;
        unsigned long long npairs = 0, dbg_sink = 0;
        for (int t = 0; t < ntl; ++t) {
            const int4 tl = stile[t];
            const uint32_t acc = t & 1, tr = t >> 1;
            const int rows = tl.z - tl.y;
            const int dl = sdelta[row * a.m + tl.x];
            const int thr = dl >= 0 ? a.L - 2 * dl : INT_MAX;
            const uint32_t fj = (uint32_t)(tl.x * (a.L + 1) + a.L);   // flat (j,h) = fj - (L+dot)/2
            npairs += rows;
            const long long c0 = clock64();
            tc::mbar_wait(&tfull[acc], tr & 1);
            tc::tc_fence_after();
            const long long c1 = clock64();
            const uint32_t taddr =
                tmem_base + ((uint32_t)(grp * 32) << 16) + acc * ST_N + sub * 64;
#pragma unroll 1
            for (int g = 0; g < (a.dbg == 2 ? 0 : 2); ++g) {
                uint32_t r[32];
                tc::tmem_ld_32x32b_x32(taddr + 32 * g, r);
                tc::tmem_ld_wait();
                if (a.dbg == 1) continue;
                int mx = (int)r[0];   // cheap screen: most groups of cold tiles pass nothing
#pragma unroll
                for (int e = 1; e < 32; ++e) mx = max(mx, (int)r[e]);
                if (mx < thr) continue;
                const int cbase = sub * 64 + 32 * g;
                uint32_t mask = 0;
#pragma unroll
                for (int e = 0; e < 32; ++e) mask |= (uint32_t)((int)r[e] >= thr) << e;
                const int valid_cols = rows - cbase;     // columns past the tile's rows
                if (valid_cols < 32) mask &= valid_cols <= 0 ? 0u : ((1u << valid_cols) - 1u);
                if (mask == 0u) continue;
                const uint32_t np = __popc(mask);
                nvalid += np;
                if (!have) {   // first pass of this (thread, unit): reserve two chunks
                    cb = atomicAdd(&a.cnt[q], (uint32_t)ST_CH);
                    nb = atomicAdd(&a.cnt[q], (uint32_t)ST_CH);
                    cl = ST_CH;
                    have = true;
                }
                const uint32_t pos0 = (uint32_t)(tl.y + cbase);
                if (np <= cl) {
                    // common path: the current chunk holds the group (no use of nb)
                    uint32_t slot = cb + (ST_CH - cl);
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        if ((mask >> e) & 1u) {
                            const unsigned long long v =
                                ((unsigned long long)(fj - (uint32_t)((a.L + (int)r[e]) >> 1)) << 32) | (pos0 + e);
                            if (a.dbg == 4) dbg_sink ^= v;
                            else if (slot < a.C) bq[slot] = v;
                            ++slot;
                        }
                    }
                    cl -= np;
                } else {
                    // spill into the reserved chunk (reserved at least one group ago)
                    const uint32_t cur0 = cb + (ST_CH - cl);
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        const uint32_t i = __popc(mask & ((1u << e) - 1u));
                        const uint32_t slot = i < cl ? cur0 + i : nb + (i - cl);
                        if (((mask >> e) & 1u) && slot < a.C)
                            bq[slot] = ((unsigned long long)(fj - (uint32_t)((a.L + (int)r[e]) >> 1)) << 32) |
                                       (pos0 + e);
                    }
                    cl = ST_CH - (np - cl);
                    cb = nb;
                    nb = atomicAdd(&a.cnt[q], (uint32_t)ST_CH);
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
            if (a.clk && warp == 8 && lane == 0) {
                a.clk[blockIdx.x * 8 + 4] += c1 - c0;
                a.clk[blockIdx.x * 8 + 5] += clock64() - c1;
            }
        }
        if (vq && have) {   // unused slots of the current and the reserved chunk
            for (uint32_t e = ST_CH - cl; e < (uint32_t)ST_CH; ++e)
                if (cb + e < a.C) bq[cb + e] = ~0ull;
            for (uint32_t e = 0; e < (uint32_t)ST_CH; ++e)
                if (nb + e < a.C) bq[nb + e] = ~0ull;
        }
        if (vq && nvalid) atomicAdd(&a.cntv[q], nvalid);
        if (vq && sub == 0 && a.pairs) atomicAdd(a.pairs, npairs + (dbg_sink == 1 ? 1 : 0));
    }
    __syncthreads();
    if (a.clk && threadIdx.x == 0) a.clk[blockIdx.x * 8 + 6] = (unsigned long long)ntl;
    if (warp == 4) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, 512);
    }
}

// blk_act[qb][j] = any query of block qb has delta_j(q) >= 0
__global__ void scan_blk_act(const int8_t *__restrict__ delta, int Qb, int m,
                             uint8_t *__restrict__ blk_act) {
    const int qb = blockIdx.x;
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        int any = 0;
        const int q1 = min(Qb, (qb + 1) * ST_M);
        for (int q = qb * ST_M; q < q1; ++q) any |= delta[(int64_t)q * m + j] >= 0;
        blk_act[(int64_t)qb * m + j] = (uint8_t)any;
    }
}

static size_t scan_tc_smem(int m, int L, int tiles_per_split, int stages) {
    (void)L;
    return 1024 + ST_A + (size_t)stages * ST_B +
           (size_t)((ST_M * m + 15) & ~15) + (size_t)tiles_per_split * 16 +
           (2 * ST_STAGES + 6) * 8 + 16;
}

// Opt-in (NRLSH_SCAN_TC=1): exact and parity-tested, but measured slower than the
// popcount scan on c4 (4.8 vs 0.9 ms per 1024 queries): the per-column epilogue
// (mask + predicated (j,h,pos) stores, ~350 instructions per 32 columns of a dense
// group) is instruction-bound while the MMA takes ~300 cycles per tile.
// "Tensor-core scan" has the measurements and the redesign (grouped appends).
bool scan_tc_supported(const nrlsh_index *ix) {
    // (smem: 16 KB queries + 128 KB ring + rank table + delta rows + tile list)
    return ix->tiles_d != nullptr && ix->L <= 128 && ix->W != 3 &&
           scan_tc_smem(ix->m, ix->L, 2048, 2) <= 226 * 1024 && getenv("NRLSH_SCAN_TC") &&
           atoi(getenv("NRLSH_SCAN_TC")) != 0;
}

void launch_scan_tc(const nrlsh_index *ix, const uint32_t *qcodes, const int8_t *delta, int Qb,
                    uint8_t *blk_act, unsigned long long *buf, uint32_t *cnt, uint32_t *cntv,
                    int64_t C, unsigned long long *pairs, cudaStream_t s) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    ScanTcArgs a;
    a.codes = ix->codes;
    a.qcodes = qcodes;
    a.delta = delta;
    a.blk_act = blk_act;
    a.tiles = ix->tiles_d;
    a.ntiles = ix->ntiles;
    a.Qb = Qb;
    a.m = ix->m;
    a.L = ix->L;
    a.W = ix->W;
    a.nqb = (Qb + ST_M - 1) / ST_M;
    // one unit per CTA; splits small enough that the tile list fits in smem
    a.nsplit = std::max(1, std::min(ix->ntiles, sms / a.nqb));
    while ((ix->ntiles + a.nsplit - 1) / a.nsplit > 2048) ++a.nsplit;
    a.tiles_per_split = (ix->ntiles + a.nsplit - 1) / a.nsplit;
    a.nsplit = (ix->ntiles + a.tiles_per_split - 1) / a.tiles_per_split;
    a.buf = buf;
    a.cnt = cnt;
    a.cntv = cntv;
    a.C = C;
    a.pairs = pairs;
    a.dbg = getenv("NRLSH_SCAN_DBG") ? atoi(getenv("NRLSH_SCAN_DBG")) : 0;
    scan_blk_act<<<a.nqb, 256, 0, s>>>(delta, Qb, ix->m, blk_act);
    a.stages = 2;
    for (int st = ST_STAGES; st > 2; --st)
        if (scan_tc_smem(ix->m, ix->L, a.tiles_per_split, st) <= 226 * 1024) { a.stages = st; break; }
    const size_t sm = scan_tc_smem(ix->m, ix->L, a.tiles_per_split, a.stages);
    const int grid = a.nqb * a.nsplit;
    a.clk = nullptr;
    if (getenv("NRLSH_SCAN_CLK")) {
        cudaMalloc(&a.clk, (size_t)grid * 64);
        cudaMemsetAsync(a.clk, 0, (size_t)grid * 64, s);
    }
#define NR_STC(W_)                                                                             \
    cudaFuncSetAttribute(k6_scan_tc<W_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k6_scan_tc<W_><<<grid, ST_THREADS, sm, s>>>(a)
    if (ix->W == 4) { NR_STC(4); } else if (ix->W == 2) { NR_STC(2); } else { NR_STC(1); }
#undef NR_STC
    note_launch(2);
    if (a.clk) {
        std::vector<unsigned long long> h((size_t)grid * 8);
        cudaMemcpyAsync(h.data(), a.clk, h.size() * 8, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        double acc[8] = {0};
        for (int b = 0; b < grid; ++b)
            for (int i = 0; i < 8; ++i) acc[i] += (double)h[(size_t)b * 8 + i];
        fprintf(stderr, "scan_tc clk/CTA: conv wait %.0f store %.0f | mma wait_tempty %.0f wait_full %.0f | "
                        "epi wait %.0f work %.0f | tiles %.0f\n",
                acc[0] / grid, acc[1] / grid, acc[2] / grid, acc[3] / grid, acc[4] / grid,
                acc[5] / grid, acc[6] / grid);
        cudaFree(a.clk);
    }
}

}  // namespace nrlsh
