// codes_tc.cu — K3 on the 5th-generation tensor cores (sm_100a): the SRP
// projection of the SIMPLE-LSH-transformed items, fused with sign and bit-pack.
//
//   y_ib = sum_k x_ik A_kb + A_db t_i,   t_i = sqrt(max(0, V_j - ||x_i||^2))
//   bit b of item i = [y_ib >= 0]
//
// y = U_j * (A_b . P(x_i)) with P(x) = [x/U_j; sqrt(1 - ||x/U_j||^2)] (Eq. (8),
// PAPER:85-87, applied after Alg. 1 l.6), and U_j > 0 does not change the sign of
// Eq. (4); V_j = 0 (a sub-dataset of zero vectors) gives P(x) = [0;1],
// i.e. t = 1.  Codes are written at the item's position in sub-dataset order.
//
// Precision: A is TF32-exact by construction (include/nrlsh.h), so two kind::tf32
// MMAs on X = X_big + X_small (X_big = the top 11 significant bits of x, written
// explicitly; X_small = x - X_big, exact in fp32) give fp32-grade products
// (|x - X_big - tf32(X_small)| < 2^-20 |x|), far inside the 1e-5 parity band.
//
// CTA (persistent, one per SM): tile = 128 items (TMEM lanes) x N = 32W columns.
//   warps 0-7  convert: coalesced cp.async loads of X into per-thread raw
//              slots (up to 3 K-blocks ahead), split, store both halves into
//              128B-swizzled K-major smem K-blocks (32 tf32 wide), ring of stages
//   warp  8    TMEM allocator + single-thread tcgen05.mma issuer
//   warps 9-12 epilogue: tcgen05.ld the accumulator row, add A_d t_i, sign, pack,
//              scatter the W code words to pos_of_id[i]
// The projection matrix (B operand, N x K) stays resident in smem.
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"
#include "tc_sm100.cuh"

namespace nrlsh {

constexpr int CT_M = 128;
constexpr int CT_KB = 32;                 // tf32 elements per K-block (128-byte rows)
constexpr int CT_A_BLK = CT_M * 128;      // 16 KB per operand per K-block
constexpr int CT_STAGE = 2 * CT_A_BLK;    // big + small
constexpr int CT_CONV = 256;              // converter threads (warps 0-7)
constexpr int CT_THREADS = 13 * 32;

struct CodesArgs {
    const float *X;
    int64_t n;
    int d, KB, L, N, stages, raw;   // raw: cp.async slots per converter thread (lookahead raw-1)
    int64_t ntiles;
    const double *norm2;
    const uint8_t *part;
    const double *V;
    const float *Apad;       // [(d+1) x N]
    const int32_t *pos_of_id;
    uint32_t *codes;         // [n x N/32], partition order
    __nv_bfloat16 *Xb;       // optional bf16 row copy [n x dpb], PARTITION order (row pos_of_id[i])
    int dpb;
    float *Xpad;             // optional fp32 row copy [n x dpad], 16-byte rows (re-rank gathers)
    int dpad;
    // per-sub-dataset projections (reading Q4, NEXT-4): items in partition
    // order, tile t = ctiles[t] = (j, p0, p1) of <= 128 positions of sub-dataset j,
    // projected by A_j = Apad + j (d+1) N; each CTA takes a contiguous run of tiles, so
    // the resident B operand is reloaded only when j changes
    const int4 *ctiles;      // nullptr: shared A, tiles of 128 consecutive items
    const int32_t *perm;     // position -> item id
};

// tile sequence of a CTA: shared A — tiles blockIdx.x + t gridDim.x; per-sub-dataset
// A_j — the contiguous run [lo, hi)
template <bool PP>
__device__ __forceinline__ void ct_range(const CodesArgs &a, int64_t &lo, int64_t &hi) {
    if (PP) {
        lo = a.ntiles * blockIdx.x / gridDim.x;
        hi = a.ntiles * (blockIdx.x + 1) / gridDim.x;
    } else {
        lo = blockIdx.x;
        hi = a.ntiles;
    }
}
template <bool PP>
__device__ __forceinline__ int64_t ct_step(const CodesArgs &a) { return PP ? 1 : gridDim.x; }

// row rr of tile `tile`: item id (i < 0: past the tile / past n) and destination position
template <bool PP>
__device__ __forceinline__ void ct_row(const CodesArgs &a, int64_t tile, int rr, int64_t &i, int64_t &pos) {
    if (PP) {
        const int4 t = __ldg(a.ctiles + tile);
        const int64_t p = (int64_t)t.y + rr;
        if (p < t.z) { pos = p; i = __ldg(a.perm + p); }
        else { pos = -1; i = -1; }
    } else {
        i = tile * CT_M + rr;
        if (i >= a.n) i = -1;
        pos = -1;   // (shared A: pos_of_id[i], read where needed)
    }
}

__device__ __forceinline__ uint32_t swz(int row, int kbyte) {
    return (uint32_t)(row * 128 + ((((kbyte >> 4) ^ (row & 7))) << 4) + (kbyte & 15));
}

// Loads go through cp.async (zero-filled past n and d) into a per-thread raw slot
// ring: RAW K-blocks in flight per SM without holding them in registers.
constexpr int CT_RAW_SLOT = CT_CONV * 16 * 4;   // 16 KB: 16 floats per converter thread

template <int VEC, bool PP>
__device__ __forceinline__ void conv_issue(const CodesArgs &a, int64_t tile, int kb, int w, int l,
                                           uint8_t *slot, int32_t *posr) {
    // with the first K-block of a tile, the warp's 16 rows' partition positions (the
    // bf16 copy's destination rows; read back by the warp only)
    if (kb == 0 && a.Xb && l < 16) {
        if (PP) {   // destination rows are the positions themselves
            int64_t i, pos;
            ct_row<PP>(a, tile, 16 * w + l, i, pos);
            posr[16 * w + l] = (int32_t)pos;
        } else {
            const int64_t i = tile * CT_M + 16 * w + l;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, 4;" ::"r"(tc::smem_u32(posr + 16 * w + l)),
                         "l"(a.pos_of_id + (i < a.n ? i : a.n - 1))
                         : "memory");
        }
    }
    constexpr int lpr = VEC == 4 ? 8 : (VEC == 2 ? 16 : 32);
    constexpr int rpi = 32 / lpr;
    constexpr int ni = 16 / rpi;
    const int col = kb * CT_KB + (l % lpr) * VEC;
    const int cc = min(col, a.d - VEC);
    const int tid = w * 32 + l;
#pragma unroll
    for (int j = 0; j < ni; ++j) {
        const int rr = 16 * w + j * rpi + l / lpr;
        int64_t i, pos;
        ct_row<PP>(a, tile, rr, i, pos);
        const int64_t ic = i >= 0 ? i : 0;
        const float *p = a.X + ic * a.d + cc;
        const uint32_t dst = tc::smem_u32(slot + (size_t)(j * CT_CONV + tid) * VEC * 4);
        const int nb = ((i >= 0) && (col < a.d)) ? VEC * 4 : 0;
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(dst), "l"(p), "n"(VEC * 4),
                     "r"(nb)
                     : "memory");
    }
}

template <int VEC, bool PP>
__device__ __forceinline__ void conv_read(const uint8_t *slot, int w, int l, float (&v)[16]) {
    constexpr int lpr = VEC == 4 ? 8 : (VEC == 2 ? 16 : 32);
    constexpr int rpi = 32 / lpr;
    constexpr int ni = 16 / rpi;
    const int tid = w * 32 + l;
#pragma unroll
    for (int j = 0; j < ni; ++j) {
        const float *q = reinterpret_cast<const float *>(slot + (size_t)(j * CT_CONV + tid) * VEC * 4);
        if (VEC == 4) {
            const float4 t = *reinterpret_cast<const float4 *>(q);
            v[j * 4] = t.x; v[j * 4 + 1] = t.y; v[j * 4 + 2] = t.z; v[j * 4 + 3] = t.w;
        } else if (VEC == 2) {
            const float2 t = *reinterpret_cast<const float2 *>(q);
            v[j * 2] = t.x; v[j * 2 + 1] = t.y;
        } else {
            v[j] = q[0];
        }
    }
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait(int la) {
    if (la >= 3) asm volatile("cp.async.wait_group 3;" ::: "memory");
    else if (la == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
    else asm volatile("cp.async.wait_group 1;" ::: "memory");
}

template <int VEC, bool PP>
__device__ __forceinline__ void conv_store(uint8_t *stage, int w, int l, const float (&v)[16]) {
    constexpr int lpr = VEC == 4 ? 8 : (VEC == 2 ? 16 : 32);
    constexpr int rpi = 32 / lpr;
    constexpr int ni = 16 / rpi;
    const int kbyte = (l % lpr) * VEC * 4;
#pragma unroll
    for (int j = 0; j < ni; ++j) {
        const int rr = 16 * w + j * rpi + l / lpr;
        const uint32_t off = swz(rr, kbyte);
        uint32_t bg[VEC], sm[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
            const float x = v[j * VEC + e];
            const uint32_t b = __float_as_uint(x) & 0xFFFFE000u;   // top 11 significant bits
            bg[e] = b;
            sm[e] = __float_as_uint(x - __uint_as_float(b));       // exact residual
        }
        if (VEC == 4) {
            *reinterpret_cast<uint4 *>(stage + off) = make_uint4(bg[0], bg[1], bg[2], bg[3]);
            *reinterpret_cast<uint4 *>(stage + CT_A_BLK + off) = make_uint4(sm[0], sm[1], sm[2], sm[3]);
        } else if (VEC == 2) {
            *reinterpret_cast<uint2 *>(stage + off) = make_uint2(bg[0], bg[1]);
            *reinterpret_cast<uint2 *>(stage + CT_A_BLK + off) = make_uint2(sm[0], sm[1]);
        } else {
            *reinterpret_cast<uint32_t *>(stage + off) = bg[0];
            *reinterpret_cast<uint32_t *>(stage + CT_A_BLK + off) = sm[0];
        }
    }
}


// bf16 copy of the converter's slice of the rows (columns < dpb; zeros past d)
template <int VEC, bool PP>
__device__ __forceinline__ void conv_store_bf16(const CodesArgs &a, int64_t tile, int kb, int w, int l,
                                                const float (&v)[16], const int32_t *posr) {
    constexpr int lpr = VEC == 4 ? 8 : (VEC == 2 ? 16 : 32);
    constexpr int rpi = 32 / lpr;
    constexpr int ni = 16 / rpi;
    const int col = kb * CT_KB + (l % lpr) * VEC;
    if (col >= a.dpb) return;
#pragma unroll
    for (int j = 0; j < ni; ++j) {
        const int rr = 16 * w + j * rpi + l / lpr;
        const int32_t prow = posr[rr];
        if (PP ? prow < 0 : tile * CT_M + rr >= a.n) continue;
        __nv_bfloat16 *dst = a.Xb + (int64_t)prow * a.dpb + col;
        if (VEC == 4) {
            const __nv_bfloat162 p0 = __floats2bfloat162_rn(v[j * 4 + 0], v[j * 4 + 1]);
            const __nv_bfloat162 p1 = __floats2bfloat162_rn(v[j * 4 + 2], v[j * 4 + 3]);
            uint2 u;
            u.x = *reinterpret_cast<const uint32_t *>(&p0);
            u.y = *reinterpret_cast<const uint32_t *>(&p1);
            *reinterpret_cast<uint2 *>(dst) = u;
        } else if (VEC == 2) {
            *reinterpret_cast<__nv_bfloat162 *>(dst) = __floats2bfloat162_rn(v[j * 2], v[j * 2 + 1]);
        } else {
            *dst = __float2bfloat16_rn(v[j]);
        }
    }
}

template <int VEC, bool PP>
__device__ __forceinline__ void conv_store_pad(const CodesArgs &a, int64_t tile, int kb, int w, int l,
                                               const float (&v)[16]) {
    constexpr int lpr = VEC == 4 ? 8 : (VEC == 2 ? 16 : 32);
    constexpr int rpi = 32 / lpr;
    constexpr int ni = 16 / rpi;
    const int col = kb * CT_KB + (l % lpr) * VEC;
    if (col >= a.dpad) return;
#pragma unroll
    for (int j = 0; j < ni; ++j) {
        const int rr = 16 * w + j * rpi + l / lpr;
        int64_t i, pos;
        ct_row<PP>(a, tile, rr, i, pos);
        if (i < 0) continue;
        float *dst = a.Xpad + i * a.dpad + col;
        if (VEC == 4) *reinterpret_cast<float4 *>(dst) = make_float4(v[j * 4], v[j * 4 + 1], v[j * 4 + 2], v[j * 4 + 3]);
        else if (VEC == 2) *reinterpret_cast<float2 *>(dst) = make_float2(v[j * 2], v[j * 2 + 1]);
        else dst[0] = v[j];
    }
}

template <int VEC, bool PP>
__global__ void __launch_bounds__(CT_THREADS, 1) k3_codes_tc(CodesArgs a) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *ring = smem;                                        // stages x 32 KB
    uint8_t *rawr = ring + a.stages * CT_STAGE;                  // raw x 16 KB
    uint8_t *Bs = rawr + (size_t)a.raw * CT_RAW_SLOT;            // KB x N x 128 B
    float *Ad = reinterpret_cast<float *>(Bs + (size_t)a.KB * a.N * 128);   // [N]
    uint64_t *bars = reinterpret_cast<uint64_t *>(Ad + a.N);
    uint64_t *full = bars, *empty = bars + a.stages;
    uint64_t *tfull = bars + 2 * a.stages, *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);
    int32_t *posr = reinterpret_cast<int32_t *>(tempty + 4);     // [4][CT_M], ring by tile
    uint64_t *bdone = reinterpret_cast<uint64_t *>(posr + 4 * CT_M);   // MMAs drained (B reload)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int N = a.N;
    // resident B operand (A^T, K-major, swizzled) and A_d (shared A; per-sub-dataset
    // projections load A_j in the MMA warp when the tile's j changes)
    auto load_B = [&](const float *Aj, int t0, int nt) {
        for (int e = t0; e < a.KB * N * CT_KB; e += nt) {
            const int kb = e / (N * CT_KB), rem = e % (N * CT_KB);
            const int b = rem / CT_KB, k = rem % CT_KB;
            const int kg = kb * CT_KB + k;
            const float v = kg < a.d ? Aj[(size_t)kg * N + b] : 0.f;
            *reinterpret_cast<float *>(Bs + (size_t)kb * N * 128 + swz(b, k * 4)) = v;
        }
    };
    if (!PP) {
        load_B(a.Apad, threadIdx.x, blockDim.x);
        for (int b = threadIdx.x; b < N; b += blockDim.x) Ad[b] = a.Apad[(size_t)a.d * N + b];
    }
    tc::fence_async_shared();
    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            tc::mbar_init(&full[s], CT_CONV / 32);
            tc::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&tfull[s], 1);
            tc::mbar_init(&tempty[s], 4);
        }
        tc::mbar_init(bdone, 1);
        tc::fence_mbar_init();
    }
    const uint32_t tcols = N <= 16 ? 32 : (2 * N <= 64 ? 64 : (2 * N <= 128 ? 128 : 256));
    if (warp == 8) tc::tmem_alloc(tmem_slot, tcols);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp < 8) {
        // ================= converters
        // K-block g of this CTA = (tile blockIdx.x + (g / KB) gridDim.x, kb g % KB);
        // issue and consume cursors advance incrementally (no 64-bit divisions)
        int64_t tlo, thi;
        ct_range<PP>(a, tlo, thi);
        const int64_t tst = ct_step<PP>(a);
        const int64_t my_tiles = thi > tlo ? (thi - 1 - tlo) / tst + 1 : 0;
        const int64_t G = my_tiles * a.KB;
        const int la = a.raw - 1;
        int64_t i_tile = tlo, issued = 0;
        int i_kb = 0, i_ti = 0, i_slot = 0;
        auto issue = [&]() {
            if (issued < G) {
                conv_issue<VEC, PP>(a, i_tile, i_kb, warp, lane, rawr + (size_t)i_slot * CT_RAW_SLOT,
                                posr + (i_ti & 3) * CT_M);
                if (++i_kb == a.KB) { i_kb = 0; i_tile += tst; ++i_ti; }
                if (++i_slot == a.raw) i_slot = 0;
            }
            ++issued;
            cp_async_commit();   // (empty groups keep the group count uniform)
        };
        for (int g = 0; g < la; ++g) issue();
        int64_t tile = tlo;
        int kb = 0, ti = 0, rslot = 0;
        uint32_t s = 0, ph = 0;
        for (int64_t g = 0; g < G; ++g) {
            issue();               // into the slot this thread emptied at g - 1
            cp_async_wait(la);     // this thread's copies for K-block g have landed
            __syncwarp();          // (and the warp's positions of the tile's rows)
            float cur[16];
            conv_read<VEC, PP>(rawr + (size_t)rslot * CT_RAW_SLOT, warp, lane, cur);
            tc::mbar_wait(&empty[s], ph ^ 1);
            conv_store<VEC, PP>(ring + s * CT_STAGE, warp, lane, cur);
            if (a.Xb) conv_store_bf16<VEC, PP>(a, tile, kb, warp, lane, cur, posr + (ti & 3) * CT_M);
            if (a.Xpad) conv_store_pad<VEC, PP>(a, tile, kb, warp, lane, cur);
            tc::fence_async_shared();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&full[s]);
            if (++kb == a.KB) { kb = 0; tile += tst; ++ti; }
            if (++rslot == a.raw) rslot = 0;
            if (++s == (uint32_t)a.stages) { s = 0; ph ^= 1; }
        }
    } else if (warp == 8) {
        {
            // ================= MMA issuer (lane 0); per-sub-dataset projections: the
            // warp reloads B = A_j^T when the tile's sub-dataset changes, after every
            // MMA issued so far has completed
            const uint32_t idesc = tc::umma_idesc(2, CT_M, N);
            uint32_t g = 0, t = 0, nb = 0;
            int curj = -1;
            int64_t tlo, thi;
            ct_range<PP>(a, tlo, thi);
            const int64_t tst = ct_step<PP>(a);
            for (int64_t tile = tlo; tile < thi; tile += tst, ++t) {
                if (PP) {
                    const int j = __ldg(a.ctiles + tile).x;
                    if (j != curj) {
                        if (t > 0) {
                            if (lane == 0) tc::mma_commit(bdone);
                            __syncwarp();
                            tc::mbar_wait(bdone, nb & 1);
                            ++nb;
                        }
                        load_B(a.Apad + (size_t)j * (a.d + 1) * N, lane, 32);
                        tc::fence_async_shared();
                        __syncwarp();
                        curj = j;
                    }
                }
                if (lane != 0) continue;
                const uint32_t acc = t & 1, tr = t >> 1;
                tc::mbar_wait(&tempty[acc], (tr & 1) ^ 1);
                tc::tc_fence_after();
                const uint32_t dt = tmem_base + acc * N;
                for (int kb = 0; kb < a.KB; ++kb, ++g) {
                    const uint32_t s = g % a.stages, ph = (g / a.stages) & 1;
                    tc::mbar_wait(&full[s], ph);
                    tc::tc_fence_after();
                    const uint32_t abig = tc::smem_u32(ring + s * CT_STAGE);
                    const uint32_t bb = tc::smem_u32(Bs + (size_t)kb * N * 128);
                    const int nk = min(4, (a.d - kb * CT_KB + 7) / 8);   // K = 8 per MMA
                    for (int kk = 0; kk < nk; ++kk)
                        tc::mma_tf32(dt, tc::umma_desc_sw128(abig + kk * 32),
                                     tc::umma_desc_sw128(bb + kk * 32), idesc, (kb | kk) != 0);
                    for (int kk = 0; kk < nk; ++kk)
                        tc::mma_tf32(dt, tc::umma_desc_sw128(abig + CT_A_BLK + kk * 32),
                                     tc::umma_desc_sw128(bb + kk * 32), idesc, 1);
                    tc::mma_commit(&empty[s]);
                }
                tc::mma_commit(&tfull[acc]);
            }
        }
        __syncwarp();
    } else {
        // ================= epilogue: thread <-> item row (TMEM lane)
        const int qd = warp & 3;
        const int row = qd * 32 + lane;
        const int W = N / 32;
        uint32_t t = 0;
        int64_t tlo, thi;
        ct_range<PP>(a, tlo, thi);
        const int64_t tst = ct_step<PP>(a);
        for (int64_t tile = tlo; tile < thi; tile += tst, ++t) {
            const uint32_t acc = t & 1, tr = t >> 1;
            int64_t i, pos = 0;
            ct_row<PP>(a, tile, row, i, pos);
            const bool valid = i >= 0;
            // A_d of the tile's projection
            const float *Adj = PP ? a.Apad + ((size_t)__ldg(a.ctiles + tile).x * (a.d + 1) + a.d) * N : Ad;
            float tt = 0.f;
            if (valid) {
                const double Vj = a.V[a.part[i]];
                if (Vj == 0.0) tt = 1.f;
                else {
                    const double df = Vj - a.norm2[i];
                    tt = (float)sqrt(df > 0.0 ? df : 0.0);
                }
                if (!PP) pos = a.pos_of_id[i];
            }
            tc::mbar_wait(&tfull[acc], tr & 1);
            tc::tc_fence_after();
            uint32_t words[4] = {0u, 0u, 0u, 0u};
            const uint32_t taddr = tmem_base + ((uint32_t)(qd * 32) << 16) + acc * N;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (c < W) {
                    uint32_t r[32];
                    tc::tmem_ld_32x32b_x32(taddr + c * 32, r);
                    tc::tmem_ld_wait();
                    uint32_t wd = 0u;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int b = c * 32 + j;
                        const float y = fmaf(Adj[b], tt, __uint_as_float(r[j]));
                        wd |= (uint32_t)(b < a.L && y >= 0.f) << j;
                    }
                    words[c] = wd;
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
            if (valid) {
                uint32_t *dst = a.codes + pos * W;
                if (W == 4) *reinterpret_cast<uint4 *>(dst) = make_uint4(words[0], words[1], words[2], words[3]);
                else if (W == 2) *reinterpret_cast<uint2 *>(dst) = make_uint2(words[0], words[1]);
                else dst[0] = words[0];
            }
        }
    }
    __syncthreads();
    if (warp == 8) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, tcols);
    }
}

// ---------------------------------------------------------------- TMA-fed variant
// (shared A, the default): the tile's rows are consecutive items, so its K-blocks
// come in by TMA instead of per-element cp.async (whose 64-bit address arithmetic
// made the cp.async kernel issue-bound: ~7.5K issue cycles per tile per SMSP).
//   d % 4 == 0: one 128-row box per K-block lands 128B-swizzled in the MMA stage
//     itself; the converters split it in place (big = top 11 bits) and write the
//     residual half next to it.
//   d % 4 != 0 (RAW): rows are not 16-byte aligned, so X is viewed as [n / G]
//     super-rows of G = 4 / gcd(d, 4) items (stride G d 4 bytes, a multiple of 16);
//     sub-row r of K-block kb is a box of 128 / G super-rows x 36 floats starting at
//     the 16-byte-aligned column r d - delta_r + 32 kb (delta_r = r d mod 4), landed
//     densely in a raw ring; the converters read item columns 32 kb .. +31 at offset
//     delta_r and write both halves into the swizzled MMA stage.
// Stage row r (128 / G) + s holds item tile 128 + s G + r.  Columns past d are zeroed
// by the converters; the last n % G items, outside the tensor map, are loaded by
// them directly.
//   warps 0-7   converters            warp 8   TMA producer (lane 0)
//   warp  9     TMEM + MMA issuer     warps 10-13 epilogue
// (CW converter warps: 8 or 16)
template <int CW> constexpr int cm_threads() { return (CW + 6) * 32; }

struct CodesTmaArgs {
    int64_t n, nfull, ntiles;   // nfull = G floor(n / G): items covered by the tensor map
    int d, KB, L, N, stages, rstages, G, m;
    const float *X;
    const double *norm2;
    const uint8_t *part;
    const double *V;
    const float *Apad;
    const int32_t *pos_of_id;
    uint32_t *codes;
    __nv_bfloat16 *Xb;
    int dpb;
};

template <int G>
__device__ __forceinline__ int64_t cm_item(int64_t tile, int row) {
    constexpr int R = CT_M / G;
    return tile * CT_M + (int64_t)(row % R) * G + row / R;
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

constexpr int CM_BW = 36;                            // RAW box width (floats)
constexpr int CM_RAW = CT_M * CM_BW * 4;             // 18 KB per raw stage

template <int G, int CW>
__global__ void __launch_bounds__(cm_threads<CW>(), 1)
    k3_codes_tma(const __grid_constant__ CUtensorMap tmx, CodesTmaArgs a) {
    constexpr int CT = CW * 32, CPT = 1024 / CT;   // converter threads, chunks per thread
    constexpr bool RAW = G > 1;
    constexpr int RG = CT_M / G;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    const int N = a.N, S = a.stages;
    const int SR = RAW ? a.rstages : S;
    uint8_t *ring = smem;                                          // S x (big 16 KB | small 16 KB)
    uint8_t *rawr = ring + (size_t)S * CT_STAGE;                   // RAW: SR x 128 rows x 36 floats
    uint8_t *Bs = rawr + (RAW ? (size_t)SR * CM_RAW : 0);          // KB x N x 128 B
    float *Ad = reinterpret_cast<float *>(Bs + (size_t)a.KB * N * 128);
    double *Vs = reinterpret_cast<double *>(Ad + N);               // [m]
    int32_t *posr = reinterpret_cast<int32_t *>(Vs + 256);         // [2][CT_M]
    uint64_t *bars = reinterpret_cast<uint64_t *>(posr + 2 * CT_M);
    uint64_t *full = bars, *empty = bars + S;
    uint64_t *rawfull = bars + 2 * S, *rawempty = rawfull + SR;   // (rawempty: RAW only)
    uint64_t *tfull = rawempty + SR, *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < a.KB * N * CT_KB; e += blockDim.x) {
        const int kb = e / (N * CT_KB), rem = e % (N * CT_KB);
        const int b = rem / CT_KB, k = rem % CT_KB;
        const int kg = kb * CT_KB + k;
        const float v = kg < a.d ? a.Apad[(size_t)kg * N + b] : 0.f;
        *reinterpret_cast<float *>(Bs + (size_t)kb * N * 128 + swz(b, k * 4)) = v;
    }
    for (int b = threadIdx.x; b < N; b += blockDim.x) Ad[b] = a.Apad[(size_t)a.d * N + b];
    for (int j = threadIdx.x; j < a.m; j += blockDim.x) Vs[j] = a.V[j];
    tc::fence_async_shared();
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            tc::mbar_init(&full[s], CW);
            tc::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < SR; ++s) {
            tc::mbar_init(&rawfull[s], 1);
            tc::mbar_init(&rawempty[s], CW);
        }
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&tfull[s], 1);
            tc::mbar_init(&tempty[s], 4);
        }
        tc::fence_mbar_init();
    }
    const uint32_t tcols = N <= 16 ? 32 : (2 * N <= 64 ? 64 : (2 * N <= 128 ? 128 : 256));
    if (warp == CW + 1) tc::tmem_alloc(tmem_slot, tcols);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp < CW) {
        // ================= converters: thread t owns 16-byte chunks t + 256 u of a stage
        const int t = threadIdx.x;
        auto load_pos = [&](int64_t tile) -> int32_t {
            const int64_t i = cm_item<G>(tile, t);
            return (tile < a.ntiles && i < a.n) ? __ldg(a.pos_of_id + i) : -1;
        };
        if (t < CT_M) posr[t] = load_pos(blockIdx.x);
        named_sync(1, CT);
        uint32_t s = 0, ph = 0, sr = 0, rph = 0;
        int ti = 0;
        for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++ti) {
            const int32_t pn = t < CT_M ? load_pos(tile + gridDim.x) : -1;   // next tile's, in flight
            const int32_t *pr = posr + (ti & 1) * CT_M;
            const bool tail = (tile + 1) * CT_M > a.nfull;   // (the last n % G items inside)
            for (int kb = 0; kb < a.KB; ++kb) {
                const bool edge = (kb + 1) * CT_KB > a.d;        // (columns past d inside)
                uint8_t *big = ring + (size_t)s * CT_STAGE;
                const float *raw = reinterpret_cast<const float *>(rawr + (size_t)sr * CM_RAW);
                tc::mbar_wait_sleep(&rawfull[sr], rph);
                if (RAW) tc::mbar_wait_sleep(&empty[s], ph ^ 1);
#pragma unroll
                for (int u = 0; u < CPT; ++u) {
                    const int c = t + CT * u;
                    const int row = c >> 3;
                    // in place: thread <-> physical chunk; RAW: thread <-> logical chunk
                    const int lc = RAW ? (c & 7) : ((c & 7) ^ (row & 7));
                    const int pc = RAW ? ((c & 7) ^ (row & 7)) : (c & 7);
                    const int col = kb * CT_KB + 4 * lc;
                    float v[4];
                    if (RAW) {
                        const int r = row / RG, dr = (r * a.d) & 3;
                        const float *q = raw + (size_t)row * CM_BW + dr + 4 * lc;
                        if ((dr & 1) == 0) {
                            const float2 x0 = *reinterpret_cast<const float2 *>(q);
                            const float2 x1 = *reinterpret_cast<const float2 *>(q + 2);
                            v[0] = x0.x; v[1] = x0.y; v[2] = x1.x; v[3] = x1.y;
                        } else {
#pragma unroll
                            for (int e = 0; e < 4; ++e) v[e] = q[e];
                        }
                    } else {
                        const uint4 w = *reinterpret_cast<const uint4 *>(big + 16 * c);
                        v[0] = __uint_as_float(w.x); v[1] = __uint_as_float(w.y);
                        v[2] = __uint_as_float(w.z); v[3] = __uint_as_float(w.w);
                    }
                    if (RAW && tail) {
                        const int64_t i = cm_item<G>(tile, row);
                        if (i >= a.nfull && i < a.n) {   // (the last n % G items: plain loads)
#pragma unroll
                            for (int e = 0; e < 4; ++e) v[e] = col + e < a.d ? __ldg(a.X + i * a.d + col + e) : 0.f;
                        }
                    }
                    if (edge) {
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            if (col + e >= a.d) v[e] = 0.f;
                    }
                    uint32_t bg[4], sm[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        bg[e] = __float_as_uint(v[e]) & 0xFFFFE000u;
                        sm[e] = __float_as_uint(v[e] - __uint_as_float(bg[e]));
                    }
                    const int off = 16 * (row * 8 + pc);
                    *reinterpret_cast<uint4 *>(big + off) = make_uint4(bg[0], bg[1], bg[2], bg[3]);
                    *reinterpret_cast<uint4 *>(big + CT_A_BLK + off) = make_uint4(sm[0], sm[1], sm[2], sm[3]);
                    const int32_t prow = pr[row];
                    if (a.Xb && prow >= 0 && col < a.dpb) {
                        const __nv_bfloat162 p0 = __floats2bfloat162_rn(v[0], v[1]);
                        const __nv_bfloat162 p1 = __floats2bfloat162_rn(v[2], v[3]);
                        uint2 q;
                        q.x = *reinterpret_cast<const uint32_t *>(&p0);
                        q.y = *reinterpret_cast<const uint32_t *>(&p1);
                        *reinterpret_cast<uint2 *>(a.Xb + (int64_t)prow * a.dpb + col) = q;
                    }
                }
                tc::fence_async_shared();
                __syncwarp();
                if (lane == 0) {
                    if (RAW) tc::mbar_arrive(&rawempty[sr]);
                    tc::mbar_arrive(&full[s]);
                }
                if (++s == (uint32_t)S) { s = 0; ph ^= 1; }
                if (RAW) { if (++sr == (uint32_t)SR) { sr = 0; rph ^= 1; } }
                else { sr = s; rph = ph; }
            }
            if (t < CT_M) posr[((ti + 1) & 1) * CT_M + t] = pn;
            named_sync(1, CT);
        }
    } else if (warp == CW) {
        // ================= TMA producer
        if (lane == 0) {
            tc::tma_prefetch(&tmx);
            uint32_t s = 0, ph = 0;
            for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
                for (int kb = 0; kb < a.KB; ++kb) {
                    if (RAW) {
                        tc::mbar_wait_sleep(&rawempty[s], ph ^ 1);
                        tc::mbar_arrive_expect_tx(&rawfull[s], CM_RAW);
                        uint8_t *dst = rawr + (size_t)s * CM_RAW;
                        for (int r = 0; r < G; ++r)
                            tc::tma_load_2d(dst + (size_t)r * RG * CM_BW * 4, &tmx, &rawfull[s],
                                            r * a.d - ((r * a.d) & 3) + kb * CT_KB, (int)(tile * RG));
                    } else {
                        tc::mbar_wait_sleep(&empty[s], ph ^ 1);
                        tc::mbar_arrive_expect_tx(&rawfull[s], CT_A_BLK);
                        tc::tma_load_2d(ring + (size_t)s * CT_STAGE, &tmx, &rawfull[s], kb * CT_KB, (int)tile * CT_M);
                    }
                    if (++s == (uint32_t)SR) { s = 0; ph ^= 1; }
                }
            }
        }
        __syncwarp();
    } else if (warp == CW + 1) {
        // ================= MMA issuer
        if (lane == 0) {
            const uint32_t idesc = tc::umma_idesc(2, CT_M, N);
            uint32_t s = 0, ph = 0, t = 0;
            for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++t) {
                const uint32_t acc = t & 1, tr = t >> 1;
                tc::mbar_wait_sleep(&tempty[acc], (tr & 1) ^ 1);
                tc::tc_fence_after();
                const uint32_t dt = tmem_base + acc * N;
                for (int kb = 0; kb < a.KB; ++kb) {
                    tc::mbar_wait_sleep(&full[s], ph);
                    tc::tc_fence_after();
                    const uint32_t abig = tc::smem_u32(ring + (size_t)s * CT_STAGE);
                    const uint32_t bb = tc::smem_u32(Bs + (size_t)kb * N * 128);
                    const int nk = min(4, (a.d - kb * CT_KB + 7) / 8);   // K = 8 per MMA
                    for (int kk = 0; kk < nk; ++kk)
                        tc::mma_tf32(dt, tc::umma_desc_sw128(abig + kk * 32), tc::umma_desc_sw128(bb + kk * 32),
                                     idesc, (kb | kk) != 0);
                    for (int kk = 0; kk < nk; ++kk)
                        tc::mma_tf32(dt, tc::umma_desc_sw128(abig + CT_A_BLK + kk * 32),
                                     tc::umma_desc_sw128(bb + kk * 32), idesc, 1);
                    tc::mma_commit(&empty[s]);
                    if (++s == (uint32_t)S) { s = 0; ph ^= 1; }
                }
                tc::mma_commit(&tfull[acc]);
            }
        }
        __syncwarp();
    } else {
        // ================= epilogue: thread <-> stage row (TMEM lane); the next tile's
        // sub-dataset, ||x||^2 and position are loaded while this tile's MMAs run
        const int qd = warp & 3;
        const int row = qd * 32 + lane;
        const int W = N / 32;
        auto fetch = [&](int64_t tile, int64_t &i, int &pj, double &nv, int32_t &pos) {
            i = cm_item<G>(tile, row);
            if (tile < a.ntiles && i < a.n) {
                pj = __ldg(a.part + i);
                nv = __ldg(a.norm2 + i);
                pos = __ldg(a.pos_of_id + i);
            } else {
                i = -1;
            }
        };
        int64_t ci;
        int cj = 0;
        double cn = 0.0;
        int32_t cp = 0;
        fetch(blockIdx.x, ci, cj, cn, cp);
        uint32_t t = 0;
        for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++t) {
            int64_t ni;
            int nj = 0;
            double nn = 0.0;
            int32_t np = 0;
            fetch(tile + gridDim.x, ni, nj, nn, np);
            const uint32_t acc = t & 1, tr = t >> 1;
            float tt = 0.f;
            if (ci >= 0) {
                const double Vj = Vs[cj];
                if (Vj == 0.0) tt = 1.f;
                else {
                    const double df = Vj - cn;
                    tt = (float)sqrt(df > 0.0 ? df : 0.0);
                }
            }
            tc::mbar_wait_sleep(&tfull[acc], tr & 1);
            tc::tc_fence_after();
            uint32_t words[4] = {0u, 0u, 0u, 0u};
            const uint32_t taddr = tmem_base + ((uint32_t)(qd * 32) << 16) + acc * N;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                if (c < W) {
                    uint32_t r[32];
                    tc::tmem_ld_32x32b_x32(taddr + c * 32, r);
                    tc::tmem_ld_wait();
                    uint32_t wd = 0u;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int b = c * 32 + j;
                        const float y = fmaf(Ad[b], tt, __uint_as_float(r[j]));
                        wd |= (uint32_t)(b < a.L && y >= 0.f) << j;
                    }
                    words[c] = wd;
                }
            }
            tc::tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&tempty[acc]);
            if (ci >= 0) {
                uint32_t *dst = a.codes + (int64_t)cp * W;
                if (W == 4) *reinterpret_cast<uint4 *>(dst) = make_uint4(words[0], words[1], words[2], words[3]);
                else if (W == 2) *reinterpret_cast<uint2 *>(dst) = make_uint2(words[0], words[1]);
                else dst[0] = words[0];
            }
            ci = ni; cj = nj; cn = nn; cp = np;
        }
    }
    __syncthreads();
    if (warp == CW + 1) {
        tc::tc_fence_after();
        tc::tmem_dealloc(tmem_base, tcols);
    }
}

// (rstages = 0: in place — the TMA barriers are per MMA stage)
static size_t codes_tma_smem(int KB, int N, int stages, int rstages) {
    return 1024 + (size_t)stages * CT_STAGE + (size_t)rstages * CM_RAW + (size_t)KB * N * 128 + (size_t)N * 4 +
           256 * 8 + 2 * CT_M * 4 + (2 * stages + 2 * (rstages ? rstages : stages) + 4) * 8 + 16;
}

bool make_tmap_2d(CUtensorMap *m, const void *base, CUtensorMapDataType dt, int esize, uint64_t cols,
                  uint64_t rows, uint32_t box_cols, uint32_t box_rows, int swizzle);

// the TMA-fed K3 (shared A); false: not applicable here (the caller takes the cp.async kernel)
static bool launch_codes_tma(const float *X, int64_t n, int d, const double *norm2, const uint8_t *part,
                             const double *V, int m, const float *Apad, int L, int W, const int32_t *pos_of_id,
                             uint32_t *codes, void *Xb, int dpb, cudaStream_t s) {
    if (getenv("NRLSH_CODES_CPASYNC") || ((uintptr_t)X & 15u) || m > 256) return false;
    const int G = d % 4 == 0 ? 1 : (d % 2 == 0 ? 2 : 4);
    const bool raw = G > 1;
    if (n < (int64_t)G * CT_M) return false;
    CodesTmaArgs a;
    a.n = n;
    a.nfull = n / G * G;
    a.ntiles = (n + CT_M - 1) / CT_M;
    a.d = d;
    a.KB = (d + CT_KB - 1) / CT_KB;
    a.L = L;
    a.N = 32 * W;
    a.G = G;
    a.m = m;
    a.X = X;
    a.norm2 = norm2;
    a.part = part;
    a.V = V;
    a.Apad = Apad;
    a.pos_of_id = pos_of_id;
    a.codes = codes;
    a.Xb = (__nv_bfloat16 *)Xb;
    a.dpb = dpb;
    // stages: in place, up to 6 MMA stages; RAW, 3 MMA stages and up to 4 raw ones
    int st = raw ? 3 : 6, rs = raw ? 4 : 0;
    if (getenv("NRLSH_CODES_STAGES")) {
        int x = 0, y = 0;
        if (sscanf(getenv("NRLSH_CODES_STAGES"), "%d,%d", &x, &y) >= 1) {
            st = std::max(2, std::min(8, x));
            if (raw && y > 0) rs = std::max(2, std::min(8, y));
        }
    }
    while (codes_tma_smem(a.KB, a.N, st, rs) > 227 * 1024) {
        if (raw && rs > 2 && rs >= st) --rs;
        else if (st > 2) --st;
        else if (raw && rs > 2) --rs;
        else return false;
    }
    a.stages = st;
    a.rstages = rs;
    CUtensorMap tm;
    if (raw ? !make_tmap_2d(&tm, X, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (uint64_t)G * d, (uint64_t)(n / G), CM_BW,
                            CT_M / G, 0)
            : !make_tmap_2d(&tm, X, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (uint64_t)d, (uint64_t)n, CT_KB, CT_M, 128))
        return false;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t sm = codes_tma_smem(a.KB, a.N, st, rs);
    const int grid = (int)std::min<int64_t>(sms, a.ntiles);
    const bool cw16 = !(getenv("NRLSH_CODES_CW") && atoi(getenv("NRLSH_CODES_CW")) == 8);
#define NR_CM(G_, CW_)                                                                                  \
    cudaFuncSetAttribute(k3_codes_tma<G_, CW_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);  \
    k3_codes_tma<G_, CW_><<<grid, cm_threads<CW_>(), sm, s>>>(tm, a)
    if (cw16) {
        if (G == 1) { NR_CM(1, 16); } else if (G == 2) { NR_CM(2, 16); } else { NR_CM(4, 16); }
    } else {
        if (G == 1) { NR_CM(1, 8); } else if (G == 2) { NR_CM(2, 8); } else { NR_CM(4, 8); }
    }
#undef NR_CM
    note_launch();
    return true;
}

static size_t codes_tc_smem(int KB, int N, int stages, int raw) {
    return 1024 + (size_t)stages * CT_STAGE + (size_t)raw * CT_RAW_SLOT + (size_t)KB * N * 128 +
           (size_t)N * 4 + (2 * stages + 4) * 8 + 32 + 4 * CT_M * 4 + 16;
}

// (MMA stages, raw slots): two MMA stages and up to 4 raw slots (48 KB of loads in
// flight per SM).  A third MMA stage measured slower (c4: 1.16 vs 0.85 ms) — the
// shared-memory carve-out it takes comes out of L1, which the cp.async loads and
// the row-copy stores go through.
static void codes_tc_config(int d, int N, int &stages, int &raw) {
    const int KB = (d + CT_KB - 1) / CT_KB;
    if (getenv("NRLSH_CODES_CFG")) {   // experiments: "stages,raw"
        int st = 0, rw = 0;
        if (sscanf(getenv("NRLSH_CODES_CFG"), "%d,%d", &st, &rw) == 2 && st >= 2 && rw >= 2 && rw <= 4 &&
            codes_tc_smem(KB, N, st, rw) <= 227 * 1024) { stages = st; raw = rw; return; }
    }
    const int opts[][2] = {{2, 4}, {2, 3}, {2, 2}};
    for (const auto &o : opts)
        if (codes_tc_smem(KB, N, o[0], o[1]) <= 227 * 1024) { stages = o[0]; raw = o[1]; return; }
    stages = raw = 0;
}

static int codes_tc_stages(int d, int N) {
    int st, raw;
    codes_tc_config(d, N, st, raw);
    return st;
}

bool codes_tc_supported(int d, int W) {
    return W != 3 && codes_tc_stages(d, 32 * W) > 0 && !getenv("NRLSH_CODES_SIMT");
}

void launch_item_codes_tc(const float *X, int64_t n, int d, const double *norm2,
                          const uint8_t *part, const double *V, const float *Apad, int L, int W,
                          const int32_t *pos_of_id, uint32_t *codes, void *Xb, int dpb,
                          float *Xpad, int dpad, cudaStream_t s, const int4 *ctiles, int nctiles,
                          const int32_t *perm, int m) {
    if (!ctiles && !Xpad && m > 0 &&
        launch_codes_tma(X, n, d, norm2, part, V, m, Apad, L, W, pos_of_id, codes, Xb, dpb, s))
        return;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    CodesArgs a;
    a.X = X;
    a.n = n;
    a.d = d;
    a.KB = (d + CT_KB - 1) / CT_KB;
    a.L = L;
    a.N = 32 * W;
    codes_tc_config(d, a.N, a.stages, a.raw);
    a.ctiles = ctiles;
    a.perm = perm;
    a.ntiles = ctiles ? nctiles : (n + CT_M - 1) / CT_M;
    a.norm2 = norm2;
    a.part = part;
    a.V = V;
    a.Apad = Apad;
    a.pos_of_id = pos_of_id;
    a.codes = codes;
    a.Xb = (__nv_bfloat16 *)Xb;
    a.dpb = dpb;
    a.Xpad = Xpad;
    a.dpad = dpad;
    const size_t sm = codes_tc_smem(a.KB, a.N, a.stages, a.raw);
    const int grid = (int)std::min<int64_t>(sms, a.ntiles);
    const int vec = (d % 4 == 0) ? 4 : ((d % 2 == 0) ? 2 : 1);
#define NR_CT(V, PP_)                                                                            \
    cudaFuncSetAttribute(k3_codes_tc<V, PP_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
    k3_codes_tc<V, PP_><<<grid, CT_THREADS, sm, s>>>(a)
    if (ctiles) {
        if (vec == 4) { NR_CT(4, true); } else if (vec == 2) { NR_CT(2, true); } else { NR_CT(1, true); }
    } else {
        if (vec == 4) { NR_CT(4, false); } else if (vec == 2) { NR_CT(2, false); } else { NR_CT(1, false); }
    }
#undef NR_CT
    note_launch();
}

}  // namespace nrlsh
