// scan_bs.cu — K6 (the batched Hamming scan + metric filter)
// bit-sliced, for codes of at most 64 bits.
//
// The popcount scan spends two POPC per (query, item) pair for 64-bit codes, and on
// sm_100a POPC issues through the MIO queue at a quarter of the ALU rate, shared with
// the scan's own shared-memory traffic.  Here a thread holds 32 items of one
// sub-dataset as 32W bit-planes (plane b = bit b of the 32 codes, one word), and per
// query:
//   * the XOR with the query's bit b is moved to the FMA pipe: for m in {0, -1},
//     x ^ m = x (2m + 1) + m  (one IMAD per plane);
//   * the 32W mismatch planes are summed by a Harley-Seal carry-save adder tree
//     (two LOP3 per full adder) into the bit-planes of h for all 32 items at once;
//   * the filter h <= delta_j(q) is the carry out of h + (255 - delta) in bit-sliced
//     form (one 3-input majority LOP3 per bit).
// So a (query, 32 items) step is ~32W IMAD + ~2.4 * 32W LOP3 on the two integer
// pipes instead of 32W POPC.  Passing pairs are appended exactly as the popcount scan
// appends them — staged per (CTA, query) as (h << 16 | offset), one warp reservation
// after a prefix sum of the lanes' pass counts, copied out as ((j, h) << 32 | position)
// — so the fallback and the select are shared.
//
// Layout: the index's codes transposed per group of 32 consecutive positions of one
// sub-dataset (a sub-dataset's last group is padded): plane-major, tplane[b][g], so a
// warp's 32 groups load one coalesced line per plane.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace nrlsh {

constexpr int kBsThreads = 128;                 // one group (32 items) per thread: 4096 items per CTA

// group g -> 32 consecutive codes (positions gpos[g] .. +31, past gend[g] zero)
template <int W>
__global__ void transpose_groups(const uint32_t *__restrict__ codes, const int2 *__restrict__ gdesc,
                                 int64_t G, uint32_t *__restrict__ planes) {
    const int lane = threadIdx.x & 31;
    for (int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; g < G;
         g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int2 gd = gdesc[g];   // (first position, items in the group)
        uint32_t c[W];
#pragma unroll
        for (int w = 0; w < W; ++w) c[w] = lane < gd.y ? codes[((int64_t)gd.x + lane) * W + w] : 0u;
#pragma unroll
        for (int w = 0; w < W; ++w)
#pragma unroll 8
            for (int b = 0; b < 32; ++b) {
                const uint32_t pl = __ballot_sync(NR_FULL, (c[w] >> b) & 1u);
                if (lane == b) planes[(int64_t)(32 * w + b) * G + g] = pl;
            }
    }
}

void launch_transpose_groups(const uint32_t *codes, const int2 *gdesc, int64_t G, int W, uint32_t *planes,
                             cudaStream_t s) {
    const int grid = (int)std::min<int64_t>(4096, (G * 32 + 255) / 256);
    if (W == 1) transpose_groups<1><<<grid, 256, 0, s>>>(codes, gdesc, G, planes);
    else transpose_groups<2><<<grid, 256, 0, s>>>(codes, gdesc, G, planes);
    note_launch();
}

// carry-save adder: (h, l) = (majority, parity) of (a, b, c)
__device__ __forceinline__ void csa(uint32_t &h, uint32_t &l, uint32_t a, uint32_t b, uint32_t c) {
    uint32_t hh, ll;
    asm("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(hh) : "r"(a), "r"(b), "r"(c));   // majority
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(ll) : "r"(a), "r"(b), "r"(c));   // parity
    h = hh;
    l = ll;
}

// 16 mismatch planes -> the running ones / twos / fours / eights planes, one sixteen
// out (Harley-Seal).  y[i] = x[i] ^ m[i] on the FMA pipe: x (2m + 1) + m.
__device__ __forceinline__ uint32_t xr(uint32_t x, uint32_t m, uint32_t m1) {
    uint32_t r;   // (m1 = 2m + 1, precomputed: the product stays an IMAD on the FMA pipe)
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(m1), "r"(m));
    return r;
}

// per sub-batch: the queries' plane masks (m, 2m + 1) for m = -(bit b of the code),
// qm[q][2 NB]; and delta transposed, deltaT[j][q]
template <int NB>
__global__ void bs_query_masks(const uint32_t *__restrict__ qcodes, int Qb, uint32_t *__restrict__ qm) {
    constexpr int W = NB / 32;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)Qb * NB;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = e / NB;
        const int b = (int)(e % NB);
        const uint32_t mk = 0u - ((qcodes[q * W + (b >> 5)] >> (b & 31)) & 1u);
        qm[q * 2 * NB + 2 * b] = mk;
        qm[q * 2 * NB + 2 * b + 1] = 2u * mk + 1u;
    }
}

__global__ void bs_delta_t(const int8_t *__restrict__ delta, int Qb, int m, int8_t *__restrict__ dt) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)Qb * m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = e / Qb, q = e % Qb;
        dt[e] = delta[q * m + j];
    }
}

// CTA = (chunk of 128 groups = 4096 positions of one sub-dataset, slice of the
// sub-batch's queries).  The chunk's planes are loaded once into registers and reused
// for every active query of the slice; the queries' masks are staged through shared
// memory in batches of kBsQB (double-buffered: the next batch's global loads are in
// flight while the current batch is computed).  Appends: one global reservation per
// (warp, query) after a warp prefix sum, entries written straight to the buffer.
constexpr int kBsQB = 8;          // queries per staged mask batch
constexpr int kBsQS = 256;        // queries per CTA slice
template <int NB>
__global__ void __launch_bounds__(kBsThreads, 4) k6_scan_bs(
    const uint32_t *__restrict__ planes, int64_t G, const int4 *__restrict__ chunks,
    const int64_t *__restrict__ offsets, const uint32_t *__restrict__ qmask,
    const int8_t *__restrict__ deltaT, int Qb, int nslice, int L, unsigned long long *__restrict__ buf,
    uint32_t *__restrict__ cnt, int64_t C, unsigned long long *__restrict__ pairs) {
    pdl_wait();
    constexpr int HB = NB == 64 ? 7 : 6;        // bit-planes of h (h <= NB)
    constexpr int MW = 2 * NB;                  // mask words per query
    constexpr int LPT = kBsQB * MW / kBsThreads;   // mask words each thread stages per batch
    static_assert(LPT % 4 == 0, "batch staging uses 16-byte loads");
    __shared__ __align__(16) uint32_t smk[2][kBsQB * MW];
    __shared__ int sq[kBsQS];
    __shared__ int sdl[kBsQS];
    __shared__ int s_nact;
    const int4 ch = chunks[blockIdx.x / nslice];   // (j, g0, g1, p0)
    const int slice = blockIdx.x % nslice;
    const int j = ch.x, g0 = ch.y, g1 = ch.z, p0 = ch.w;
    const int p1 = (int)offsets[j + 1];
    const int g = g0 + threadIdx.x;
    const bool has = g < g1;
    // this thread's 32 items (loads in flight during the compaction)
    uint32_t x[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) x[b] = has ? __ldg(planes + (int64_t)b * G + g) : 0u;
    const int lane = threadIdx.x & 31;
    // the slice's active queries (delta_j(q) >= 0), in ascending order
    const int qs0 = slice * kBsQS, qs1 = min(Qb, qs0 + kBsQS);
    if (threadIdx.x < 32) {
        int base = 0;
        for (int t0 = qs0; t0 < qs1; t0 += 32) {
            const int q = t0 + lane;
            const int dl = q < qs1 ? (int)deltaT[(int64_t)j * Qb + q] : -1;
            const unsigned bal = __ballot_sync(NR_FULL, dl >= 0);
            if (dl >= 0) {
                const int k = base + __popc(bal & lanemask_lt());
                sq[k] = q;
                sdl[k] = dl;
            }
            base += __popc(bal);
        }
        if (lane == 0) s_nact = base;
    }
    __syncthreads();
    const int nact = s_nact;
    if (nact == 0) return;
    const int pbase = p0 + 32 * (g - g0);          // position of item 0 of the group
    const int nv = has ? max(0, min(32, p1 - pbase)) : 0;
    const uint32_t vmask = nv >= 32 ? 0xFFFFFFFFu : ((1u << nv) - 1u);
    if (threadIdx.x == 0 && pairs)
        atomicAdd(pairs, (unsigned long long)nact * (unsigned long long)max(0, min(p1, p0 + 32 * (g1 - g0)) - p0));
    const unsigned long long jb = (unsigned long long)(j * (L + 1));
    const int nbatch = (nact + kBsQB - 1) / kBsQB;
    // every CTA walks the batches from its own starting point, so the CTAs of a slice
    // do not all reserve on the same query's counter at once
    const int rot = (int)((blockIdx.x * 2654435761u) % (unsigned)nbatch);
    // stage the first batch
    uint4 stg[LPT / 4];
    auto load_batch = [&](int bt) {
        bt += rot;
        if (bt >= nbatch) bt -= nbatch;
#pragma unroll
        for (int u = 0; u < LPT / 4; ++u) {
            const int w = (threadIdx.x * (LPT / 4) + u) * 4;     // word of the batch
            const int qi = bt * kBsQB + w / MW;
            stg[u] = qi < nact ? *reinterpret_cast<const uint4 *>(qmask + (int64_t)sq[qi] * MW + (w % MW))
                               : make_uint4(0u, 0u, 0u, 0u);
        }
    };
    auto store_batch = [&](int buf_) {
#pragma unroll
        for (int u = 0; u < LPT / 4; ++u)
            *reinterpret_cast<uint4 *>(&smk[buf_][(threadIdx.x * (LPT / 4) + u) * 4]) = stg[u];
    };
    load_batch(0);
    store_batch(0);
    __syncthreads();
    for (int bt = 0; bt < nbatch; ++bt) {
        if (bt + 1 < nbatch) load_batch(bt + 1);   // (in flight during this batch)
        const int bb = bt + rot < nbatch ? bt + rot : bt + rot - nbatch;   // the batch's place
        const int nq = min(kBsQB, nact - bb * kBsQB);
        for (int qi = 0; qi < nq; ++qi) {
            const uint32_t *qm = smk[bt & 1] + qi * MW;
            const int ia = bb * kBsQB + qi;
            const int dl = sdl[ia];
            // Harley-Seal over the NB mismatch planes
            uint32_t ones = 0u, twos = 0u, fours = 0u, eights = 0u, s0 = 0u, s1 = 0u, s2 = 0u;
#pragma unroll
            for (int blk = 0; blk < NB / 16; ++blk) {
                uint32_t d[16];
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                    const uint4 mm = *reinterpret_cast<const uint4 *>(qm + 2 * (16 * blk + i));
                    d[i] = xr(x[16 * blk + i], mm.x, mm.y);
                    d[i + 1] = xr(x[16 * blk + i + 1], mm.z, mm.w);
                }
                uint32_t twosA, twosB, foursA, foursB, eightsA, eightsB, sixteens;
                csa(twosA, ones, ones, d[0], d[1]);
                csa(twosB, ones, ones, d[2], d[3]);
                csa(foursA, twos, twos, twosA, twosB);
                csa(twosA, ones, ones, d[4], d[5]);
                csa(twosB, ones, ones, d[6], d[7]);
                csa(foursB, twos, twos, twosA, twosB);
                csa(eightsA, fours, fours, foursA, foursB);
                csa(twosA, ones, ones, d[8], d[9]);
                csa(twosB, ones, ones, d[10], d[11]);
                csa(foursA, twos, twos, twosA, twosB);
                csa(twosA, ones, ones, d[12], d[13]);
                csa(twosB, ones, ones, d[14], d[15]);
                csa(foursB, twos, twos, twosA, twosB);
                csa(eightsB, fours, fours, foursA, foursB);
                csa(sixteens, eights, eights, eightsA, eightsB);
                const uint32_t c0 = s0 & sixteens;   // s2 s1 s0 += sixteens
                s0 ^= sixteens;
                const uint32_t c1 = s1 & c0;
                s1 ^= c0;
                s2 ^= c1;
            }
            // pass iff no carry out of h + (255 - delta) (bit 7 of 255 - delta is set)
            const uint32_t hp[7] = {ones, twos, fours, eights, s0, s1, s2};
            const uint32_t cval = (uint32_t)(255 - dl);
            uint32_t carry = hp[0] & (0u - (cval & 1u));
#pragma unroll
            for (int i = 1; i < HB; ++i) {
                const uint32_t cm = 0u - ((cval >> i) & 1u);
                uint32_t cc;
                asm("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(cc) : "r"(hp[i]), "r"(cm), "r"(carry));
                carry = cc;
            }
#pragma unroll
            for (int i = HB; i < 7; ++i) carry &= 0u - ((cval >> i) & 1u);   // (h has no bit i)
            const uint32_t mask = ~carry & vmask;
            if (!__any_sync(NR_FULL, mask != 0u)) continue;
            // warp prefix sum of the pass counts -> one global reservation per (warp, query)
            const int q = sq[ia];
            const int np = __popc(mask);
            int inc = np;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(NR_FULL, inc, o);
                if (lane >= o) inc += y;
            }
            uint32_t base = 0;
            if (lane == 31) base = atomicAdd(&cnt[q], (uint32_t)inc);
            base = __shfl_sync(NR_FULL, base, 31);
            uint32_t slot = base + inc - np;
            unsigned long long *bq = buf + (int64_t)q * C;
            uint32_t mk = mask;
            while (mk) {
                const int i = __ffs(mk) - 1;
                mk &= mk - 1;
                uint32_t h = 0;
#pragma unroll
                for (int k = 0; k < HB; ++k) h |= ((hp[k] >> i) & 1u) << k;
                if (slot < C) bq[slot] = ((jb + h) << 32) | (uint32_t)(pbase + i);
                ++slot;
            }
        }
        if (bt + 1 < nbatch) {
            __syncthreads();   // (everyone is done with buffer (bt + 1) & 1's previous batch)
            store_batch((bt + 1) & 1);
            __syncthreads();
        }
    }
}

int scan_bs_groups_per_chunk() { return kBsThreads; }

// Opt-in (NRLSH_SCAN_BS=1 at build and query; shared projection, L <= 64): exact and
// parity-tested, but measured slower than the popcount scan on c4 (9.4 vs 5.5 ms per
// 10,000 queries at 64 bits; an earlier 32-query-group variant reached 6.0 / 3.7 ms at
// 64 / 32 bits): the tree itself is ~250 instructions per 1024 pairs, but the per-entry
// work (h rebuilt from 7 planes, divergent over the lanes) and the imbalance between
// chunks of high- and low-norm sub-datasets (ncu: 16% achieved occupancy) dominate.
bool scan_bs_supported(const nrlsh_index *ix) {
    if (!ix->bs_planes || ix->L > 64 || ix->QM != 1) return false;
    const char *e = getenv("NRLSH_SCAN_BS");
    return e && atoi(e) != 0;
}

void launch_scan_bs(const nrlsh_index *ix, const uint32_t *qcodes, const int8_t *delta, int Qb,
                    unsigned long long *buf, uint32_t *cnt, int64_t C, unsigned long long *pairs,
                    cudaStream_t s, void *ws) {
    const int NB = 32 * ix->W;
    uint32_t *qm = reinterpret_cast<uint32_t *>(ws);
    int8_t *dt = reinterpret_cast<int8_t *>(qm + (size_t)Qb * 2 * NB);
    const int nslice = (Qb + kBsQS - 1) / kBsQS;
    const unsigned grid = (unsigned)(ix->bs_nchunks * nslice);
    bs_delta_t<<<grid_for((int64_t)Qb * ix->m, 256, 2048), 256, 0, s>>>(delta, Qb, ix->m, dt);
    if (ix->W == 1) {
        bs_query_masks<32><<<grid_for((int64_t)Qb * 32, 256, 2048), 256, 0, s>>>(qcodes, Qb, qm);
        launch_pdl(k6_scan_bs<32>, dim3(grid), dim3(kBsThreads), 0, s, ix->bs_planes, ix->bs_G, ix->bs_chunks,
                   ix->offsets_d, qm, dt, Qb, nslice, ix->L, buf, cnt, C, pairs);
    } else {
        bs_query_masks<64><<<grid_for((int64_t)Qb * 64, 256, 2048), 256, 0, s>>>(qcodes, Qb, qm);
        launch_pdl(k6_scan_bs<64>, dim3(grid), dim3(kBsThreads), 0, s, ix->bs_planes, ix->bs_G, ix->bs_chunks,
                   ix->offsets_d, qm, dt, Qb, nslice, ix->L, buf, cnt, C, pairs);
    }
    note_launch(3);
}

size_t scan_bs_ws_bytes(const nrlsh_index *ix, int Qb) {
    return (size_t)Qb * 2 * 32 * ix->W * 4 + (size_t)Qb * ix->m + 256;
}

}  // namespace nrlsh
