// query_kernels.cu — batched query processing (Alg. 2 + single-table multi-probe,
// PAPER:160-171, 207-217) for sm_100a.
//
//  K5  qcodes:   bit b of P(q) = [q; 0] is [sum_k A[k][b] q_k >= 0]  (Eq. (8), Eq. (4)).
//  K6  pilot:    per query, the (j, h) histogram of a strided item sample gives a
//                bound B(q) on the position in the sorted (U_j, l) structure
//                 holding ~T items; it becomes per-sub-dataset Hamming
//                radii delta_j(q) = max{h : R[j][h] <= B(q)}.
//      scan:     every (query, item) pair: h = popc(code ^ qcode); keep (R, pos)
//                iff h <= delta_j(q) — one compare per pair, j uniform per chunk.
//      fallback: exact two-pass path for any query whose buffer under- or
//                overflowed.
//  K7  select:   the exact T smallest keys (R[j][h], position) per query — the
//                first T items of the traversal; positions within a sub-dataset
//                follow ascending item id, so this is the (R, id) order of D10.
//  K8  re-rank:  exact fp32 inner products of the candidates (Alg. 2 l.6,
//                PAPER:169) and top-k by (score desc, id asc).
#include <algorithm>
#include <climits>

#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"

namespace nrlsh {

// =========================================================================== K5
template <int W>
__global__ void __launch_bounds__(32 * W) k5_qcodes(const float *__restrict__ Q, int d,
                                                    const float *__restrict__ Apad, int L,
                                                    uint32_t *__restrict__ qcodes,
                                                    int *__restrict__ flags, int64_t qbase) {
    pdl_wait();
    extern __shared__ float sq[];
    const int64_t q = blockIdx.x;
    const float *qp = Q + q * (int64_t)d;
    int bad = 0, nz = 0;
    for (int k = threadIdx.x; k < d; k += blockDim.x) {
        const float v = qp[k];
        sq[k] = v;
        bad |= !isfinite(v);
        nz |= (v != 0.f);
    }
    const int anybad = __syncthreads_or(bad);
    const int anynz = __syncthreads_or(nz);
    if (threadIdx.x == 0) {
        if (anybad) atomicMin(&flags[1], (int)(qbase + q));
        else if (!anynz) atomicMin(&flags[0], (int)(qbase + q));
    }
    const int b = threadIdx.x;
    float acc = 0.f;
    for (int k = 0; k < d; ++k) acc = fmaf(__ldg(Apad + (int64_t)k * 32 * W + b), sq[k], acc);
    const bool bit = (b < L) && (acc >= 0.f);
    const unsigned word = __ballot_sync(NR_FULL, bit);
    if ((threadIdx.x & 31) == 0) qcodes[q * W + (threadIdx.x >> 5)] = word;
}

// Per-sub-dataset projections (reading Q4, NEXT-4): the code of q under
// every A_j, qcodes[(q QM + j) W + w].  CTA = (64 queries, sub-index j): k-chunks of
// A_j [64 x 32W] and of the queries [64 x 64] staged in shared memory; thread =
// (column b, a slice of the queries); sign bits packed by warp ballots (lanes are
// consecutive columns).  The j = 0 CTAs also flag zero / non-finite queries.
constexpr int kQpT = 64;   // queries per CTA
constexpr int kQpK = 32;   // k per staged chunk
template <int W>
__global__ void __launch_bounds__(256) k5_qcodes_pp(const float *__restrict__ Q, int64_t nq, int d,
                                                    const float *__restrict__ Apad, int L, int QM,
                                                    uint32_t *__restrict__ qcodes,
                                                    int *__restrict__ flags, int64_t qbase) {
    pdl_wait();
    constexpr int NC = 32 * W;                 // columns
    constexpr int QPT = kQpT * NC / 256;       // queries per thread
    __shared__ float As[kQpK][NC];
    __shared__ float Qs[kQpT][kQpK + 1];
    __shared__ int sbad[kQpT], snz[kQpT];
    const int j = blockIdx.y;
    const int64_t q0 = (int64_t)blockIdx.x * kQpT;
    const int col = threadIdx.x % NC, qs0 = (threadIdx.x / NC) * QPT;
    const float *Aj = Apad + (int64_t)j * (d + 1) * NC;
    if (threadIdx.x < kQpT) { sbad[threadIdx.x] = 0; snz[threadIdx.x] = 0; }
    float acc[QPT];
#pragma unroll
    for (int u = 0; u < QPT; ++u) acc[u] = 0.f;
    for (int k0 = 0; k0 < d; k0 += kQpK) {
        __syncthreads();
        for (int e = threadIdx.x; e < kQpK * NC; e += 256) {
            const int k = e / NC, b = e % NC;
            As[k][b] = k0 + k < d ? Aj[(int64_t)(k0 + k) * NC + b] : 0.f;
        }
        for (int e = threadIdx.x; e < kQpT * kQpK; e += 256) {
            const int qi = e / kQpK, k = e % kQpK;
            float v = 0.f;
            if (q0 + qi < nq && k0 + k < d) {
                v = Q[(q0 + qi) * d + k0 + k];
                if (j == 0) {
                    if (!isfinite(v)) sbad[qi] = 1;
                    if (v != 0.f) snz[qi] = 1;
                }
            }
            Qs[qi][k] = v;
        }
        __syncthreads();
        const int kn = min(kQpK, d - k0);
        for (int k = 0; k < kn; ++k) {   // k ascending: the fp32 FMA chain of k5_qcodes
            const float a = As[k][col];
#pragma unroll
            for (int u = 0; u < QPT; ++u) acc[u] = fmaf(a, Qs[qs0 + u][k], acc[u]);
        }
    }
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int u = 0; u < QPT; ++u) {
        const int64_t q = q0 + qs0 + u;
        const unsigned word = __ballot_sync(NR_FULL, col < L && acc[u] >= 0.f);
        if (lane == 0 && q < nq) qcodes[(q * QM + j) * W + col / 32] = word;
    }
    if (j == 0) {
        __syncthreads();
        if (threadIdx.x < kQpT && q0 + threadIdx.x < nq) {
            if (sbad[threadIdx.x]) atomicMin(&flags[1], (int)(qbase + q0 + threadIdx.x));
            else if (!snz[threadIdx.x]) atomicMin(&flags[0], (int)(qbase + q0 + threadIdx.x));
        }
    }
}

void launch_qcodes(const float *Q, int64_t nq, int d, const float *Apad, int L, int W,
                   uint32_t *qcodes, int *flags, int64_t qbase, cudaStream_t s, int QM) {
    if (QM > 1) {
        const dim3 grid((unsigned)((nq + kQpT - 1) / kQpT), (unsigned)QM);
        switch (W) {
            case 1: launch_pdl(k5_qcodes_pp<1>, grid, dim3(256), 0, s, Q, nq, d, Apad, L, QM, qcodes, flags, qbase); break;
            case 2: launch_pdl(k5_qcodes_pp<2>, grid, dim3(256), 0, s, Q, nq, d, Apad, L, QM, qcodes, flags, qbase); break;
            default: launch_pdl(k5_qcodes_pp<4>, grid, dim3(256), 0, s, Q, nq, d, Apad, L, QM, qcodes, flags, qbase); break;
        }
        note_launch();
        return;
    }
    const size_t sm = (size_t)d * 4;
    switch (W) {
        case 1: launch_pdl(k5_qcodes<1>, dim3((int)nq), dim3(32), sm, s, Q, d, Apad, L, qcodes, flags, qbase); break;
        case 2: launch_pdl(k5_qcodes<2>, dim3((int)nq), dim3(64), sm, s, Q, d, Apad, L, qcodes, flags, qbase); break;
        default: launch_pdl(k5_qcodes<4>, dim3((int)nq), dim3(128), sm, s, Q, d, Apad, L, qcodes, flags, qbase); break;
    }
    note_launch();
}

// ------------------------------------------------------------------ helpers
template <int W>
__device__ __forceinline__ void load_code(const uint32_t *__restrict__ codes, int64_t p,
                                          uint32_t (&c)[W]) {
    if (W == 4) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(codes) + p);
        c[0] = v.x; c[1] = v.y; c[2] = v.z; c[3] = v.w;
    } else if (W == 2) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(codes) + p);
        c[0] = v.x; c[1] = v.y;
    } else {
#pragma unroll
        for (int w = 0; w < W; ++w) c[w] = __ldg(codes + p * W + w);
    }
}

// Hamming distance to a query code held in (shared) memory
template <int W>
__device__ __forceinline__ int hamming_at(const uint32_t (&c)[W], const uint32_t *q) {
    int h = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) h += __popc(c[w] ^ q[w]);
    return h;
}

// Histogram of (j, h) over the ns sample entries (codes[t], part[t]) into smem
// `hist` [m*(L+1)] (the sample is every position, or the index's compacted
// strided sample); then the smallest structure position r whose cumulative
// count reaches `need` (in histogram units).  Returns r (NR-1 if never reached)
// and the count strictly before r in *cum_lt.  Lanes holding the same bin add
// once (match_any), which turns most shared atomics of a warp into one.
template <int W, bool AGG = true>
__device__ void hist_and_bound(const uint32_t *__restrict__ codes,
                               const uint8_t *__restrict__ part, int64_t ns,
                               const uint32_t (&qc)[W], int L, int NR,
                               const int32_t *__restrict__ order, uint32_t *hist, uint32_t need,
                               uint32_t *ws, int *sB, uint32_t *sLt, int64_t per = 0,
                               int64_t ns_real = 0, const uint32_t *sqc = nullptr) {
    for (int e = threadIdx.x; e < NR; e += blockDim.x) hist[e] = 0u;
    if (threadIdx.x == 0) { *sB = NR - 1; *sLt = 0u; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    if (AGG) {
        for (int64_t b0 = 0; b0 < ns; b0 += blockDim.x) {
            const int64_t t = b0 + threadIdx.x;
            int bin = -1;
            if (t < ns) {
                uint32_t c[W];
                load_code<W>(codes, t, c);
                const int pj = (int)part[t];
                bin = pj * (L + 1) + (sqc ? hamming_at<W>(c, sqc + pj * W) : hamming<W>(c, qc));
            }
            const unsigned peers = __match_any_sync(NR_FULL, bin);
            if (bin >= 0 && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
        }
    } else {
        // (interleaved sample: slot s holds sample (s % 32) * per + s / 32 if that is
        // < ns_real — the 32 slots a warp reads come from positions ~n/32 apart.)  PU
        // slots' loads are issued before their atomics.
        const uint32_t per32 = (uint32_t)per, nsr = (uint32_t)ns_real;
        constexpr int PU = 4;
        for (int64_t b0 = 0; b0 < ns; b0 += PU * (int64_t)blockDim.x) {
            uint32_t c[PU][W];
            int pt[PU];
#pragma unroll
            for (int u = 0; u < PU; ++u) {
                const int64_t t = b0 + (int64_t)u * blockDim.x + threadIdx.x;
                pt[u] = -1;
                const uint32_t t32 = (uint32_t)t;
                if (t < ns && (t32 & 31u) * per32 + (t32 >> 5) < nsr) {
                    load_code<W>(codes, t, c[u]);
                    pt[u] = (int)part[t];
                }
            }
#pragma unroll
            for (int u = 0; u < PU; ++u)
                if (pt[u] >= 0)
                    atomicAdd(&hist[pt[u] * (L + 1) +
                                    (sqc ? hamming_at<W>(c[u], sqc + pt[u] * W) : hamming<W>(c[u], qc))],
                              1u);
        }
    }
    __syncthreads();
    const int seg = (NR + blockDim.x - 1) / blockDim.x;
    const int r0 = threadIdx.x * seg, r1 = min(NR, r0 + seg);
    uint32_t loc = 0;
    for (int r = r0; r < r1; ++r) loc += hist[order[r]];
    uint32_t tot;
    const uint32_t ex = block_excl_scan(loc, ws, &tot);
    if (ex < need && ex + loc >= need) {
        uint32_t c = ex;
        for (int r = r0; r < r1; ++r) {
            const uint32_t hr = hist[order[r]];
            if (c + hr >= need) { *sB = r; *sLt = c; break; }
            c += hr;
        }
    } else if (threadIdx.x == 0 && tot < need) {
        *sLt = tot;  // bound never reached: everything qualifies
    }
    __syncthreads();
}

// ------------------------------------------------------------------ pilot sample
template <int W>
__global__ void gather_sample(const uint32_t *__restrict__ codes, const uint8_t *__restrict__ part,
                              int64_t ns, int stride, uint32_t *__restrict__ sc,
                              uint8_t *__restrict__ sp) {
    // sample t (position t * stride, t < ns) goes to slot (t % per) * 32 + t / per,
    // per = ceil(ns / 32): slot s then holds sample (s % 32) * per + s / 32, so the 32
    // slots a warp reads together come from positions ~n/32 apart
    const int64_t per = (ns + 31) / 32;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ns;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = t * stride;
        const int64_t slot = (t % per) * 32 + t / per;
#pragma unroll
        for (int w = 0; w < W; ++w) sc[slot * W + w] = codes[p * W + w];
        sp[slot] = part[p];
    }
}

void launch_gather_sample(const nrlsh_index *ix, int stride, uint32_t *sc, uint8_t *sp,
                          cudaStream_t s) {
    const int64_t ns = (ix->n + stride - 1) / stride;
    const int grid = grid_for(ns, 256, 1024);
    switch (ix->W) {
        case 1: gather_sample<1><<<grid, 256, 0, s>>>(ix->codes, ix->part_of_pos, ns, stride, sc, sp); break;
        case 2: gather_sample<2><<<grid, 256, 0, s>>>(ix->codes, ix->part_of_pos, ns, stride, sc, sp); break;
        default: gather_sample<4><<<grid, 256, 0, s>>>(ix->codes, ix->part_of_pos, ns, stride, sc, sp); break;
    }
    note_launch();
}

// =========================================================================== K6 pilot
template <int W>
__global__ void __launch_bounds__(1024) k6_pilot(
    const uint32_t *__restrict__ codes, const uint8_t *__restrict__ part_of_pos, int64_t n,
    const uint32_t *__restrict__ qcodes, int L, int m,
    const int32_t *__restrict__ order, const uint16_t *__restrict__ R, uint32_t need,
    int8_t *__restrict__ delta, uint32_t *__restrict__ cnt, int interleaved, int64_t ns_real,
    int QM, uint32_t *__restrict__ zero_word) {
    pdl_wait();
    extern __shared__ uint32_t hist[];   // [NR] (+ [QM x W] query codes, per-sub-dataset A_j)
    __shared__ uint32_t ws[32];
    __shared__ int sB;
    __shared__ uint32_t sLt;
    const int q = blockIdx.x;
    const int NR = m * (L + 1);
    uint32_t qc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) qc[w] = qcodes[(int64_t)q * QM * W + w];
    uint32_t *sqc = nullptr;
    if (QM > 1) {
        sqc = hist + NR;
        for (int e = threadIdx.x; e < QM * W; e += blockDim.x) sqc[e] = qcodes[(int64_t)q * QM * W + e];
    }
    // the compacted sample is stored interleaved (neighbouring slots from distant
    // sub-datasets), so a warp's bins rarely collide and plain shared atomics beat
    // the match_any aggregation the full-data fallback needs
    if (interleaved)
        hist_and_bound<W, false>(codes, part_of_pos, n, qc, L, NR, order, hist, need, ws, &sB, &sLt,
                                 n / 32, ns_real, sqc);
    else hist_and_bound<W>(codes, part_of_pos, n, qc, L, NR, order, hist, need, ws, &sB, &sLt, 0, 0, sqc);
    const int B = sB;
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        int c = 0;
        for (int h = 0; h <= L; ++h) c += (R[j * (L + 1) + h] <= B);
        delta[q * m + j] = (int8_t)(c - 1);
    }
    if (threadIdx.x == 0) cnt[q] = 0u;
    // (the fallback's failed-query counter, zeroed here instead of by a memset node)
    if (zero_word && q == 0 && threadIdx.x == 0) *zero_word = 0u;
}

// The pilot for QP queries per CTA (shared projection, compacted interleaved sample):
// each sampled code and sub-dataset is loaded once for the QP queries, each with its
// own histogram of the structure's (j, h) cells in shared memory; the bound and radii
// then follow per query exactly as in k6_pilot.
template <int W, int QP>
__global__ void __launch_bounds__(1024) k6_pilot_mq(
    const uint32_t *__restrict__ codes, const uint8_t *__restrict__ part, int64_t ns, int Qb,
    const uint32_t *__restrict__ qcodes, int L, int m, const int32_t *__restrict__ order,
    const uint16_t *__restrict__ R, uint32_t need, int8_t *__restrict__ delta,
    uint32_t *__restrict__ cnt, int64_t ns_real, uint32_t *__restrict__ zero_word) {
    pdl_wait();
    extern __shared__ uint32_t hist[];   // [QP][NR]
    __shared__ uint32_t ws[32];
    __shared__ int sB[QP];
    __shared__ uint32_t sLt[QP];
    const int NR = m * (L + 1);
    const int q0 = blockIdx.x * QP;
    uint32_t qc[QP][W];
#pragma unroll
    for (int i = 0; i < QP; ++i)
#pragma unroll
        for (int w = 0; w < W; ++w) qc[i][w] = q0 + i < Qb ? qcodes[(int64_t)(q0 + i) * W + w] : 0u;
    for (int e = threadIdx.x; e < QP * NR; e += blockDim.x) hist[e] = 0u;
    if (threadIdx.x < QP) { sB[threadIdx.x] = NR - 1; sLt[threadIdx.x] = 0u; }
    __syncthreads();
    // (interleaved sample: slot s holds sample (s % 32) * per + s / 32 if that is
    // < ns_real; two slots' loads are issued before their atomics)
    const uint32_t per32 = (uint32_t)(ns / 32), nsr = (uint32_t)ns_real;
    constexpr int PU = 2;
    for (int64_t b0 = 0; b0 < ns; b0 += PU * (int64_t)blockDim.x) {
        uint32_t c[PU][W];
        int pt[PU];
#pragma unroll
        for (int u = 0; u < PU; ++u) {
            const int64_t t = b0 + (int64_t)u * blockDim.x + threadIdx.x;
            pt[u] = -1;
            const uint32_t t32 = (uint32_t)t;
            if (t < ns && (t32 & 31u) * per32 + (t32 >> 5) < nsr) {
                load_code<W>(codes, t, c[u]);
                pt[u] = (int)part[t];
            }
        }
#pragma unroll
        for (int u = 0; u < PU; ++u) {
            if (pt[u] < 0) continue;
            const int base = pt[u] * (L + 1);
#pragma unroll
            for (int i = 0; i < QP; ++i) atomicAdd(&hist[i * NR + base + hamming<W>(c[u], qc[i])], 1u);
        }
    }
    __syncthreads();
    const int seg = (NR + blockDim.x - 1) / blockDim.x;
    const int r0 = threadIdx.x * seg, r1 = min(NR, r0 + seg);
    for (int i = 0; i < QP; ++i) {
        const uint32_t *h = hist + i * NR;
        uint32_t loc = 0;
        for (int r = r0; r < r1; ++r) loc += h[order[r]];
        uint32_t tot;
        const uint32_t ex = block_excl_scan(loc, ws, &tot);
        if (ex < need && ex + loc >= need) {
            uint32_t cc = ex;
            for (int r = r0; r < r1; ++r) {
                const uint32_t hr = h[order[r]];
                if (cc + hr >= need) { sB[i] = r; sLt[i] = cc; break; }
                cc += hr;
            }
        } else if (threadIdx.x == 0 && tot < need) {
            sLt[i] = tot;
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < QP * m; e += blockDim.x) {
        const int i = e / m, j = e - i * m;
        const int q = q0 + i;
        if (q >= Qb) continue;
        const int B = sB[i];
        int cj = 0;
        for (int hh = 0; hh <= L; ++hh) cj += (R[j * (L + 1) + hh] <= B);
        delta[(int64_t)q * m + j] = (int8_t)(cj - 1);
    }
    if (threadIdx.x < QP && q0 + threadIdx.x < Qb) cnt[q0 + threadIdx.x] = 0u;
    if (zero_word && blockIdx.x == 0 && threadIdx.x == 0) *zero_word = 0u;
}

void launch_pilot(const nrlsh_index *ix, const uint32_t *qcodes, int Qb, int64_t Tq, int stride,
                  int8_t *delta, uint32_t *cnt, cudaStream_t s, uint32_t *zero_word) {
    // target: T plus 4 standard deviations of the sampled estimate (+ one stride of
    // discreteness); exact (= T) when stride == 1.
    double target = (double)Tq;
    if (stride > 1) target += 4.0 * sqrt((double)Tq * stride) + stride;
    uint32_t need = (uint32_t)ceil(target / stride);
    // a few sampled items make a noisy bound: with T tiny the sampled count at the
    // bound is a handful and a query now and then under-shoots into the (slow) exact
    // fallback; 16 sampled items keep that rare at little extra scan cost
    if (stride > 1 && need < 16) need = 16;
    if (need < 1) need = 1;
    const int NR = ix->m * (ix->L + 1);
    const size_t sm = (size_t)NR * 4 + (ix->QM > 1 ? (size_t)ix->QM * ix->W * 4 : 0);
    const int32_t *order = ix->order_d;
    // the strided sample p = t * stride, compacted at build time (or every position)
    const bool cmp = stride > 1 && ix->samp_codes;
    const uint32_t *sc = cmp ? ix->samp_codes : ix->codes;
    const uint8_t *sp = cmp ? ix->samp_part : ix->part_of_pos;
    const int64_t ns = cmp ? ix->nsamp : ix->n;
    // QP queries per CTA when their histograms fit (shared projection, compacted
    // sample): c4 0.673 -> 0.614 ms per step with 2 (0.617 with 4); NRLSH_PILOT_QP
    // overrides (1: the one-query kernel)
    int QP = 2;
    if (getenv("NRLSH_PILOT_QP")) QP = atoi(getenv("NRLSH_PILOT_QP"));
    while (QP > 1 && (size_t)QP * NR * 4 > 200 * 1024) QP >>= 1;
    if (cmp && ix->QM == 1 && QP > 1) {
        const size_t smq = (size_t)QP * NR * 4;
        const int64_t nsr = (ix->n + stride - 1) / stride;
        const dim3 grid((unsigned)((Qb + QP - 1) / QP));
#define NR_PMQ(W_, QP_)                                                                                      \
        cudaFuncSetAttribute(k6_pilot_mq<W_, QP_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smq); \
        launch_pdl(k6_pilot_mq<W_, QP_>, grid, dim3(1024), smq, s, sc, sp, ns, Qb, qcodes, ix->L, ix->m,   \
                   order, ix->R_d, need, delta, cnt, nsr, zero_word)
        if (QP >= 4) {
            if (ix->W == 1) { NR_PMQ(1, 4); } else if (ix->W == 2) { NR_PMQ(2, 4); } else { NR_PMQ(4, 4); }
        } else {
            if (ix->W == 1) { NR_PMQ(1, 2); } else if (ix->W == 2) { NR_PMQ(2, 2); } else { NR_PMQ(4, 2); }
        }
#undef NR_PMQ
        note_launch();
        return;
    }
    switch (ix->W) {
        case 1:
            cudaFuncSetAttribute(k6_pilot<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            launch_pdl(k6_pilot<1>, dim3(Qb), dim3(1024), sm, s, sc, sp, ns, qcodes, ix->L, ix->m, order, ix->R_d, need, delta, cnt, cmp, (ix->n + stride - 1) / stride, ix->QM, zero_word);
            break;
        case 2:
            cudaFuncSetAttribute(k6_pilot<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            launch_pdl(k6_pilot<2>, dim3(Qb), dim3(1024), sm, s, sc, sp, ns, qcodes, ix->L, ix->m, order, ix->R_d, need, delta, cnt, cmp, (ix->n + stride - 1) / stride, ix->QM, zero_word);
            break;
        default:
            cudaFuncSetAttribute(k6_pilot<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            launch_pdl(k6_pilot<4>, dim3(Qb), dim3(1024), sm, s, sc, sp, ns, qcodes, ix->L, ix->m, order, ix->R_d, need, delta, cnt, cmp, (ix->n + stride - 1) / stride, ix->QM, zero_word);
            break;
    }
    note_launch();
}

// inclusive warp prefix sum: five shuffles whose in-range predicate guards the add
__device__ __forceinline__ uint32_t warp_scan_incl(uint32_t v) {
    asm volatile(
        "{\n\t.reg .u32 r;\n\t.reg .pred p;\n\t"
        "shfl.sync.up.b32 r|p, %0, 1, 0, 0xffffffff;\n\t@p add.u32 %0, %0, r;\n\t"
        "shfl.sync.up.b32 r|p, %0, 2, 0, 0xffffffff;\n\t@p add.u32 %0, %0, r;\n\t"
        "shfl.sync.up.b32 r|p, %0, 4, 0, 0xffffffff;\n\t@p add.u32 %0, %0, r;\n\t"
        "shfl.sync.up.b32 r|p, %0, 8, 0, 0xffffffff;\n\t@p add.u32 %0, %0, r;\n\t"
        "shfl.sync.up.b32 r|p, %0, 16, 0, 0xffffffff;\n\t@p add.u32 %0, %0, r;\n\t}"
        : "+r"(v));
    return v;
}
// atomics by inline PTX (ptxas still aggregates them per warp at SASS level: a
// direct ATOMS unless all 32 lanes are active, a shuffle-scan + one atomic then)
__device__ __forceinline__ uint32_t atom_add_shared(uint32_t *p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                 : "=r"(old) : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ uint32_t atom_add_global(uint32_t *p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// A lane's run of a dense cell: for each set bit u of mask, *p++ = (hib - dd[u]) << 32 |
// (lob + 256 u).  Inline PTX, five instructions per item (bit test, two value adds, a
// predicated store, a predicated 32-bit address add): the compiler's predicated 64-bit
// pointer increments cost ~11.  The run (<= 64 bytes) must not cross a 4 GB boundary
// (the caller checks), so only the low address word moves.
__device__ __forceinline__ void emit_run8(uint32_t mask, unsigned long long *p, uint32_t lob,
                                          uint32_t hib, const int *dd) {
    asm volatile(
        "{\n\t.reg .pred q;\n\t.reg .u32 lo, hi, t, vl, vh;\n\t.reg .u64 a;\n\t"
        "mov.b64 {lo, hi}, %1;\n\t"
#define NR_EMIT(U, BIT, OFF)                                                         \
        "and.b32 t, %0, " BIT ";\n\tsetp.ne.u32 q, t, 0;\n\t"                        \
        "add.u32 vl, %2, " OFF ";\n\tsub.u32 vh, %3, " U ";\n\t"                     \
        "mov.b64 a, {lo, hi};\n\t@q st.global.v2.u32 [a], {vl, vh};\n\t"           \
        "@q add.u32 lo, lo, 8;\n\t"
        NR_EMIT("%4", "1", "0") NR_EMIT("%5", "2", "256") NR_EMIT("%6", "4", "512")
        NR_EMIT("%7", "8", "768") NR_EMIT("%8", "16", "1024") NR_EMIT("%9", "32", "1280")
        NR_EMIT("%10", "64", "1536") NR_EMIT("%11", "128", "1792")
#undef NR_EMIT
        "}"
        :: "r"(mask), "l"(p), "r"(lob), "r"(hib), "r"(dd[0]), "r"(dd[1]), "r"(dd[2]), "r"(dd[3]),
           "r"(dd[4]), "r"(dd[5]), "r"(dd[6]), "r"(dd[7])
        : "memory");
}

// =========================================================================== K6 scan
constexpr int kScanThreads = 256;
// items per thread (a work unit = one CTA's chunk of 256 x IPT positions of one
// sub-dataset), queries per CTA, staged appends per (CTA, query)
#ifndef NRLSH_SCAN_IPT
#define NRLSH_SCAN_IPT 8
#endif
constexpr int kScanIPT = NRLSH_SCAN_IPT;
constexpr int kChunk = kScanThreads * kScanIPT;   // items per work unit
#ifndef NRLSH_SCAN_QG
#define NRLSH_SCAN_QG (NRLSH_SCAN_IPT >= 16 ? 32 : 64)
#endif
#ifndef NRLSH_SCAN_SB
#define NRLSH_SCAN_SB (NRLSH_SCAN_IPT >= 16 ? 256 : 128)
#endif
constexpr int kQG = NRLSH_SCAN_QG;     // queries per CTA
constexpr int kSB = NRLSH_SCAN_SB;     // staged appends per (CTA, query)

// Appends, two regimes by the cell's radius delta_j(q) (warp-uniform):
//  - sparse cells (delta < `dense`): each passing lane reserves its own run in the
//    query's shared-memory stage of packed 4-byte entries (h << 16 | offset in chunk)
//    with one shared atomic (no warp prefix sum: the order of a row's entries is
//    free); the stage is copied out, expanded to (flat (j, h) << 32 | position), with
//    one global reservation per (CTA, query); a lane whose run passes the end of the
//    stage writes the rest straight to global;
//  - dense cells: a warp prefix sum of the lanes' pass counts, one global
//    reservation per warp, and lane-owned runs written straight to the query's row
//    with predicated stores (no per-entry branches).
// ncu (instructions executed per SASS line) showed the previous single path — a
// prefix sum, an aggregated shared atomic and eight branchy per-item bodies for
// every (warp, query) with a pass, 30% of the bodies spilling past the stage —
// issuing half of the kernel's instructions at 75% issue-slot use.
// The CTA's active queries (delta_j(q) >= 0) are packed as (code words, radius,
// index) records read with one 16-byte shared load per word pair, and a thread's
// pass bits are the sign bits of delta - h (funnel shifts).
#ifndef NRLSH_SCAN_MINB
#define NRLSH_SCAN_MINB 5
#endif
template <int W>
__global__ void __launch_bounds__(kScanThreads, W == 4 ? 4 : NRLSH_SCAN_MINB) k6_scan(
    const uint32_t *__restrict__ codes, const int4 *__restrict__ chunks,
    const uint32_t *__restrict__ qcodes, const int8_t *__restrict__ delta, int Qb, int m,
    const uint16_t *__restrict__ R, int L, unsigned long long *__restrict__ buf,
    uint32_t *__restrict__ cnt, int64_t C, unsigned long long *__restrict__ pairs, int QM,
    int lbmax, unsigned long long *__restrict__ lbc, int dense, uint32_t *__restrict__ uws,
    int lb0max, int all_units) {
    pdl_wait();
    constexpr int RW = W <= 2 ? 4 : 8;             // record words: codes, radius, query
    __shared__ uint32_t s_unit[2];
    __shared__ unsigned long long s_lb[3];   // (pairs a lower bound ran on / decided alone; 2 x POPCs)
    __shared__ __align__(16) uint32_t srec[kQG][RW];
    __shared__ uint32_t sbuf[kQG][kSB];
    __shared__ uint32_t scnt[kQG];
    __shared__ uint32_t sbase[kQG];
    // Persistent CTAs take the active (chunk, query group) units that scan_units listed
    // from a work counter (the next unit's index is fetched while this one runs); the
    // last CTA to finish resets the counters for the next launch on this workspace.
    const int ngroups = (Qb + kQG - 1) / kQG;
    // (all_units > 0: small problems skip the list — every (chunk, group) is a unit, an
    // inactive one costs a radius read and a barrier)
    const uint32_t nunits = all_units > 0 ? (uint32_t)all_units : uws[0];
    const uint32_t *units = uws + 4;
    if (threadIdx.x == 0) s_unit[0] = atomicAdd(&uws[1], 1u);
    __syncthreads();
    uint32_t ui = s_unit[0];
    for (int upar = 0; ui < nunits; upar ^= 1, ui = s_unit[upar]) {
    uint32_t nxt = 0;   // (stored after the main loop: the atomic's round trip stays off the path)
    if (threadIdx.x == 0) nxt = atomicAdd(&uws[1], 1u);
    const uint32_t unit = all_units > 0 ? ui : units[ui];
    const int4 ch = chunks[unit / (uint32_t)ngroups];
    const int j = ch.x, p0 = ch.y, p1 = ch.z;
    const int q0 = (int)(unit % (uint32_t)ngroups) * kQG;
    const int nqg = min(kQG, Qb - q0);
    // every warp reads the group's radii itself (kQG bytes, L1-resident after the first
    // warp), so it knows the active set without a barrier and issues its code loads
    // while warps 0..kQG/32-1 fetch and pack the active queries' records (one global
    // latency instead of a serial delta -> ballot -> qcodes chain per 32 queries)
    const int lane = threadIdx.x & 31;
    constexpr int NH = kQG / 32;
    int dlv[NH];
    unsigned bal[NH];
    int nact = 0;
#pragma unroll
    for (int h = 0; h < NH; ++h) {
        const int t = h * 32 + lane;
        dlv[h] = t < nqg ? radius_of(delta[(int64_t)(q0 + t) * m + j]) : -1;
        bal[h] = __ballot_sync(NR_FULL, dlv[h] >= 0);
        nact += __popc(bal[h]);
    }
    if (nact == 0) {   // (only without the list; uniform: every warp computed the same count)
        if (threadIdx.x == 0) s_unit[upar ^ 1] = nxt;
        __syncthreads();
        continue;
    }
    uint32_t c[kScanIPT][W];
    uint32_t vmask = 0;   // bit u: item u of this thread exists
#pragma unroll
    for (int u = 0; u < kScanIPT; ++u) {
        const int p = p0 + threadIdx.x + kScanThreads * u;
        if (p < p1) {
            load_code<W>(codes, p, c[u]);
            vmask |= 1u << u;
        } else {
#pragma unroll
            for (int w = 0; w < W; ++w) c[u][w] = 0u;
        }
    }
    {
        int base = 0;
#pragma unroll
        for (int h = 0; h < NH; ++h) {
            if ((int)(threadIdx.x >> 5) == h) {
                const int t = h * 32 + lane;
                scnt[t] = 0;
                if (dlv[h] >= 0) {
                    uint32_t *r = srec[base + __popc(bal[h] & lanemask_lt())];
#pragma unroll
                    for (int w = 0; w < W; ++w)   // (per-sub-dataset A_j: the code under A_j)
                        r[w] = qcodes[((int64_t)(q0 + t) * QM + (QM > 1 ? j : 0)) * W + w];
                    r[W] = (uint32_t)dlv[h];
                    r[W + 1] = (uint32_t)t;
                }
            }
            base += __popc(bal[h]);
        }
    }
    if (threadIdx.x == 0 && pairs) atomicAdd(pairs, (unsigned long long)nact * (p1 - p0));
    if (threadIdx.x == 0) { s_lb[0] = 0ull; s_lb[1] = 0ull; s_lb[2] = 0ull; }
    // (this warp's iterations: coarse bound ran / skipped, pair bound ran / skipped, exact)
    uint32_t l0t = 0, l0s = 0, lbt = 0, lbs = 0, ext = 0;
    __syncthreads();
    // (the record's shared address is carried in a register: the compiler otherwise
    // rebuilds it from the CTA's window base with five uniform instructions per query)
    uint32_t rec_a = (uint32_t)__cvta_generic_to_shared(&srec[0][0]);
    for (int ia = 0; ia < nact; ++ia, rec_a += RW * 4) {
        uint32_t rec[RW];
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(rec[0]), "=r"(rec[1]), "=r"(rec[2]), "=r"(rec[3]) : "r"(rec_a));
        if (RW == 8)
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4+16];"
                         : "=r"(rec[4]), "=r"(rec[5]), "=r"(rec[6]), "=r"(rec[7]) : "r"(rec_a));
        const int dl = (int)rec[W];
        const int qq = (int)rec[W + 1];
        uint32_t qc[W];
#pragma unroll
        for (int w = 0; w < W; ++w) qc[w] = rec[w];
        if (W >= 2 && dl <= lb0max) {
            // very small radius: a coarser bound at half the POPCs of the next one.
            // 128 bits: h >= popc(OR of the four XOR words), one POPC per item; 64 bits:
            // min(h_u, h_v) >= popc((a_u | b_u) & (a_v | b_v)), one POPC per two items
            // (an absent item's code 0 only weakens it).  On near-random codes a warp's
            // 256 items all exceed it with probability > 1/2 up to delta = 24 (Bin(32,
            // 15/16)) and 10 (Bin(32, 9/16)).
            int l0min = 255;
            if (W == 4) {
#pragma unroll
                for (int u = 0; u < kScanIPT; ++u)
                    l0min = min(l0min, __popc((c[u][0] ^ qc[0]) | (c[u][1] ^ qc[1]) |
                                              (c[u][2] ^ qc[2]) | (c[u][3] ^ qc[3])));
            } else {
#pragma unroll
                for (int u = 0; u + 1 < kScanIPT; u += 2)
                    l0min = min(l0min, __popc(((c[u][0] ^ qc[0]) | (c[u][1] ^ qc[1])) &
                                              ((c[u + 1][0] ^ qc[0]) | (c[u + 1][1] ^ qc[1]))));
            }
            l0t += 1;
            if (!__any_sync(NR_FULL, l0min <= dl)) { l0s += 1; continue; }
        }
        if (W >= 2 && dl <= lbmax) {
            // small radius: a one-POPC lower bound per word pair first,
            // h = popc(a) + popc(b) >= popc(a | b); where no item of the warp can pass,
            // the exact distances are skipped (on near-random codes, most warps at
            // delta <= 16 of 64 bits)
            int lbmin = 255;
#pragma unroll
            for (int u = 0; u < kScanIPT; ++u) {
                int lb = 0;
#pragma unroll
                for (int w = 0; w + 1 < W; w += 2) lb += __popc((c[u][w] ^ qc[w]) | (c[u][w + 1] ^ qc[w + 1]));
                lbmin = min(lbmin, lb);   // (an absent item, code 0, can only keep the exact path on)
            }
            lbt += 1;
            if (!__any_sync(NR_FULL, lbmin <= dl)) { lbs += 1; continue; }
        }
        // dd_u = delta - h_u in one three-input add per word pair (a pass is dd_u >= 0;
        // h_u = delta - dd_u is only needed for the entries written)
        ext += 1;
        int dd[kScanIPT];
        uint32_t fail = 0;   // bit u: h_u > delta (the sign of dd_u)
#pragma unroll
        for (int u = kScanIPT - 1; u >= 0; --u) {
            int t = dl;
#pragma unroll
            for (int w = 0; w < W; ++w) t -= __popc(c[u][w] ^ qc[w]);
            dd[u] = t;
            fail = __funnelshift_l((uint32_t)t, fail, 1);
        }
        const uint32_t mask = ~fail & vmask;
        if (!__any_sync(NR_FULL, mask != 0u)) continue;
        const uint32_t np = (uint32_t)__popc(mask);
        unsigned long long *row = buf + (int64_t)(q0 + qq) * C;
        const uint32_t jhd = (uint32_t)(j * (L + 1) + dl);            // + h_u = - dd_u
        const uint32_t hd16 = ((uint32_t)dl << 16) + threadIdx.x;     // stage entry: h << 16 | offset
        const uint32_t pt = (uint32_t)p0 + threadIdx.x;
        if (dl >= dense) {
            // dense cell (many of a warp's 256 items pass): lane-owned runs straight in
            // the query's candidate row, one global reservation per warp
            // (the warp total by one REDUX, so the reservation's round trip to L2 overlaps
            // the five-step prefix sum)
            const uint32_t tot = __reduce_add_sync(NR_FULL, np);
            uint32_t gb = 0;
            if (lane == 31) gb = atom_add_global(&cnt[q0 + qq], tot);
            const uint32_t inc = warp_scan_incl(np);
            gb = __shfl_sync(NR_FULL, gb, 31);
            unsigned long long *ptr = row + (gb + inc - np);
            if ((int64_t)gb + tot <= C) {
                bool done = false;
                if constexpr (kScanIPT == 8 && kScanThreads == 256) {
                    if ((uint32_t)reinterpret_cast<uintptr_t>(ptr) <= 0xffffffbfu) {
                        emit_run8(mask, ptr, pt, jhd, dd);
                        done = true;
                    }
                }
                if (!done) {
#pragma unroll
                    for (int u = 0; u < kScanIPT; ++u)
                        if (mask >> u & 1u)
                            *ptr++ = ((unsigned long long)(jhd - (uint32_t)dd[u]) << 32) | (pt + kScanThreads * u);
                }
            } else {   // the row is full (the query is redone with a larger buffer)
                const unsigned long long *end = row + C;
#pragma unroll
                for (int u = 0; u < kScanIPT; ++u)
                    if (mask >> u & 1u) {
                        if (ptr < end)
                            *ptr = ((unsigned long long)(jhd - (uint32_t)dd[u]) << 32) | (pt + kScanThreads * u);
                        ++ptr;
                    }
            }
        } else if (mask) {
            // sparse cell: each passing lane reserves its own run in the query's stage
            // (no warp prefix sum: the order of a row's entries is free)
            uint32_t slot = atom_add_shared(&scnt[qq], np);
            if (slot + np <= (uint32_t)kSB) {
                uint32_t *sp = &sbuf[qq][slot];
#pragma unroll
                for (int u = 0; u < kScanIPT; ++u)
                    if (mask >> u & 1u) *sp++ = hd16 - ((uint32_t)dd[u] << 16) + kScanThreads * u;
            } else {   // stage full: the part of this lane's run past it goes straight to global
                const uint32_t lo = max(slot, (uint32_t)kSB);
                uint32_t g = atom_add_global(&cnt[q0 + qq], slot + np - lo);
#pragma unroll
                for (int u = 0; u < kScanIPT; ++u)
                    if (mask >> u & 1u) {
                        if (slot < (uint32_t)kSB) {
                            sbuf[qq][slot] = hd16 - ((uint32_t)dd[u] << 16) + kScanThreads * u;
                        } else {
                            if (g < C)
                                row[g] = ((unsigned long long)(jhd - (uint32_t)dd[u]) << 32) | (pt + kScanThreads * u);
                            ++g;
                        }
                        ++slot;
                    }
            }
        }
    }
    if (lbc) {   // (per warp: iterations x its items; POPCs in halves: the coarse 64-bit bound is 1/2 per item)
        const uint32_t wv = __reduce_add_sync(NR_FULL, (uint32_t)__popc(vmask));
        if (lane == 0) {
            if (l0t | lbt) {
                // (a pair counts once in [0] even if both bounds ran on it)
                atomicAdd(&s_lb[0], (unsigned long long)(l0s + lbt) * wv);
                atomicAdd(&s_lb[1], (unsigned long long)(l0s + lbs) * wv);
            }
            atomicAdd(&s_lb[2], (unsigned long long)(l0t * (W == 4 ? 2u : 1u) + lbt * (uint32_t)W +
                                                     ext * 2u * (uint32_t)W) * wv);
        }
    }
    if (threadIdx.x == 0) s_unit[upar ^ 1] = nxt;
    __syncthreads();
    if (lbc && threadIdx.x == 0) {
        if (s_lb[0]) {
            atomicAdd(&lbc[0], s_lb[0]);
            atomicAdd(&lbc[1], s_lb[1]);
        }
        atomicAdd(&lbc[2], s_lb[2]);
    }
    for (int t = threadIdx.x; t < nqg; t += blockDim.x) {
        const uint32_t nst = min(scnt[t], (uint32_t)kSB);
        sbase[t] = nst ? atomicAdd(&cnt[q0 + t], nst) : 0u;
    }
    __syncthreads();
    // copy-out: warp w handles queries w, w+8, ...; lanes stride the staged entries
    // entry: (flat (j, h) index of the sorted structure << 32) | position; select maps
    // it to the structure position R[j][h]
    const int warp = threadIdx.x >> 5;
    const unsigned long long jb = (unsigned long long)(j * (L + 1));
    for (int t = warp; t < nqg; t += kScanThreads / 32) {
        const uint32_t nst = min(scnt[t], (uint32_t)kSB);
        const int64_t q = q0 + t;
        for (uint32_t e = lane; e < nst; e += 32) {
            const uint32_t g = sbase[t] + e;
            const uint32_t v = sbuf[t][e];
            if (g < C) buf[q * C + g] = ((jb + (v >> 16)) << 32) | (uint32_t)(p0 + (v & 0xffffu));
        }
    }
    __syncthreads();   // (the stage, the records and s_unit are reused by the next unit)
    }
    if (threadIdx.x == 0 && atomicAdd(&uws[2], 1u) == gridDim.x - 1) {
        uws[0] = 0u;
        uws[1] = 0u;
        uws[2] = 0u;
    }
}

// The active (chunk, query group) units of a sub-batch: a group is active on a
// sub-dataset iff one of its queries has a radius there (delta != -1).  One CTA per
// group; ws: [0] unit count, [1] work counter, [2] finished CTAs (all zero on entry,
// reset by the scan), [4...] units as chunk * ngroups + group.
__global__ void __launch_bounds__(1024) scan_units(const int8_t *__restrict__ delta, int Qb, int m,
                                                   const int4 *__restrict__ chunks, int nchunks,
                                                   uint32_t *__restrict__ ws) {
    pdl_wait();
    __shared__ uint8_t act[kMaxParts];
    const int g = blockIdx.x, ngroups = gridDim.x, q0 = g * kQG;
    const int nqg = min(kQG, Qb - q0);
    for (int j = threadIdx.x; j < m; j += blockDim.x) act[j] = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < nqg * m; e += blockDim.x)
        if (delta[(int64_t)q0 * m + e] != (int8_t)-1) act[e % m] = 1;   // (benign race: all write 1)
    __syncthreads();
    const int lane = threadIdx.x & 31;
    // (listed from the last chunk down: the sub-datasets of largest norm, which are active
    // for the most queries and hold the dense cells, start first and the cheap units
    // fill the tail of the persistent CTAs' schedule)
    for (int c0 = 0; c0 < nchunks; c0 += blockDim.x) {
        const int c = nchunks - 1 - (c0 + (int)threadIdx.x);
        const bool f = c >= 0 && act[chunks[c].x];
        const unsigned bal = __ballot_sync(NR_FULL, f);
        if (bal) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&ws[0], (uint32_t)__popc(bal));
            base = __shfl_sync(NR_FULL, base, 0);
            if (f) ws[4 + base + __popc(bal & lanemask_lt())] = (uint32_t)c * (uint32_t)ngroups + (uint32_t)g;
        }
    }
}

int scan_chunk_items() { return kChunk; }
size_t scan_units_ws_bytes(const nrlsh_index *ix, int Qmax) {
    return 16 + (size_t)ix->nchunks * (size_t)((Qmax + kQG - 1) / kQG) * 4;
}

// ---------------------------------------------------------------- K6 scan, queries in lanes

void launch_scan(const nrlsh_index *ix, const uint32_t *qcodes, const int8_t *delta, int Qb,
                 unsigned long long *buf, uint32_t *cnt, int64_t C, unsigned long long *pairs,
                 cudaStream_t s, unsigned long long *lbc, void *units_ws) {
    // radii up to which the pair lower bound runs first: where a warp's 256 near-random
    // codes all miss it with probability > 1/2 (Bin(32, 3/4) per word pair; 64 bits:
    // delta <= 16, 128 bits: delta <= 37); NRLSH_SCAN_LBMAX overrides (-1: off)
    int lbmax = ix->W == 2 ? 16 : (ix->W == 4 ? 37 : -1);
    if (getenv("NRLSH_SCAN_LBMAX")) lbmax = atoi(getenv("NRLSH_SCAN_LBMAX"));
    // ... and the coarser bound before it (NRLSH_SCAN_LB0MAX, -1: off)
    int lb0max = ix->W == 2 ? 10 : (ix->W == 4 ? 24 : -1);
    if (getenv("NRLSH_SCAN_LB0MAX")) lb0max = atoi(getenv("NRLSH_SCAN_LB0MAX"));
    lb0max = std::min(lb0max, lbmax);
    // radius from which a cell counts as dense (L/2 - 0.75 sqrt(L): ~8% of random codes
    // within it; measured optimum 26 at 64 bits, 56 at 128); its appends go straight to
    // global, the others through the stage
    int dense = (int)lround(ix->L / 2.0 - 0.75 * sqrt((double)ix->L));
    if (getenv("NRLSH_SCAN_DENSE")) dense = atoi(getenv("NRLSH_SCAN_DENSE"));
    const int ngroups = (Qb + kQG - 1) / kQG;
    uint32_t *uws = static_cast<uint32_t *>(units_ws);
    // one wave of resident CTAs (NRLSH_SCAN_WAVES: CTAs per resident slot, default 1)
    static int res[5] = {0, 0, 0, 0, 0};
    if (!res[ix->W]) {
        int r = 0;
        if (ix->W == 1) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k6_scan<1>, kScanThreads, 0);
        else if (ix->W == 2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k6_scan<2>, kScanThreads, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k6_scan<4>, kScanThreads, 0);
        res[ix->W] = std::max(1, r);
    }
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    static const int waves = getenv("NRLSH_SCAN_WAVES") ? std::max(1, atoi(getenv("NRLSH_SCAN_WAVES"))) : 1;
    const unsigned grid = (unsigned)std::min<int64_t>((int64_t)sms * res[ix->W] * waves,
                                                      (int64_t)ix->nchunks * ngroups);
    // at most two waves of units: not worth the list's launch (small indexes, a handful
    // of queries)
    const int64_t total = (int64_t)ix->nchunks * ngroups;
    const int all_units = total <= 2 * (int64_t)sms * res[ix->W] ? (int)total : 0;
    if (!all_units)
        launch_pdl(scan_units, dim3(ngroups), dim3(1024), 0, s, delta, Qb, ix->m, ix->chunks_d,
                   (int)ix->nchunks, uws);
    switch (ix->W) {
        case 1: launch_pdl(k6_scan<1>, dim3(grid), dim3(kScanThreads), 0, s, ix->codes, ix->chunks_d, qcodes, delta, Qb, ix->m, ix->R_d, ix->L, buf, cnt, C, pairs, ix->QM, lbmax, lbc, dense, uws, lb0max, all_units); break;
        case 2: launch_pdl(k6_scan<2>, dim3(grid), dim3(kScanThreads), 0, s, ix->codes, ix->chunks_d, qcodes, delta, Qb, ix->m, ix->R_d, ix->L, buf, cnt, C, pairs, ix->QM, lbmax, lbc, dense, uws, lb0max, all_units); break;
        default: launch_pdl(k6_scan<4>, dim3(grid), dim3(kScanThreads), 0, s, ix->codes, ix->chunks_d, qcodes, delta, Qb, ix->m, ix->R_d, ix->L, buf, cnt, C, pairs, ix->QM, lbmax, lbc, dense, uws, lb0max, all_units); break;
    }
    note_launch(all_units ? 1 : 2);
}


// =========================================================================== fallback
template <int W>
__global__ void __launch_bounds__(1024) k6_fallback(
    const uint32_t *__restrict__ codes, const uint8_t *__restrict__ part_of_pos, int64_t n,
    const uint32_t *__restrict__ qcodes, int L, int m, const int32_t *__restrict__ order,
    const uint16_t *__restrict__ R, int64_t Tq, unsigned long long *__restrict__ buf,
    uint32_t *__restrict__ cnt, const uint32_t *__restrict__ cntv, int64_t C,
    int *__restrict__ flags, int QM) {
    pdl_wait();
    extern __shared__ uint32_t hist[];   // [NR] (+ [QM x W] query codes)
    __shared__ uint32_t ws[32];
    __shared__ int sB;
    __shared__ uint32_t sLt, s_out, s_eq;
    const int q = blockIdx.x;
    const uint32_t c0 = cnt[q], cv = cntv[q];
    if (cv >= (uint64_t)Tq && c0 <= (uint64_t)C) return;
    if (threadIdx.x == 0 && flags) atomicAdd(&flags[2], 1);
    const int NR = m * (L + 1);
    uint32_t qc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) qc[w] = qcodes[(int64_t)q * QM * W + w];
    uint32_t *sqc = nullptr;
    if (QM > 1) {
        sqc = hist + NR;
        for (int e = threadIdx.x; e < QM * W; e += blockDim.x) sqc[e] = qcodes[(int64_t)q * QM * W + e];
    }
    hist_and_bound<W>(codes, part_of_pos, n, qc, L, NR, order, hist, (uint32_t)Tq, ws, &sB, &sLt, 0, 0,
                      sqc);
    const int B = sB;
    const uint32_t need_eq = (uint32_t)Tq - sLt;
    // R[j][h] lookup straight from the structure (global, cached)
    if (threadIdx.x == 0) { s_out = 0; s_eq = 0; }
    __syncthreads();
    for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t p = base + threadIdx.x;
        int r = NR, f = 0;
        if (p < n) {
            uint32_t c[W];
            load_code<W>(codes, p, c);
            const int pj = part_of_pos[p];
            f = pj * (L + 1) + (sqc ? hamming_at<W>(c, sqc + pj * W) : hamming<W>(c, qc));
            r = R[f];
        }
        const uint32_t lt = r < B, eq = r == B;
        uint32_t tot_eq, tot_take;
        const uint32_t eq_rank = block_excl_scan(eq, ws, &tot_eq) + s_eq;
        const uint32_t take = lt || (eq && eq_rank < need_eq);
        const uint32_t slot = block_excl_scan(take, ws, &tot_take) + s_out;
        if (take) buf[(int64_t)q * C + slot] = ((unsigned long long)f << 32) | (uint32_t)p;
        __syncthreads();
        if (threadIdx.x == 0) { s_out += tot_take; s_eq += tot_eq; }
        __syncthreads();
    }
    if (threadIdx.x == 0) cnt[q] = (uint32_t)Tq;
}

// ---------------------------------------------------------------- parallel fallback
// Queries whose pilot bound under- or overshot are re-done exactly by all SMs at once
// (the one-CTA-per-query k6_fallback takes ~4.5 ms for a query on c4): an exact
// histogram of the structure positions over all n items (slices of n per CTA,
// flushed to a per-query global histogram), the exact bound B, then every item with
// R <= B appended — the select resolves the ties at B as usual (the buffer holds
// them: count(< B) < T and the cell at B is at most one sub-dataset, C covers both).
// Persistent grids over a device-side list of the failed queries: nothing to do
// costs three near-empty launches.
constexpr int kFbSlices = 32;
constexpr int kFbMax = 64;   // failed queries handled per sub-batch this way

__global__ void fb_list(const uint32_t *__restrict__ cnt, const uint32_t *__restrict__ cntv, int Qb,
                        int64_t Tq, int64_t C, int32_t *__restrict__ fl, uint32_t *__restrict__ nf,
                        int *__restrict__ flags) {
    pdl_wait();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Qb) return;
    const uint32_t v = cntv ? cntv[q] : cnt[q];
    if ((uint64_t)v >= (uint64_t)Tq && (uint64_t)cnt[q] <= (uint64_t)C) return;
    atomicAdd(&flags[2], 1);   // counted here; the serial kernel then counts nothing
    const uint32_t i = atomicAdd(nf, 1u);
    if (i < (uint32_t)kFbMax) fl[i] = q;
}

template <int W>
__global__ void __launch_bounds__(1024) fb_hist(const uint32_t *__restrict__ codes,
                                                const uint8_t *__restrict__ part, int64_t n,
                                                const uint32_t *__restrict__ qcodes, int L, int NR,
                                                const uint16_t *__restrict__ R,
                                                const int32_t *__restrict__ fl, const uint32_t *__restrict__ nf,
                                                uint32_t *__restrict__ ghist, int QM) {
    pdl_wait();
    extern __shared__ uint32_t hist[];
    const int nfl = (int)min(*nf, (uint32_t)kFbMax);
    const int lane = threadIdx.x & 31;
    for (int w = blockIdx.x; w < nfl * kFbSlices; w += gridDim.x) {
        const int fi = w / kFbSlices, sl = w % kFbSlices;
        const int q = fl[fi];
        uint32_t qc[W];
#pragma unroll
        for (int k = 0; k < W; ++k) qc[k] = qcodes[(int64_t)q * QM * W + k];
        const uint32_t *qall = qcodes + (int64_t)q * QM * W;
        for (int e = threadIdx.x; e < NR; e += blockDim.x) hist[e] = 0u;
        __syncthreads();
        const int64_t p0 = n * sl / kFbSlices, p1 = n * (sl + 1) / kFbSlices;
        for (int64_t b0 = p0; b0 < p1; b0 += blockDim.x) {
            const int64_t p = b0 + threadIdx.x;
            int r = -1;
            if (p < p1) {
                uint32_t c[W];
                load_code<W>(codes, p, c);
                const int pj = part[p];
                r = R[pj * (L + 1) + (QM > 1 ? hamming_at<W>(c, qall + pj * W) : hamming<W>(c, qc))];
            }
            const unsigned peers = __match_any_sync(NR_FULL, r);
            if (r >= 0 && lane == __ffs(peers) - 1) atomicAdd(&hist[r], (uint32_t)__popc(peers));
        }
        __syncthreads();
        for (int e = threadIdx.x; e < NR; e += blockDim.x)
            if (hist[e]) atomicAdd(&ghist[(int64_t)fi * NR + e], hist[e]);
        __syncthreads();
    }
}

// exact bound per failed query; clears its histogram row and its buffer counters
__global__ void __launch_bounds__(1024) fb_bound(const int32_t *__restrict__ fl,
                                                 const uint32_t *__restrict__ nf, int NR, int64_t Tq,
                                                 uint32_t *__restrict__ ghist, uint32_t *__restrict__ Bout,
                                                 uint32_t *__restrict__ cnt, uint32_t *__restrict__ cntv) {
    pdl_wait();
    __shared__ uint32_t ws[32];
    __shared__ int sB;
    const int nfl = (int)min(*nf, (uint32_t)kFbMax);
    for (int fi = blockIdx.x; fi < nfl; fi += gridDim.x) {
        uint32_t *h = ghist + (int64_t)fi * NR;
        if (threadIdx.x == 0) sB = NR - 1;
        __syncthreads();
        const int seg = (NR + blockDim.x - 1) / blockDim.x;
        const int r0 = threadIdx.x * seg, r1 = min(NR, r0 + seg);
        uint32_t loc = 0;
        for (int r = r0; r < r1; ++r) loc += h[r];
        uint32_t tot;
        const uint32_t ex = block_excl_scan(loc, ws, &tot);
        if (ex < (uint64_t)Tq && ex + loc >= (uint64_t)Tq) {
            uint32_t cc = ex;
            for (int r = r0; r < r1; ++r) {
                if (cc + h[r] >= (uint64_t)Tq) { sB = r; break; }
                cc += h[r];
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            Bout[fi] = (uint32_t)sB;
            cnt[fl[fi]] = 0u;
            if (cntv) cntv[fl[fi]] = 0u;
        }
        for (int r = threadIdx.x; r < NR; r += blockDim.x) h[r] = 0u;
        __syncthreads();
    }
}

template <int W>
__global__ void __launch_bounds__(1024) fb_take(const uint32_t *__restrict__ codes,
                                                const uint8_t *__restrict__ part, int64_t n,
                                                const uint32_t *__restrict__ qcodes, int L,
                                                const uint16_t *__restrict__ R,
                                                const int32_t *__restrict__ fl, const uint32_t *__restrict__ nf,
                                                const uint32_t *__restrict__ Bq,
                                                unsigned long long *__restrict__ buf, uint32_t *__restrict__ cnt,
                                                uint32_t *__restrict__ cntv, int64_t C, int QM) {
    pdl_wait();
    const int nfl = (int)min(*nf, (uint32_t)kFbMax);
    const int lane = threadIdx.x & 31;
    for (int w = blockIdx.x; w < nfl * kFbSlices; w += gridDim.x) {
        const int fi = w / kFbSlices, sl = w % kFbSlices;
        const int q = fl[fi];
        const uint32_t B = Bq[fi];
        uint32_t qc[W];
#pragma unroll
        for (int k = 0; k < W; ++k) qc[k] = qcodes[(int64_t)q * QM * W + k];
        const uint32_t *qall = qcodes + (int64_t)q * QM * W;
        const int64_t p0 = n * sl / kFbSlices, p1 = n * (sl + 1) / kFbSlices;
        uint32_t mine = 0;
        for (int64_t b0 = p0; b0 < p1; b0 += blockDim.x) {
            const int64_t p = b0 + threadIdx.x;
            bool take = false;
            uint32_t f = 0;
            if (p < p1) {
                uint32_t c[W];
                load_code<W>(codes, p, c);
                const int pj = part[p];
                f = pj * (L + 1) + (QM > 1 ? hamming_at<W>(c, qall + pj * W) : hamming<W>(c, qc));
                take = R[f] <= B;
            }
            const unsigned bal = __ballot_sync(NR_FULL, take);
            if (!bal) continue;
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&cnt[q], (uint32_t)__popc(bal));
            base = __shfl_sync(NR_FULL, base, 0);
            if (take) {
                const uint32_t slot = base + __popc(bal & lanemask_lt());
                if (slot < C) buf[(int64_t)q * C + slot] = ((unsigned long long)f << 32) | (uint32_t)p;
                ++mine;
            }
        }
        if (mine && cntv) atomicAdd(&cntv[q], mine);
    }
}

size_t fallback_ws_bytes(const nrlsh_index *ix) {
    return ((size_t)kFbMax * ix->m * (ix->L + 1) + 2 * kFbMax + 64) * 4;
}

uint32_t *fallback_counter(const nrlsh_index *ix, void *ws) {
    if (!ws) return nullptr;
    const int NR = ix->m * (ix->L + 1);
    return reinterpret_cast<uint32_t *>(ws) + (size_t)kFbMax * NR + 2 * kFbMax;
}

void launch_fallback(const nrlsh_index *ix, const uint32_t *qcodes, int Qb, int64_t Tq,
                     unsigned long long *buf, uint32_t *cnt, uint32_t *cntv, int64_t C,
                     int *flags, void *ws, cudaStream_t s) {
    const int NR = ix->m * (ix->L + 1);
    const bool par = ws && !getenv("NRLSH_FALLBACK_SERIAL");
    if (par) {
        uint32_t *cv_sep = cntv != cnt ? cntv : nullptr;   // (popcount scan: cntv is cnt)
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
        uint32_t *ghist = reinterpret_cast<uint32_t *>(ws);   // [kFbMax x NR], zero between uses
        int32_t *fl = reinterpret_cast<int32_t *>(ghist + (size_t)kFbMax * NR);
        uint32_t *Bq = reinterpret_cast<uint32_t *>(fl + kFbMax);
        uint32_t *nf = Bq + kFbMax;   // (zeroed by the pilot: fallback_counter)
        launch_pdl(fb_list, dim3((Qb + 255) / 256), dim3(256), 0, s, cnt, cv_sep, Qb, Tq, C, fl, nf, flags);
        const size_t sm = (size_t)NR * 4;
        const int QM = ix->QM;
#define NR_FB(W_)                                                                                   \
        cudaFuncSetAttribute(fb_hist<W_>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);    \
        launch_pdl(fb_hist<W_>, dim3(sms), dim3(1024), sm, s, ix->codes, ix->part_of_pos, ix->n, qcodes, ix->L, NR,     \
                                          ix->R_d, fl, nf, ghist, QM);                              \
        launch_pdl(fb_bound, dim3(sms), dim3(1024), 0, s, fl, nf, NR, Tq, ghist, Bq, cnt, cv_sep);                      \
        launch_pdl(fb_take<W_>, dim3(sms), dim3(1024), 0, s, ix->codes, ix->part_of_pos, ix->n, qcodes, ix->L, ix->R_d, \
                                         fl, nf, Bq, buf, cnt, cv_sep, C, QM)
        if (ix->W == 1) { NR_FB(1); } else if (ix->W == 2) { NR_FB(2); } else { NR_FB(4); }
#undef NR_FB
        note_launch(4);
        // the serial kernel below still counts every failed query (flags[2]) and
        // handles any beyond kFbMax; the ones done here now pass its test
    }
    const size_t sm = (size_t)NR * 4 + (ix->QM > 1 ? (size_t)ix->QM * ix->W * 4 : 0);
    const int32_t *order = ix->order_d;
    switch (ix->W) {
        case 1:
            cudaFuncSetAttribute(k6_fallback<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            launch_pdl(k6_fallback<1>, dim3(Qb), dim3(1024), sm, s, ix->codes, ix->part_of_pos, ix->n, qcodes, ix->L, ix->m, order, ix->R_d, Tq, buf, cnt, cntv, C, par ? nullptr : flags, ix->QM);
            break;
        case 2:
            cudaFuncSetAttribute(k6_fallback<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            launch_pdl(k6_fallback<2>, dim3(Qb), dim3(1024), sm, s, ix->codes, ix->part_of_pos, ix->n, qcodes, ix->L, ix->m, order, ix->R_d, Tq, buf, cnt, cntv, C, par ? nullptr : flags, ix->QM);
            break;
        default:
            cudaFuncSetAttribute(k6_fallback<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            launch_pdl(k6_fallback<4>, dim3(Qb), dim3(1024), sm, s, ix->codes, ix->part_of_pos, ix->n, qcodes, ix->L, ix->m, order, ix->R_d, Tq, buf, cnt, cntv, C, par ? nullptr : flags, ix->QM);
            break;
    }
    note_launch();
}

// =========================================================================== K7 select
// mode 0: bound + emit (all candidates); mode 1: bound only — writes the boundary
// structure position B and tie position bound pk per query, and the ks best-ranked
// candidates (seeds) of the tensor-core re-rank.
__global__ void __launch_bounds__(1024) k7_select(
    const unsigned long long *__restrict__ buf, const uint32_t *__restrict__ cnt, int64_t C,
    int64_t Tq, int NR, int tie_cap, const uint16_t *__restrict__ R,
    const int32_t *__restrict__ perm, int32_t *__restrict__ cand,
    uint16_t *__restrict__ cand_rank, int mode, uint32_t *__restrict__ sel_B,
    uint32_t *__restrict__ sel_pk, int32_t *__restrict__ seeds, int ks,
    const int32_t *__restrict__ order) {
    pdl_wait();
    extern __shared__ uint32_t hist[];   // [max(NR, tie_cap)] + R copy [NR] (uint16)
    uint16_t *sRt = reinterpret_cast<uint16_t *>(hist + tie_cap);
    __shared__ uint32_t ws[32];
    __shared__ uint32_t h256[256];
    __shared__ int sB, s_bseed;
    __shared__ uint32_t sLt, s_out, s_pfx, s_kth, s_seed, s_tlo, s_thi;
    const int q = blockIdx.x;
    const int64_t c = min((int64_t)cnt[q], C);
    const unsigned long long *b = buf + (int64_t)q * C;
    {   // zero the histogram, copy R (16-byte accesses; R is 16-byte aligned)
        const int nv = NR / 8;
        const uint4 *R4 = reinterpret_cast<const uint4 *>(R);
        uint4 *sR4 = reinterpret_cast<uint4 *>(sRt);
        uint4 *h4 = reinterpret_cast<uint4 *>(hist);
        for (int e = threadIdx.x; e < nv; e += blockDim.x) {
            sR4[e] = __ldg(R4 + e);
            h4[2 * e] = make_uint4(0u, 0u, 0u, 0u);
            h4[2 * e + 1] = make_uint4(0u, 0u, 0u, 0u);
        }
        for (int e = nv * 8 + threadIdx.x; e < NR; e += blockDim.x) { hist[e] = 0u; sRt[e] = R[e]; }
    }
    if (threadIdx.x == 0) { sB = NR - 1; sLt = 0; s_out = 0; s_bseed = NR - 1; }
    __syncthreads();
    // entries carry the flat (j, h) index f; the histogram is kept per f (one shared
    // atomic per entry, no R lookup), and the bound walks the structure through its
    // inverse order[] (~0 = unused append slot of the tensor-core scan)
    if ((C & 1) == 0) {   // 8 entries in flight per thread: 16-byte loads of entry pairs
        const int64_t c2 = c / 2;
        const ulonglong2 *b2 = reinterpret_cast<const ulonglong2 *>(b);
        int64_t e2 = threadIdx.x;
        for (; e2 + 3 * (int64_t)blockDim.x < c2; e2 += 4 * (int64_t)blockDim.x) {
            ulonglong2 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = b2[e2 + u * (int64_t)blockDim.x];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t f0 = (uint32_t)(v[u].x >> 32), f1 = (uint32_t)(v[u].y >> 32);
                if (f0 < (uint32_t)NR) atomicAdd(&hist[f0], 1u);
                if (f1 < (uint32_t)NR) atomicAdd(&hist[f1], 1u);
            }
        }
        for (; e2 < c2; e2 += blockDim.x) {
            const ulonglong2 v = b2[e2];
            const uint32_t f0 = (uint32_t)(v.x >> 32), f1 = (uint32_t)(v.y >> 32);
            if (f0 < (uint32_t)NR) atomicAdd(&hist[f0], 1u);
            if (f1 < (uint32_t)NR) atomicAdd(&hist[f1], 1u);
        }
        if ((c & 1) && threadIdx.x == 0) {
            const uint32_t f = (uint32_t)(b[c - 1] >> 32);
            if (f < (uint32_t)NR) atomicAdd(&hist[f], 1u);
        }
    } else {
        for (int64_t e = threadIdx.x; e < c; e += blockDim.x) {
            const uint32_t f = (uint32_t)(b[e] >> 32);
            if (f < (uint32_t)NR) atomicAdd(&hist[f], 1u);
        }
    }
    __syncthreads();
    const uint32_t need = (uint32_t)Tq;
    {
        const int seg = (NR + blockDim.x - 1) / blockDim.x;
        const int r0 = threadIdx.x * seg, r1 = min(NR, r0 + seg);
        uint32_t loc = 0;
        for (int r = r0; r < r1; ++r) loc += hist[__ldg(order + r)];
        uint32_t tot;
        const uint32_t ex = block_excl_scan(loc, ws, &tot);
        if (ex < need && ex + loc >= need) {
            uint32_t cc = ex;
            for (int r = r0; r < r1; ++r) {
                const uint32_t hr = hist[__ldg(order + r)];
                if (cc + hr >= need) { sB = r; sLt = cc; break; }
                cc += hr;
            }
        }
        if (seeds) {   // structure position holding the ks-th best-ranked entry
            if (ex < (uint32_t)ks && ex + loc >= (uint32_t)ks) {
                uint32_t cc = ex;
                for (int r = r0; r < r1; ++r) {
                    const uint32_t hr = hist[__ldg(order + r)];
                    if (cc + hr >= (uint32_t)ks) { s_bseed = r; break; }
                    cc += hr;
                }
            }
        }
        __syncthreads();
    }
    const uint32_t B = (uint32_t)sB;
    const uint32_t fB = (uint32_t)__ldg(order + B);   // the flat (j, h) cell at the bound
    const uint32_t need_eq = need - sLt;
    const uint32_t n_eq = hist[fB];
    // the need_eq-th smallest position among the ties (R == B): when they fit, one
    // pass gathers them into shared memory (reusing the histogram's space) and a
    // radix select runs there; otherwise radix select over the buffer, 8 bits/round
    if (threadIdx.x == 0) { s_pfx = 0; s_kth = need_eq; s_out = 0; s_tlo = 0xffffffffu; s_thi = 0u; }
    __syncthreads();
    uint32_t *teq = hist;   // the histogram is dead once B and n_eq are known
    const bool in_smem = need_eq < n_eq && n_eq <= (uint32_t)tie_cap;
    // the seeds ride along with the tie gather when they all rank before B (they then
    // need no tie cut-off): one pass over the buffer fewer
    const uint32_t Bsd = (uint32_t)s_bseed;
    const bool merge_seeds = mode == 1 && seeds && in_smem && Bsd < B;
    if (threadIdx.x == 0) s_seed = 0;
    __syncthreads();
    if (in_smem) {
        auto take = [&](unsigned long long v) {
            const uint32_t f = (uint32_t)(v >> 32);
            if (f >= (uint32_t)NR) return;
            if (f == fB) teq[atomicAdd(&s_out, 1u)] = (uint32_t)v;
            else if (merge_seeds && sRt[f] <= Bsd) {
                const uint32_t slot = atomicAdd(&s_seed, 1u);
                if (slot < (uint32_t)ks) seeds[(int64_t)q * ks + slot] = perm[(uint32_t)v];
            }
        };
        if ((C & 1) == 0) {   // (paired 16-byte loads, 8 entries in flight per thread)
            const int64_t c2 = c / 2;
            const ulonglong2 *b2 = reinterpret_cast<const ulonglong2 *>(b);
            int64_t e2 = threadIdx.x;
            for (; e2 + 3 * (int64_t)blockDim.x < c2; e2 += 4 * (int64_t)blockDim.x) {
                ulonglong2 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = b2[e2 + u * (int64_t)blockDim.x];
#pragma unroll
                for (int u = 0; u < 4; ++u) { take(v[u].x); take(v[u].y); }
            }
            for (; e2 < c2; e2 += blockDim.x) {
                const ulonglong2 v = b2[e2];
                take(v.x);
                take(v.y);
            }
            if ((c & 1) && threadIdx.x == 0) take(b[c - 1]);
        } else {
            for (int64_t e = threadIdx.x; e < c; e += blockDim.x) take(b[e]);
        }
        __syncthreads();
        // the ties share one sub-dataset (a contiguous position range): the radix
        // select starts at the highest byte where their positions differ, with the
        // common prefix above it
        {
            uint32_t lo = 0xffffffffu, hi = 0u;
            for (uint32_t e = threadIdx.x; e < n_eq; e += blockDim.x) {
                const uint32_t pos = teq[e];
                lo = min(lo, pos);
                hi = max(hi, pos);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                lo = min(lo, __shfl_xor_sync(NR_FULL, lo, o));
                hi = max(hi, __shfl_xor_sync(NR_FULL, hi, o));
            }
            if ((threadIdx.x & 31) == 0) { atomicMin(&s_tlo, lo); atomicMax(&s_thi, hi); }
        }
        __syncthreads();
        const uint32_t tdiff = s_tlo ^ s_thi;
        const int shift0 = tdiff ? ((31 - __clz(tdiff)) / 8) * 8 : 0;
        if (threadIdx.x == 0 && shift0 < 24) s_pfx = s_tlo & (0xffffffffu << (shift0 + 8));
        __syncthreads();
        for (int shift = shift0; shift >= 0; shift -= 8) {
            for (int e = threadIdx.x; e < 256; e += blockDim.x) h256[e] = 0;
            __syncthreads();
            const uint32_t pfx = s_pfx;
            for (uint32_t e = threadIdx.x; e < n_eq; e += blockDim.x) {
                const uint32_t pos = teq[e];
                if (shift < 24 && (pos >> (shift + 8)) != (pfx >> (shift + 8))) continue;
                atomicAdd(&h256[(pos >> shift) & 255u], 1u);
            }
            __syncthreads();
            if (threadIdx.x < 32) {   // warp-parallel scan of the 256 digit counts
                uint32_t v[8], loc = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) { v[i] = h256[threadIdx.x * 8 + i]; loc += v[i]; }
                uint32_t inc = loc;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(NR_FULL, inc, o);
                    if (threadIdx.x >= o) inc += y;
                }
                const uint32_t k = s_kth;
                uint32_t ex = inc - loc;
                if (ex < k && inc >= k) {
                    for (int i = 0; i < 8; ++i) {
                        if (ex + v[i] >= k) {
                            s_pfx = pfx | ((uint32_t)(threadIdx.x * 8 + i) << shift);
                            s_kth = k - ex;
                            break;
                        }
                        ex += v[i];
                    }
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) s_out = 0;
        __syncthreads();
    }
    if (!in_smem && need_eq < n_eq) {
        for (int shift = 24; shift >= 0; shift -= 8) {
            for (int e = threadIdx.x; e < 256; e += blockDim.x) h256[e] = 0;
            __syncthreads();
            const uint32_t pfx = s_pfx;
            for (int64_t e = threadIdx.x; e < c; e += blockDim.x) {
                const unsigned long long v = b[e];
                const uint32_t f = (uint32_t)(v >> 32);
                if (f != fB) continue;
                const uint32_t pos = (uint32_t)v;
                if (shift < 24 && (pos >> (shift + 8)) != (pfx >> (shift + 8))) continue;
                atomicAdd(&h256[(pos >> shift) & 255u], 1u);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t k = s_kth, acc = 0;
                for (int dg = 0; dg < 256; ++dg) {
                    if (acc + h256[dg] >= k) { s_pfx = pfx | ((uint32_t)dg << shift); s_kth = k - acc; break; }
                    acc += h256[dg];
                }
            }
            __syncthreads();
        }
    } else if (!in_smem && threadIdx.x == 0) {
        s_pfx = 0xffffffffu;
    }
    __syncthreads();
    const uint32_t pk = s_pfx;
    if (mode == 1) {
        if (threadIdx.x == 0) { sel_B[q] = B; sel_pk[q] = pk; }
        if (seeds && merge_seeds) {   // (gathered with the ties)
            for (uint32_t t = min(s_seed, (uint32_t)ks) + threadIdx.x; t < (uint32_t)ks; t += blockDim.x)
                seeds[(int64_t)q * ks + t] = -1;
        } else if (seeds) {   // up to ks candidates among the best-ranked structure positions
            if (threadIdx.x == 0) s_out = 0;
            __syncthreads();
            const uint32_t Bs = (uint32_t)s_bseed;
            for (int64_t e = threadIdx.x; e < c; e += blockDim.x) {
                const unsigned long long v = b[e];
                const uint32_t f = (uint32_t)(v >> 32), pos = (uint32_t)v;
                if (f >= (uint32_t)NR) continue;
                const uint32_t r = sRt[f];
                if (r <= Bs && (r < B || (r == B && pos <= pk))) {
                    const uint32_t slot = atomicAdd(&s_out, 1u);
                    if (slot < (uint32_t)ks) seeds[(int64_t)q * ks + slot] = perm[pos];
                }
            }
            __syncthreads();
            for (uint32_t t = s_out + threadIdx.x; t < (uint32_t)ks; t += blockDim.x)
                seeds[(int64_t)q * ks + t] = -1;
        }
        return;
    }
    for (int64_t e = threadIdx.x; e < c; e += blockDim.x) {
        const unsigned long long v = b[e];
        const uint32_t f = (uint32_t)(v >> 32), pos = (uint32_t)v;
        if (f >= (uint32_t)NR) continue;
        const uint32_t r = sRt[f];
        if (r < B || (r == B && pos <= pk)) {
            const uint32_t slot = atomicAdd(&s_out, 1u);
            if (slot < need) {
                cand[(int64_t)q * Tq + slot] = perm[pos];
                if (cand_rank) cand_rank[(int64_t)q * Tq + slot] = (uint16_t)r;
            }
        }
    }
}

void launch_select(const nrlsh_index *ix, int Qb, int64_t Tq, const unsigned long long *buf,
                   const uint32_t *cnt, int64_t C, int32_t *cand, uint16_t *cand_rank,
                   cudaStream_t s) {
    const int NR = ix->m * (ix->L + 1);
    const int tie_cap = std::max(NR, 16384);
    const size_t sm = (size_t)tie_cap * 4 + (size_t)NR * 2;
    cudaFuncSetAttribute(k7_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_pdl(k7_select, dim3(Qb), dim3(1024), sm, s, buf, cnt, C, Tq, NR, tie_cap, ix->R_d, ix->perm, cand, cand_rank,
                                   0, nullptr, nullptr, nullptr, 0, ix->order_d);
    note_launch();
}


void launch_select_seeds(const nrlsh_index *ix, int Qb, int64_t Tq, const unsigned long long *buf,
                         const uint32_t *cnt, int64_t C, uint32_t *sel_B, uint32_t *sel_pk,
                         int32_t *seeds, int ks, cudaStream_t s) {
    const int NR = ix->m * (ix->L + 1);
    const int tie_cap = std::max(NR, 16384);
    const size_t sm = (size_t)tie_cap * 4 + (size_t)NR * 2;
    cudaFuncSetAttribute(k7_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    launch_pdl(k7_select, dim3(Qb), dim3(1024), sm, s, buf, cnt, C, Tq, NR, tie_cap, ix->R_d, ix->perm, nullptr, nullptr,
                                   1, sel_B, sel_pk, seeds, ks, ix->order_d);
    note_launch();
}

// ------------------------------------------------------- tensor-core re-rank helpers
__global__ void gather_f32(const float *__restrict__ src, const int32_t *__restrict__ idx, int64_t n,
                           float *__restrict__ dst) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x)
        dst[p] = src[idx[p]];
}

void launch_gather_f32(const float *src, const int32_t *idx, int64_t n, float *dst, cudaStream_t s) {
    gather_f32<<<grid_for(n, 256, 4096), 256, 0, s>>>(src, idx, n, dst);
    note_launch();
}

// rows idx[r] of src -> row r of dst (scatter: row r of src -> row idx[r] of dst);
// rows of `words` 32-bit words
__global__ void move_rows(const uint32_t *__restrict__ src, const int64_t *__restrict__ idx, int nrows,
                          int64_t words, uint32_t *__restrict__ dst, int scatter) {
    for (int r = blockIdx.x; r < nrows; r += gridDim.x) {
        const int64_t a = scatter ? r : idx[r], b = scatter ? idx[r] : r;
        for (int64_t w = threadIdx.x; w < words; w += blockDim.x) dst[b * words + w] = src[a * words + w];
    }
}

void launch_move_rows(const void *src, const int64_t *idx, int nrows, size_t row_bytes, void *dst,
                      bool scatter, cudaStream_t s) {
    if (nrows <= 0) return;
    move_rows<<<std::min(nrows, 4096), 128, 0, s>>>((const uint32_t *)src, idx, nrows,
                                                     (int64_t)(row_bytes / 4), (uint32_t *)dst, scatter);
    note_launch();
}

__global__ void theta_from_topk(const int64_t *__restrict__ ids, const float *__restrict__ sc, int Qb,
                                int k, uint32_t *__restrict__ theta_glob, int assign,
                                uint32_t *__restrict__ zero_cnt) {
    pdl_wait();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Qb) return;
    const int64_t e = (int64_t)q * k + k - 1;
    const uint32_t o = ids[e] >= 0 ? float_order(sc[e]) : 0u;
    theta_glob[q] = assign ? o : max(theta_glob[q], o);
    if (zero_cnt) zero_cnt[q] = 0u;
}

void launch_theta_from_topk(const int64_t *ids, const float *scores, int Qb, int k,
                            uint32_t *theta_glob, cudaStream_t s, bool assign, uint32_t *zero_cnt) {
    launch_pdl(theta_from_topk, dim3((Qb + 255) / 256), dim3(256), 0, s, ids, scores, Qb, k, theta_glob,
               (int)assign, zero_cnt);
    note_launch();
}

// Restart each query's survivor list from its exact top-k so far (the first pass's
// survivors re-ranked): top-k(A u B) = top-k(top-k(A) u B), so the final re-rank
// only re-scores k rows of the first pass.  An overflowed list (cnt > C) is kept
// as it is (the overflow redo needs its count).
__global__ void restart_from_topk(const int64_t *__restrict__ ids, int Qb, int k,
                                  int32_t *__restrict__ cand, int64_t C, uint32_t *__restrict__ cnt) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Qb || (int64_t)cnt[q] > C) return;
    uint32_t c = 0;
    for (int t = 0; t < k && (int64_t)t < C; ++t) {
        const int64_t id = ids[(int64_t)q * k + t];
        if (id >= 0) cand[(int64_t)q * C + c++] = (int32_t)id;
    }
    cnt[q] = c;
}

void launch_restart_from_topk(const int64_t *ids, int Qb, int k, int32_t *cand, int64_t C,
                              uint32_t *cnt, cudaStream_t s) {
    restart_from_topk<<<(Qb + 255) / 256, 256, 0, s>>>(ids, Qb, k, cand, C, cnt);
    note_launch();
}

__global__ void collect_overflow(const uint32_t *__restrict__ cnt, int Qb, int64_t C, int64_t q0,
                                 int64_t *__restrict__ list, uint32_t *__restrict__ n) {
    pdl_wait();
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < Qb && (int64_t)cnt[q] > C) list[atomicAdd(n, 1u)] = q0 + q;
}

__global__ void sum_counts(const uint32_t *__restrict__ cnt, int Qb, int64_t C,
                           unsigned long long *__restrict__ out) {
    pdl_wait();
    unsigned long long v = 0;
    for (int q = threadIdx.x; q < Qb; q += blockDim.x) v += (unsigned long long)min((int64_t)cnt[q], C);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(NR_FULL, v, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, v);
}

void launch_sum_counts(const uint32_t *cnt, int Qb, int64_t C, unsigned long long *out,
                       cudaStream_t s) {
    launch_pdl(sum_counts, dim3(1), dim3(256), 0, s, cnt, Qb, C, out);
    note_launch();
}

__global__ void count_stats(const uint32_t *__restrict__ cnt, int Qb,
                            unsigned long long *__restrict__ out) {
    unsigned long long mx = 0, sm = 0;
    for (int q = threadIdx.x; q < Qb; q += blockDim.x) {
        mx = max(mx, (unsigned long long)cnt[q]);
        sm += cnt[q];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(NR_FULL, mx, o));
        sm += __shfl_xor_sync(NR_FULL, sm, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMax(out, mx);
        atomicAdd(out + 1, sm);
    }
}

void launch_count_stats(const uint32_t *cnt, int Qb, unsigned long long *out, cudaStream_t s) {
    count_stats<<<1, 256, 0, s>>>(cnt, Qb, out);
    note_launch();
}

void launch_collect_overflow(const uint32_t *cnt, int Qb, int64_t C, int64_t q0, int64_t *list,
                             uint32_t *n, cudaStream_t s) {
    launch_pdl(collect_overflow, dim3((Qb + 255) / 256), dim3(256), 0, s, cnt, Qb, C, q0, list, n);
    note_launch();
}

// =========================================================================== K8 score
// CTA = (query, slice of candidates); one warp per candidate row, lanes stride d
// (coalesced 128 B), fp32 FMA + xor-shuffle reduction.
__global__ void __launch_bounds__(256) k8_score(
    const float *__restrict__ X, int d, const float *__restrict__ Q,
    const int32_t *__restrict__ cand, int64_t ncand, int64_t cand_ld,
    const uint32_t *__restrict__ ncand_per_q, int stride, const float *__restrict__ xnorm,
    const float *__restrict__ qnorm, float lb_eps, float *__restrict__ scores) {
    extern __shared__ float sq[];
    const int q = blockIdx.x;
    for (int k = threadIdx.x; k < d; k += blockDim.x) sq[k] = Q[(int64_t)q * d + k];
    __syncthreads();
    int64_t nc = ncand;
    if (ncand_per_q) nc = min((int64_t)ncand_per_q[q], cand_ld);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float qn = qnorm ? qnorm[q] : 0.f;
    for (int64_t t = (int64_t)blockIdx.y * 8 + warp; t < nc; t += (int64_t)gridDim.y * 8) {
        const int64_t id = cand ? (int64_t)cand[(int64_t)q * cand_ld + t] : t * stride;
        const float *x = X + id * d;
        float acc = 0.f;
        for (int k = lane; k < d; k += 32) acc = fmaf(sq[k], __ldg(x + k), acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(NR_FULL, acc, o);
        if (lane == 0) {
            float sc = acc;
            if (lb_eps > 0.f) sc = __fsub_rd(acc, lb_eps * qn * xnorm[id]);
            scores[(int64_t)q * cand_ld + t] = sc;
        }
    }
}

void launch_score(const float *X, int d, const float *Q, int Qb, const int32_t *cand,
                  int64_t ncand, int64_t cand_ld, const uint32_t *ncand_per_q, int stride,
                  const float *xnorm, const float *qnorm, float lb_eps, float *scores,
                  cudaStream_t s) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int64_t per = (ncand + 7) / 8;
    int gy = (int)std::min<int64_t>(std::max<int64_t>(1, per / 16), std::max(1, (sms * 16) / std::max(1, Qb)));
    if (gy < 1) gy = 1;
    dim3 grid(Qb, gy);
    k8_score<<<grid, 256, (size_t)d * 4, s>>>(X, d, Q, cand, ncand, cand_ld, ncand_per_q, stride,
                                             xnorm, qnorm, lb_eps, scores);
    note_launch();
}

// =========================================================================== K8 top-k
// Key = (~order(score)) << 32 | id: ascending key order is (score desc, id asc).
// Radix-select the k-th smallest key (8 rounds of 8 bits), collect the k keys <=
// it, bitonic-sort them.  Keys are cached in shared memory when they fit.
constexpr int kTopkSmemKeys = 26624;   // 208 KB of keys: covers T = 1% of the c4 config
constexpr int kMaxK = 1024;

__device__ __forceinline__ unsigned long long topk_key(float sc, uint32_t id) {
    return ((unsigned long long)(~float_order(sc)) << 32) | id;
}

__global__ void __launch_bounds__(1024) k8_topk(
    const float *__restrict__ scores, const int32_t *__restrict__ cand, int64_t ncand,
    int64_t cand_ld, const uint32_t *__restrict__ ncand_per_q, int stride, int k,
    int64_t smem_cap, int64_t *__restrict__ out_ids, float *__restrict__ out_scores,
    float *__restrict__ kth_out) {
    extern __shared__ unsigned long long skeys[];
    __shared__ uint32_t h256[256];
    __shared__ unsigned long long s_pfx;
    __shared__ uint32_t s_kth, s_n;
    __shared__ unsigned long long sel[kMaxK];
    const int q = blockIdx.x;
    int64_t c = ncand;
    if (ncand_per_q) c = min((int64_t)ncand_per_q[q], cand_ld);
    const bool cached = c <= smem_cap;
    auto key_at = [&](int64_t e) -> unsigned long long {
        const float sc = scores[(int64_t)q * cand_ld + e];
        const uint32_t id = cand ? (uint32_t)cand[(int64_t)q * cand_ld + e] : (uint32_t)(e * stride);
        return topk_key(sc, id);
    };
    if (cached)
        for (int64_t e = threadIdx.x; e < c; e += blockDim.x) skeys[e] = key_at(e);
    const int kk = (int)min((int64_t)k, c);
    if (threadIdx.x == 0) { s_pfx = 0; s_kth = kk; s_n = 0; }
    __syncthreads();
    if (kk > 0 && kk < c) {
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int e = threadIdx.x; e < 256; e += blockDim.x) h256[e] = 0;
            __syncthreads();
            const unsigned long long pfx = s_pfx;
            for (int64_t e = threadIdx.x; e < c; e += blockDim.x) {
                const unsigned long long v = cached ? skeys[e] : key_at(e);
                if (shift < 56 && (v >> (shift + 8)) != (pfx >> (shift + 8))) continue;
                atomicAdd(&h256[(v >> shift) & 255u], 1u);
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t kt = s_kth, acc = 0;
                for (int dg = 0; dg < 256; ++dg) {
                    if (acc + h256[dg] >= kt) {
                        s_pfx = pfx | ((unsigned long long)dg << shift);
                        s_kth = kt - acc;
                        break;
                    }
                    acc += h256[dg];
                }
            }
            __syncthreads();
        }
    } else if (threadIdx.x == 0) {
        s_pfx = ~0ull;
    }
    __syncthreads();
    const unsigned long long thr = s_pfx;
    for (int64_t e = threadIdx.x; e < c; e += blockDim.x) {
        const unsigned long long v = cached ? skeys[e] : key_at(e);
        if (v <= thr) {
            const uint32_t slot = atomicAdd(&s_n, 1u);
            if (slot < (uint32_t)kMaxK) sel[slot] = v;
        }
    }
    __syncthreads();
    int np2 = 1;
    while (np2 < kk) np2 <<= 1;
    for (int t = threadIdx.x; t < np2; t += blockDim.x)
        if (t >= kk) sel[t] = ~0ull;
    __syncthreads();
    for (int size = 2; size <= np2; size <<= 1) {
        for (int st = size >> 1; st > 0; st >>= 1) {
            for (int t = threadIdx.x; t < np2; t += blockDim.x) {
                const int o = t ^ st;
                if (o > t) {
                    const bool up = (t & size) == 0;
                    if ((sel[t] > sel[o]) == up) {
                        unsigned long long tmp = sel[t]; sel[t] = sel[o]; sel[o] = tmp;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int t = threadIdx.x; t < k; t += blockDim.x) {
        if (t < kk) {
            const unsigned long long v = sel[t];
            out_ids[(int64_t)q * k + t] = (int64_t)(uint32_t)v;
            out_scores[(int64_t)q * k + t] = float_unorder(~(uint32_t)(v >> 32));
        } else {
            out_ids[(int64_t)q * k + t] = -1;
            out_scores[(int64_t)q * k + t] = -INFINITY;
        }
    }
    if (kth_out && threadIdx.x == 0)
        kth_out[q] = (kk == k && kk > 0) ? float_unorder(~(uint32_t)(sel[kk - 1] >> 32)) : -INFINITY;
}

void launch_topk(const float *scores, const int32_t *cand, int Qb, int64_t ncand,
                 int64_t cand_ld, const uint32_t *ncand_per_q, int stride, int k,
                 int64_t *out_ids, float *out_scores, float *kth_out, cudaStream_t s) {
    const int64_t cap = std::min<int64_t>(std::max<int64_t>(ncand, 1), kTopkSmemKeys);
    const size_t sm = (size_t)cap * 8;
    cudaFuncSetAttribute(k8_topk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    k8_topk<<<Qb, 1024, sm, s>>>(scores, cand, ncand, cand_ld, ncand_per_q, stride, k, cap,
                                 out_ids, out_scores, kth_out);
    note_launch();
}

// =========================================================================== K8 fused re-rank
// Exact re-rank (Alg. 2 l.6) fused with the top-k of (score desc, id asc).
// CTA = (query q, slice of its candidate list).  A warp scores 4 candidate rows at a
// time, 8 lanes per row, VEC-wide loads: every lane keeps ceil(d / 8VEC) independent
// loads in flight (the gather is latency-bound otherwise), and the 32 candidate ids a
// warp needs per round come from one coalesced load.  Scores never go to HBM: keys
// (~order(score) << 32 | id) better than the CTA's running k-th best enter a shared
// buffer that is bitonic-sorted and truncated to k when it fills.
constexpr int kRrThreads = 256;
constexpr int kRrRound = kRrThreads;          // candidate rows per CTA round
constexpr int kRrLPR = 8;                     // lanes per row
constexpr int kRrMaxIt = 8;                   // loads per lane kept in flight

__device__ __forceinline__ void bitonic_sort_smem(unsigned long long *a, int np2) {
    for (int size = 2; size <= np2; size <<= 1) {
        for (int st = size >> 1; st > 0; st >>= 1) {
            for (int t = threadIdx.x; t < np2; t += blockDim.x) {
                const int o = t ^ st;
                if (o > t) {
                    const bool up = (t & size) == 0;
                    const unsigned long long x = a[t], y = a[o];
                    if ((x > y) == up) { a[t] = y; a[o] = x; }
                }
            }
            __syncthreads();
        }
    }
}

template <int VEC>
__device__ __forceinline__ void vload(const float *p, float (&v)[VEC]) {
    if (VEC == 4) {
        const float4 t = __ldg(reinterpret_cast<const float4 *>(p));
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    } else if (VEC == 2) {
        const float2 t = __ldg(reinterpret_cast<const float2 *>(p));
        v[0] = t.x; v[1] = t.y;
    } else {
        v[0] = __ldg(p);
    }
}

// one lane's share of q.x for one row: xl = row + sub*VEC, ql = sq + sub*VEC,
// rem = d - sub*VEC.  NIT = ceil(d / (8 VEC)) loads, all issued before any use;
// only the last one can leave the row (its address is clamped, its value zeroed).
template <int VEC, int NIT>
__device__ __forceinline__ float row_dot(const float *__restrict__ xl, const float *ql, int rem) {
    float xv[NIT][VEC];
#pragma unroll
    for (int i = 0; i < NIT; ++i) {
        const int off = i * kRrLPR * VEC;
        vload<VEC>(xl + (i < NIT - 1 ? off : max(0, min(off, rem - VEC))), xv[i]);
    }
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < NIT; ++i) {
        const int off = i * kRrLPR * VEC;
        const bool ok = (i < NIT - 1) || off < rem;
#pragma unroll
        for (int v = 0; v < VEC; ++v) acc = fmaf(ql[ok ? off + v : v], ok ? xv[i][v] : 0.f, acc);
    }
    return acc;
}

// any d: blocks of kRrMaxIt loads with clamped addresses
template <int VEC>
__device__ __forceinline__ float row_dot_any(const float *__restrict__ xl, const float *ql, int rem) {
    float acc = 0.f;
    for (int o0 = 0; o0 < rem; o0 += kRrMaxIt * kRrLPR * VEC) {
        float xv[kRrMaxIt][VEC];
#pragma unroll
        for (int u = 0; u < kRrMaxIt; ++u)
            vload<VEC>(xl + max(0, min(o0 + u * kRrLPR * VEC, rem - VEC)), xv[u]);
#pragma unroll
        for (int u = 0; u < kRrMaxIt; ++u) {
            const int off = o0 + u * kRrLPR * VEC;
            const bool ok = off < rem;
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc = fmaf(ql[ok ? off + v : v], ok ? xv[u][v] : 0.f, acc);
        }
    }
    return acc;
}

template <int VEC, int NIT>
__global__ void __launch_bounds__(kRrThreads) k8_rerank(
    const float *__restrict__ X, int d, int dq, const float *__restrict__ Q,
    const int32_t *__restrict__ cand, int64_t cand_ld, int64_t ncand,
    const uint32_t *__restrict__ ncand_per_q, int stride, int k, int cap, int64_t slice,
    unsigned long long *__restrict__ partial, int64_t *__restrict__ out_ids,
    float *__restrict__ out_scores) {
    pdl_wait();
    extern __shared__ __align__(16) unsigned long long rr_smem[];
    unsigned long long *buf = rr_smem;                       // [cap]
    float *sq = reinterpret_cast<float *>(buf + cap);        // [dpad]
    __shared__ unsigned int s_cnt;
    __shared__ unsigned long long s_thr;
    const int q = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane & (kRrLPR - 1), grp = lane >> 3;
    // X rows hold d floats (a zero-padded copy may have d > dq); queries hold dq
    const int dpad = (d + 8 * VEC - 1) / (8 * VEC) * (8 * VEC);
    for (int e = threadIdx.x; e < dpad; e += blockDim.x) sq[e] = e < dq ? Q[(int64_t)q * dq + e] : 0.f;
    if (threadIdx.x == 0) { s_cnt = 0; s_thr = ~0ull; }
    int64_t nc = ncand;
    if (ncand_per_q) nc = min((int64_t)ncand_per_q[q], cand_ld);
    const int64_t t0 = (int64_t)blockIdx.y * slice;
    const int64_t t1 = min(nc, t0 + slice);
    const int32_t *cl = cand ? cand + (int64_t)q * cand_ld : nullptr;
    const float *ql = sq + sub * VEC;
    const int rem = d - sub * VEC;
    __syncthreads();
    for (int64_t base = t0; base < t1; base += kRrRound) {
        // ids of this warp's 32 rows (one coalesced load)
        const int64_t tw = base + warp * 32 + lane;
        int myid = -1;
        if (tw < t1) myid = cl ? cl[tw] : (int)(tw * stride);
#pragma unroll 1
        for (int st = 0; st < 8; ++st) {
            const int id = __shfl_sync(NR_FULL, myid, st * 4 + grp);
            float acc = 0.f;
            if (id >= 0) {
                const float *xl = X + (int64_t)id * d + sub * VEC;
                acc = NIT > 0 ? row_dot<VEC, (NIT > 0 ? NIT : 1)>(xl, ql, rem)
                              : row_dot_any<VEC>(xl, ql, rem);
            }
            acc += __shfl_xor_sync(NR_FULL, acc, 1);
            acc += __shfl_xor_sync(NR_FULL, acc, 2);
            acc += __shfl_xor_sync(NR_FULL, acc, 4);
            if (sub == 0 && id >= 0) {
                const unsigned long long key = topk_key(acc, (uint32_t)id);
                if (key < *((volatile unsigned long long *)&s_thr)) {
                    const unsigned slot = atomicAdd(&s_cnt, 1u);
                    buf[slot] = key;
                }
            }
        }
        __syncthreads();
        if (s_cnt > (unsigned)(cap - kRrRound)) {   // compact: keep the k best
            const int c = (int)s_cnt;
            for (int e = c + threadIdx.x; e < cap; e += blockDim.x) buf[e] = ~0ull;
            __syncthreads();
            bitonic_sort_smem(buf, cap);
            if (threadIdx.x == 0) {
                s_cnt = (unsigned)min(c, k);
                if (c >= k) s_thr = buf[k - 1];
            }
            __syncthreads();
        }
    }
    __syncthreads();
    const int c = (int)s_cnt;
    int np2 = 2;   // sort only the collected entries (padded to a power of two)
    while (np2 < c) np2 <<= 1;
    for (int e = c + threadIdx.x; e < np2; e += blockDim.x) buf[e] = ~0ull;
    __syncthreads();
    bitonic_sort_smem(buf, np2);
    if (partial) {
        unsigned long long *pp = partial + ((int64_t)q * gridDim.y + blockIdx.y) * k;
        for (int t = threadIdx.x; t < k; t += blockDim.x) pp[t] = t < c ? buf[t] : ~0ull;
    } else {
        for (int t = threadIdx.x; t < k; t += blockDim.x) {
            const unsigned long long v = t < c ? buf[t] : ~0ull;
            out_ids[(int64_t)q * k + t] = v == ~0ull ? -1 : (int64_t)(uint32_t)v;
            out_scores[(int64_t)q * k + t] = v == ~0ull ? -INFINITY : float_unorder(~(uint32_t)(v >> 32));
        }
    }
}

// merge the gy partial top-k lists of each query
__global__ void __launch_bounds__(256) k8_rerank_merge(const unsigned long long *__restrict__ partial,
                                                       int gy, int k, int np2,
                                                       int64_t *__restrict__ out_ids,
                                                       float *__restrict__ out_scores) {
    pdl_wait();
    extern __shared__ unsigned long long mk[];
    const int q = blockIdx.x;
    const int tot = gy * k;
    for (int e = threadIdx.x; e < np2; e += blockDim.x)
        mk[e] = e < tot ? partial[(int64_t)q * tot + e] : ~0ull;
    __syncthreads();
    bitonic_sort_smem(mk, np2);
    for (int t = threadIdx.x; t < k; t += blockDim.x) {
        const unsigned long long v = mk[t];
        out_ids[(int64_t)q * k + t] = v == ~0ull ? -1 : (int64_t)(uint32_t)v;
        out_scores[(int64_t)q * k + t] = v == ~0ull ? -INFINITY : float_unorder(~(uint32_t)(v >> 32));
    }
}

static int pow2_at_least(int64_t v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

// Partial-list capacity for ANY sub-batch of at most Qmax queries: launch_rerank picks
// gy <= max(1, 8 SMs' worth / Qb), so Qb * gy <= max(Qmax, 8 * sms).  (Sizing it for
// Qmax alone under-allocates the smaller last sub-batch, which splits finer.)
size_t rerank_partial_bytes(int Qmax, int64_t ncand, int k) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t rounds = std::max<int64_t>(1, (ncand + kRrRound - 1) / kRrRound);
    if (rounds <= 1) return 0;
    return (size_t)std::max(Qmax, sms * 8) * k * 8;
}

void launch_rerank(const float *X, int d, int ldx, const float *Q, int Qb, const int32_t *cand,
                   int64_t ncand, int64_t cand_ld, const uint32_t *ncand_per_q, int stride,
                   int k, unsigned long long *partial, int64_t *out_ids, float *out_scores,
                   cudaStream_t s) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t rounds = std::max<int64_t>(1, (ncand + kRrRound - 1) / kRrRound);
    int gy = (int)std::min<int64_t>(rounds, std::max(1, (sms * 8) / std::max(1, Qb)));
    gy = std::min(gy, std::max(1, 8192 / k));
    if (!partial) gy = 1;
    const int64_t slice = ((rounds + gy - 1) / gy) * kRrRound;
    gy = (int)std::max<int64_t>(1, (ncand + slice - 1) / slice);
    const int cap = pow2_at_least(k + 2 * kRrRound);
    // (the kernel sees row length ldx and query length d)
    const int vec = (ldx % 4 == 0) ? 4 : ((ldx % 2 == 0) ? 2 : 1);
    const int dpad = (ldx + 8 * vec - 1) / (8 * vec) * (8 * vec);
    const size_t sm = (size_t)cap * 8 + (size_t)dpad * 4;
    unsigned long long *pp = gy > 1 ? partial : nullptr;
    dim3 grid(Qb, gy);
    const int nit = dpad / (8 * vec);
#define NR_RR(V, N)                                                                            \
    do {                                                                                       \
        cudaFuncSetAttribute(k8_rerank<V, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                             (int)sm);                                                         \
        launch_pdl(k8_rerank<V, N>, dim3(grid), dim3(kRrThreads), sm, s, X, ldx, d, Q, cand, cand_ld, ncand,       \
                                                     ncand_per_q, stride, k, cap, slice, pp,   \
                                                     out_ids, out_scores);                     \
    } while (0)
#define NR_RR_V(V)                                                                             \
    switch (nit) {                                                                             \
        case 1: NR_RR(V, 1); break;   case 2: NR_RR(V, 2); break;                              \
        case 3: NR_RR(V, 3); break;   case 4: NR_RR(V, 4); break;                              \
        case 5: NR_RR(V, 5); break;   case 6: NR_RR(V, 6); break;                              \
        case 7: NR_RR(V, 7); break;   case 8: NR_RR(V, 8); break;                              \
        case 9: NR_RR(V, 9); break;   case 10: NR_RR(V, 10); break;                            \
        case 11: NR_RR(V, 11); break; case 12: NR_RR(V, 12); break;                            \
        default: NR_RR(V, 0); break;                                                           \
    }
    if (vec == 4) { NR_RR_V(4) } else if (vec == 2) { NR_RR_V(2) } else { NR_RR_V(1) }
#undef NR_RR_V
#undef NR_RR
    note_launch();
    if (gy > 1) {
        const int np2 = pow2_at_least((int64_t)gy * k);
        cudaFuncSetAttribute(k8_rerank_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, np2 * 8);
        launch_pdl(k8_rerank_merge, dim3(Qb), dim3(256), (size_t)np2 * 8, s, partial, gy, k, np2, out_ids, out_scores);
        note_launch();
    }
}


}  // namespace nrlsh
