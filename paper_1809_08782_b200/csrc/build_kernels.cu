// build_kernels.cu — index building kernels (Alg. 1) for sm_100a.
//
//  K1  norms:      ||x_i||^2 in fp64, sequential over k (bit-identical to the
//                  plain definition; Alg. 1 l.3).  HBM stream of X.
//  K2  partition:  exact multi-select of the m-1 percentile boundaries on the
//                  (norm2 bits, id) keys (Alg. 1 l.4; ties by id,
//                  PAPER:173), then a stable scatter into sub-dataset order.
//  K3  codes:      y = X A[:d] + A[d] t,  t = sqrt(V_j - ||x||^2)  (the
//                  SIMPLE-LSH transform of Eq. (8) scaled by U_j > 0), bit =
//                  [y >= 0] (Eq. (4)), packed LSB-first, written at the item's
//                  position in sub-dataset order.
#include <algorithm>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include <cuda_bf16.h>

#include "common.cuh"
#include "internal.h"
#include "tc_sm100.cuh"

namespace nrlsh {

// =========================================================================== K1
// One CTA tile = RT rows.  Warps stage rows coalesced into shared memory (row
// stride ld odd -> conflict-free column walk), then thread r sums row r in
// order k = 0..d-1 in fp64 (each square is exact, so the result is the
// correctly-defined sequential sum).
template <int RT>
__global__ void __launch_bounds__(RT) k1_norms_tiled(const float *__restrict__ X, int64_t n, int d,
                                                     int ld, double *__restrict__ norm2,
                                                     unsigned long long *__restrict__ bad) {
    extern __shared__ float tile[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = RT / 32;
    for (int64_t base = (int64_t)blockIdx.x * RT; base < n; base += (int64_t)gridDim.x * RT) {
        const int rows = (int)min((int64_t)RT, n - base);
#pragma unroll 4
        for (int r = warp; r < rows; r += NW) {
            const float *src = X + (base + r) * (int64_t)d;
            for (int k = lane; k < d; k += 32) tile[r * ld + k] = __ldg(src + k);
        }
        __syncthreads();
        const int r = threadIdx.x;
        if (r < rows) {
            double s = 0.0;
            const float *t = tile + r * ld;
            for (int k = 0; k < d; ++k) {
                double v = (double)t[k];
                s = __dadd_rn(s, __dmul_rn(v, v));
            }
            norm2[base + r] = s;
            if (!isfinite(s)) atomicMin(bad, (unsigned long long)(base + r));
        }
        __syncthreads();
    }
}

// Very wide rows: one thread per row straight from global memory.
__global__ void k1_norms_direct(const float *__restrict__ X, int64_t n, int d,
                                double *__restrict__ norm2, unsigned long long *__restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float *src = X + i * (int64_t)d;
        double s = 0.0;
        for (int k = 0; k < d; ++k) {
            double v = (double)__ldg(src + k);
            s = __dadd_rn(s, __dmul_rn(v, v));
        }
        norm2[i] = s;
        if (!isfinite(s)) atomicMin(bad, (unsigned long long)i);
    }
}

// Streaming version: blocks of RT consecutive rows (one contiguous byte range of
// X) are bulk-copied (cp.async.bulk, 1-D TMA) into a 2-stage smem ring while the
// previous block is summed.  Thread r owns row r and adds x_r0^2, x_r1^2, ... in
// order; for even d the row stride makes a warp's lanes hit one bank, so lane r
// runs r steps behind lane 0 (element k at step k + r): banks (r(d-1) + step) mod
// 32 are distinct, and the order of the sum is unchanged.
__global__ void __launch_bounds__(128) k1_norms_bulk(const float *__restrict__ X, int64_t n, int d,
                                                     int RT, double *__restrict__ norm2,
                                                     unsigned long long *__restrict__ bad,
                                                     __nv_bfloat16 *__restrict__ Xb, int dpb,
                                                     float *__restrict__ xnorm,
                                                     unsigned long long *__restrict__ mm) {
    extern __shared__ __align__(128) float nbuf[];       // [2][RT * d]
    // (mm: smallest positive and largest key bits, for the percentile select's window)
    unsigned long long klo = ~0ull, khi = 0ull;
    __shared__ __align__(8) uint64_t full[2];
    const int64_t ntiles = (n + RT - 1) / RT;
    const int skew = (d % 2 == 0) ? 1 : 0;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        tc::mbar_init(&full[0], 1);
        tc::mbar_init(&full[1], 1);
        tc::fence_mbar_init();
    }
    __syncthreads();
    auto issue = [&](int64_t tile, int st) {
        const int64_t r0 = tile * RT;
        const int rows = (int)min((int64_t)RT, n - r0);
        const uint32_t bytes = (uint32_t)rows * d * 4;
        if ((bytes & 15u) == 0) {
            tc::mbar_arrive_expect_tx(&full[st], bytes);
            tc::bulk_load(nbuf + (size_t)st * RT * d, X + r0 * d, bytes, &full[st]);
        } else {
            tc::mbar_arrive(&full[st]);   // ragged tail: read straight from global
        }
    };
    int64_t tile = blockIdx.x;
    if (threadIdx.x == 0) {
        if (tile < ntiles) issue(tile, 0);
        if (tile + gridDim.x < ntiles) issue(tile + gridDim.x, 1);
    }
    for (uint32_t it = 0; tile < ntiles; ++it, tile += gridDim.x) {
        const int st = it & 1;
        tc::mbar_wait(&full[st], (it >> 1) & 1);
        const int64_t r0 = tile * RT;
        const int rows = (int)min((int64_t)RT, n - r0);
        const bool in_smem = (((uint32_t)rows * d * 4) & 15u) == 0;
        const float *src = in_smem ? nbuf + (size_t)st * RT * d : X + r0 * d;
        for (int r = threadIdx.x; r < RT; r += blockDim.x) {
            const float *row = src + (size_t)min(r, rows - 1) * d;
            const int lag = skew * lane;
            double s = 0.0;
            // k ascending (the oracle's order); v*v is exact, so each step rounds once,
            // as s + v*v.  Lane l runs l steps behind lane 0 when d is even (bank skew);
            // the middle section, where every lane has a valid k, is unrolled so its
            // shared-memory loads issue ahead of the dependent fma chain.
            if (skew && d >= 32) {
                for (int step = 0; step < 31; ++step) {
                    const int k = step - lag;
                    if (k >= 0) { const double v = (double)row[k]; s = __fma_rn(v, v, s); }
                }
                const float *p = row + 31 - lag;
#pragma unroll 8
                for (int t = 0; t < d - 31; ++t) { const double v = (double)p[t]; s = __fma_rn(v, v, s); }
                for (int step = d; step < d + 31; ++step) {
                    const int k = step - lag;
                    if (k < d) { const double v = (double)row[k]; s = __fma_rn(v, v, s); }
                }
            } else if (!skew) {
#pragma unroll 8
                for (int k = 0; k < d; ++k) { const double v = (double)row[k]; s = __fma_rn(v, v, s); }
            } else {
                for (int step = 0; step < d + 31; ++step) {
                    const int k = step - lag;
                    if (k >= 0 && k < d) { const double v = (double)row[k]; s = __fma_rn(v, v, s); }
                }
            }
            if (r < rows) {
                norm2[r0 + r] = s;
                const unsigned long long kb = (unsigned long long)__double_as_longlong(s);
                if (kb != 0ull) klo = kb < klo ? kb : klo;
                khi = kb > khi ? kb : khi;
                if (!isfinite(s)) atomicMin(bad, (unsigned long long)(r0 + r));
                // |x| rounded up (with a 2^-50 margin over the fp64 sum's rounding):
                // an upper bound for the certified bf16 filters
                if (xnorm) xnorm[r0 + r] = __double2float_ru(sqrt(s) * (1.0 + 0x1p-50));
            }
        }

        __syncthreads();                            // stage st fully read
        if (threadIdx.x == 0 && tile + 2 * (int64_t)gridDim.x < ntiles)
            issue(tile + 2 * (int64_t)gridDim.x, st);
    }
    if (mm) {
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long l2 = __shfl_xor_sync(NR_FULL, klo, o);
            const unsigned long long h2 = __shfl_xor_sync(NR_FULL, khi, o);
            klo = l2 < klo ? l2 : klo;
            khi = h2 > khi ? h2 : khi;
        }
        if (lane == 0) {
            if (klo != ~0ull) atomicMin(&mm[0], klo);
            atomicMax(&mm[1], khi);
        }
    }
}

bool launch_norms(const float *X, int64_t n, int d, double *norm2, unsigned long long *bad,
                  void *Xb, int dpb, float *xnorm, cudaStream_t s, unsigned long long *mm) {
    const int ld = (d % 2 == 1) ? d : d + 1;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // rows per tile: two stages of <= 120 KB, a multiple of 32, at most 96 (c4,
    // d = 150: 96 rows, one CTA per SM, 0.30 ms; 64 rows, two CTAs, 0.385 ms)
    int RT = (int)std::min<int64_t>(96, std::max<int64_t>(32, (120 * 1024 / (8 * (int64_t)d)) / 32 * 32));
    if (getenv("NRLSH_NORMS_RT")) RT = std::max(32, std::min(128, atoi(getenv("NRLSH_NORMS_RT")) / 32 * 32));
    if (((uintptr_t)X & 15u) == 0 && (size_t)2 * RT * d * 4 <= 200 * 1024 && !getenv("NRLSH_NORMS_OLD")) {
        const size_t sm = (size_t)2 * RT * d * 4;
        cudaFuncSetAttribute(k1_norms_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        const int64_t ntiles = (n + RT - 1) / RT;
        const int per_sm = std::max(1, (int)((227 * 1024) / (sm + 1024)));
        const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sms * per_sm);
        k1_norms_bulk<<<grid, RT, sm, s>>>(X, n, d, RT, norm2, bad, nullptr, dpb, xnorm, mm);
        note_launch();
        return mm != nullptr;
    }
    const size_t lim = 200 * 1024;
    if ((size_t)256 * ld * 4 <= lim / 2) {
        size_t sm = (size_t)256 * ld * 4;
        cudaFuncSetAttribute(k1_norms_tiled<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k1_norms_tiled<256><<<grid_for(n, 256, sms * 8), 256, sm, s>>>(X, n, d, ld, norm2, bad);
    } else if ((size_t)128 * ld * 4 <= lim) {
        size_t sm = (size_t)128 * ld * 4;
        cudaFuncSetAttribute(k1_norms_tiled<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k1_norms_tiled<128><<<grid_for(n, 128, sms * 8), 128, sm, s>>>(X, n, d, ld, norm2, bad);
    } else if ((size_t)32 * ld * 4 <= lim) {
        size_t sm = (size_t)32 * ld * 4;
        cudaFuncSetAttribute(k1_norms_tiled<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k1_norms_tiled<32><<<grid_for(n, 32, sms * 16), 32, sm, s>>>(X, n, d, ld, norm2, bad);
    } else {
        k1_norms_direct<<<grid_for(n, 256, sms * 8), 256, 0, s>>>(X, n, d, norm2, bad);
    }
    note_launch();
    return false;
}

// =========================================================================== K2
// Exact multi-select.  The 96-bit composite key c_i = (bits(norm2_i) : id_i) is
// unique and its unsigned order is the ranking order of Alg. 1 (norm2 >= 0, so
// the IEEE bit pattern is monotone).  Rank r goes to sub-dataset floor(r m / n);
// boundary b_j = ceil(j n / m) is the first rank of sub-dataset j.  A level
// histograms one digit of c over a candidate list, locates the boundaries, and
// (i) assigns every item of a bin that no boundary splits directly, (ii) moves
// items of split bins into per-bin sub-lists, which are either sorted in shared
// memory (small) or refined by the next digit (large).
struct SelGroup {
    uint32_t bin;
    uint32_t count;
    int64_t base;     // rank of the bin's first item
    int64_t cand_off; // offset of the bin's sub-list
};

struct SelLevel {
    int shift, width;
};
// digits over bits 95..0 of (key64 : id32), most significant first
static const SelLevel kLevels[] = {{72, 24}, {56, 16}, {40, 16}, {32, 8}, {16, 16}, {0, 16}};
constexpr int kNumLevels = 6;
constexpr int kSmallGroup = 2048;
constexpr int kMaxGroups = kMaxParts;

__device__ __forceinline__ uint32_t digit96(uint64_t key, uint32_t id, int shift, int width) {
    const uint32_t mask = (width >= 32) ? 0xffffffffu : ((1u << width) - 1u);
    if (shift >= 32) return (uint32_t)(key >> (shift - 32)) & mask;
    return (id >> shift) & mask;
}

template <bool Implicit>
__device__ __forceinline__ void load_item(const double *norm2, const uint64_t *keys,
                                          const uint32_t *ids, int64_t i, uint64_t &key,
                                          uint32_t &id) {
    if (Implicit) {
        key = (uint64_t)__double_as_longlong(norm2[i]);
        id = (uint32_t)i;
    } else {
        key = keys[i];
        id = ids[i];
    }
}

template <bool Implicit>
__global__ void sel_hist(const double *__restrict__ norm2, const uint64_t *__restrict__ keys,
                         const uint32_t *__restrict__ ids, int64_t count, int shift, int width,
                         uint32_t *__restrict__ H) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key;
        uint32_t id;
        load_item<Implicit>(norm2, keys, ids, i, key, id);
        atomicAdd(&H[digit96(key, id, shift, width)], 1u);
    }
}

// 3-phase exclusive scan of uint32 (nbins <= 4096 * 4096).
__global__ void __launch_bounds__(1024) scan_tiles(const uint32_t *__restrict__ in,
                                                   uint32_t *__restrict__ out, int64_t nbins,
                                                   uint32_t *__restrict__ tile_sums) {
    __shared__ uint32_t ws[32];
    const int64_t base = (int64_t)blockIdx.x * 4096 + threadIdx.x * 4;
    uint32_t v[4];
    uint32_t loc = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        v[e] = (base + e < nbins) ? in[base + e] : 0u;
        loc += v[e];
    }
    uint32_t tot;
    uint32_t ex = block_excl_scan(loc, ws, &tot);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        if (base + e < nbins) out[base + e] = ex;
        ex += v[e];
    }
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) scan_sums(uint32_t *__restrict__ tile_sums, int ntiles) {
    __shared__ uint32_t ws[32];
    uint32_t v[4];
    uint32_t loc = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        int t = threadIdx.x * 4 + e;
        v[e] = t < ntiles ? tile_sums[t] : 0u;
        loc += v[e];
    }
    uint32_t ex = block_excl_scan(loc, ws, nullptr);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        int t = threadIdx.x * 4 + e;
        if (t < ntiles) tile_sums[t] = ex;
        ex += v[e];
    }
}

__global__ void scan_add(uint32_t *__restrict__ out, int64_t nbins,
                         const uint32_t *__restrict__ tile_sums) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < nbins) out[i] += tile_sums[i / 4096];
}

static void scan_excl(const uint32_t *in, uint32_t *out, int64_t nbins, uint32_t *tile_sums,
                      cudaStream_t s) {
    const int ntiles = (int)((nbins + 4095) / 4096);
    scan_tiles<<<ntiles, 1024, 0, s>>>(in, out, nbins, tile_sums);
    if (ntiles > 1) {
        scan_sums<<<1, 1024, 0, s>>>(tile_sums, ntiles);
        scan_add<<<(int)((nbins + 255) / 256), 256, 0, s>>>(out, nbins, tile_sums);
    }
}

// Locate the boundaries inside [base, base+count) and list the bins they split.
// One block of >= m threads.  out_meta[0] = ngroups, out_meta[1] = total candidates.
__global__ void sel_locate(const uint32_t *__restrict__ H, const uint32_t *__restrict__ P,
                           int64_t nbins, int64_t base, int64_t count, int64_t n, int m,
                           SelGroup *__restrict__ groups, int64_t *__restrict__ out_meta) {
    __shared__ int64_t sbin[kMaxParts];
    const int j = threadIdx.x;
    if (j < m) {
        sbin[j] = -1;
        if (j >= 1) {
            const int64_t b = (j * n + m - 1) / m;   // ceil(j n / m)
            if (b > base && b < base + count) {      // boundary strictly inside the list
                const uint32_t loc = (uint32_t)(b - base);
                int64_t lo = 0, hi = nbins - 1;      // largest bin with P[bin] <= loc
                while (lo < hi) {
                    int64_t mid = (lo + hi + 1) >> 1;
                    if (P[mid] <= loc) lo = mid; else hi = mid - 1;
                }
                // the bin containing rank loc; it is split only if loc is not its first rank
                if (P[lo] < loc) sbin[j] = lo;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int g = 0;
        int64_t last = -1, off = 0;
        for (int jj = 1; jj < m; ++jj) {
            int64_t bn = sbin[jj];
            if (bn < 0 || bn == last) continue;
            last = bn;
            groups[g].bin = (uint32_t)bn;
            groups[g].count = H[bn];
            groups[g].base = base + P[bn];
            groups[g].cand_off = off;
            off += H[bn];
            ++g;
        }
        out_meta[0] = g;
        out_meta[1] = off;
    }
}

template <bool Implicit>
__global__ void sel_classify(const double *__restrict__ norm2, const uint64_t *__restrict__ keys,
                             const uint32_t *__restrict__ ids, int64_t count, int shift,
                             int width, const uint32_t *__restrict__ P, int64_t base, int64_t n,
                             int m, const SelGroup *__restrict__ groups,
                             const int64_t *__restrict__ meta, uint32_t *__restrict__ fill,
                             uint64_t *__restrict__ out_keys, uint32_t *__restrict__ out_ids,
                             uint8_t *__restrict__ part) {
    __shared__ uint32_t gbin[kMaxGroups];
    __shared__ int64_t goff[kMaxGroups];
    const int ng = (int)meta[0];
    for (int g = threadIdx.x; g < ng; g += blockDim.x) {
        gbin[g] = groups[g].bin;
        goff[g] = groups[g].cand_off;
    }
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t key;
        uint32_t id;
        load_item<Implicit>(norm2, keys, ids, i, key, id);
        const uint32_t dg = digit96(key, id, shift, width);
        int lo = 0, hi = ng;   // first group with bin >= dg
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if (gbin[mid] < dg) lo = mid + 1; else hi = mid;
        }
        if (lo < ng && gbin[lo] == dg) {
            const uint32_t slot = atomicAdd(&fill[lo], 1u);
            out_keys[goff[lo] + slot] = key;
            out_ids[goff[lo] + slot] = id;
        } else {
            const int64_t r = base + (int64_t)P[dg];
            part[id] = (uint8_t)((r * m) / n);
        }
    }
}

// Sort each small group's (key, id) list in shared memory and assign ranks.
__global__ void __launch_bounds__(1024) sel_resolve_small(
    const SelGroup *__restrict__ groups, const int *__restrict__ gidx,
    const uint64_t *__restrict__ keys, const uint32_t *__restrict__ ids, int64_t n, int m,
    uint8_t *__restrict__ part) {
    __shared__ uint64_t sk[kSmallGroup];
    __shared__ uint32_t si[kSmallGroup];
    const SelGroup g = groups[gidx[blockIdx.x]];
    const int cnt = (int)g.count;
    int np2 = 1;
    while (np2 < cnt) np2 <<= 1;
    for (int t = threadIdx.x; t < np2; t += blockDim.x) {
        if (t < cnt) {
            sk[t] = keys[g.cand_off + t];
            si[t] = ids[g.cand_off + t];
        } else {
            sk[t] = ~0ull;
            si[t] = 0xffffffffu;
        }
    }
    __syncthreads();
    for (int size = 2; size <= np2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < np2; t += blockDim.x) {
                const int o = t ^ stride;
                if (o > t) {
                    const bool up = ((t & size) == 0);
                    const bool gt = (sk[t] > sk[o]) || (sk[t] == sk[o] && si[t] > si[o]);
                    if (gt == up) {
                        uint64_t tk = sk[t]; sk[t] = sk[o]; sk[o] = tk;
                        uint32_t ti = si[t]; si[t] = si[o]; si[o] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
        const int64_t r = g.base + t;
        part[si[t]] = (uint8_t)((r * m) / n);
    }
}

// Device-decided resolution of the level-0 groups (no host round trip): block g
// sorts group g if it exists and is small; a larger group sets *large (the host then
// redoes the partition with the multi-level path).
__global__ void __launch_bounds__(1024) sel_resolve_dev(
    const SelGroup *__restrict__ groups, const int64_t *__restrict__ meta,
    const uint64_t *__restrict__ keys, const uint32_t *__restrict__ ids, int64_t n, int m,
    uint8_t *__restrict__ part, unsigned int *__restrict__ large) {
    __shared__ uint64_t sk[kSmallGroup];
    __shared__ uint32_t si[kSmallGroup];
    if ((int64_t)blockIdx.x >= meta[0]) return;
    const SelGroup g = groups[blockIdx.x];
    const int cnt = (int)g.count;
    if (g.count > (uint32_t)kSmallGroup) {
        if (threadIdx.x == 0) atomicOr(large, 1u);
        return;
    }
    int np2 = 1;
    while (np2 < cnt) np2 <<= 1;
    for (int t = threadIdx.x; t < np2; t += blockDim.x) {
        if (t < cnt) {
            sk[t] = keys[g.cand_off + t];
            si[t] = ids[g.cand_off + t];
        } else {
            sk[t] = ~0ull;
            si[t] = 0xffffffffu;
        }
    }
    __syncthreads();
    for (int size = 2; size <= np2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < np2; t += blockDim.x) {
                const int o = t ^ stride;
                if (o > t) {
                    const bool up = ((t & size) == 0);
                    const bool gt = (sk[t] > sk[o]) || (sk[t] == sk[o] && si[t] > si[o]);
                    if (gt == up) {
                        uint64_t tk = sk[t]; sk[t] = sk[o]; sk[o] = tk;
                        uint32_t ti = si[t]; si[t] = si[o]; si[o] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) {
        const int64_t r = g.base + t;
        part[si[t]] = (uint8_t)((r * m) / n);
    }
}

namespace {
// stream-ordered scratch (memory pool): no device-wide synchronisation on free
struct DevBuf {
    void *p = nullptr;
    cudaStream_t s = nullptr;
    explicit DevBuf(cudaStream_t st = nullptr) : s(st) {}
    ~DevBuf() { if (p) cudaFreeAsync(p, s); }
    template <class T> T *get() { return (T *)p; }
    cudaError_t alloc(size_t bytes) {
        if (p) { cudaFreeAsync(p, s); p = nullptr; }
        return dmalloc(&p, bytes ? bytes : 16, s);
    }
};
}  // namespace

// ---------------------------------------------------------------- windowed level 0
// The device-decided level 0 bins the fp64 key by its bits above `shift` relative to
// the smallest positive key (zeros, the only keys below it, go to bin 0 — the binning
// stays monotone).  shift >= 40 (12 mantissa bits: ~80 items per bin at the mode of a
// lognormal(0, 1) norm law on 2.3M items) is raised until the keys' range fits
// 2^kWinBits bins, so the histogram is 1 MB instead of the 2^24 bins of a fixed digit.
constexpr int kWinBits = 18;
constexpr int kWinFinePerCoarse = 1024;
constexpr int kWinCoarse = (1 << kWinBits) / kWinFinePerCoarse;   // 256

__device__ __forceinline__ void win_params(const unsigned long long *mm, int &shift,
                                           unsigned long long &base) {
    unsigned long long lo = mm[0], hi = mm[1];
    if (lo == ~0ull) lo = 0ull;   // (no positive key)
    if (hi < lo) hi = lo;
    int sh = 40;
    while (((hi >> sh) - (lo >> sh)) >= (1ull << kWinBits)) ++sh;
    shift = sh;
    base = lo >> sh;
}

__device__ __forceinline__ uint32_t win_bin(unsigned long long key, int shift, unsigned long long base) {
    const unsigned long long b = key >> shift;
    return b < base ? 0u : (uint32_t)(b - base);
}

// mm[0] = smallest positive key (init ~0), mm[1] = largest key (init 0)
__global__ void win_minmax(const double *__restrict__ norm2, int64_t n, unsigned long long *__restrict__ mm) {
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(norm2[i]);
        if (b != 0ull) lo = b < lo ? b : lo;
        hi = b > hi ? b : hi;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long l2 = __shfl_xor_sync(NR_FULL, lo, o);
        const unsigned long long h2 = __shfl_xor_sync(NR_FULL, hi, o);
        lo = l2 < lo ? l2 : lo;
        hi = h2 > hi ? h2 : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        if (lo != ~0ull) atomicMin(&mm[0], lo);
        atomicMax(&mm[1], hi);
    }
}

// fine histogram H [2^kWinBits] (global atomics; keys in item order are spread over
// the bins, so a warp's atomics rarely collide)
__global__ void __launch_bounds__(256) win_hist(const double *__restrict__ norm2, int64_t n,
                                                const unsigned long long *__restrict__ mm,
                                                uint32_t *__restrict__ H) {
    int shift;
    unsigned long long base;
    win_params(mm, shift, base);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&H[win_bin((unsigned long long)__double_as_longlong(norm2[i]), shift, base)], 1u);
}

// coarse sums: CTA c adds the kWinFinePerCoarse fine counts of coarse bin c
__global__ void __launch_bounds__(256) win_coarse(const uint32_t *__restrict__ H, uint32_t *__restrict__ Hc) {
    __shared__ uint32_t ws[32];
    const uint4 v = reinterpret_cast<const uint4 *>(H + (size_t)blockIdx.x * kWinFinePerCoarse)[threadIdx.x];
    uint32_t tot;
    block_excl_scan(v.x + v.y + v.z + v.w, ws, &tot);
    if (threadIdx.x == 0) Hc[blockIdx.x] = tot;
}

// One CTA of 1024 threads.  Boundary j (first rank b_j = ceil(j n / m)) lies in the
// coarse bin whose prefix brackets b_j and, inside it, in the fine bin a warp finds
// by a prefix over the coarse bin's 1024 fine counts.  The bins a boundary falls
// strictly inside become the groups (sorted later); bt/btg give every boundary's bin
// and its group (-1: the boundary is the bin's first rank, the bin is not split).
__global__ void __launch_bounds__(1024) win_locate(const uint32_t *__restrict__ H,
                                                   const uint32_t *__restrict__ Hc, int64_t n, int m,
                                                   SelGroup *__restrict__ groups,
                                                   int64_t *__restrict__ meta,
                                                   uint32_t *__restrict__ bt, int32_t *__restrict__ btg) {
    __shared__ uint32_t ws[32];
    __shared__ uint32_t pc[kWinCoarse];
    __shared__ uint32_t sbin[kMaxParts], sP[kMaxParts];
    __shared__ int32_t sg[kMaxParts];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t v = threadIdx.x < kWinCoarse ? Hc[threadIdx.x] : 0u;
    const uint32_t ex = block_excl_scan(v, ws, nullptr);
    if (threadIdx.x < kWinCoarse) pc[threadIdx.x] = ex;
    __syncthreads();
    for (int j = 1 + warp; j < m; j += 32) {
        const uint32_t b = (uint32_t)(((int64_t)j * n + m - 1) / m);
        int lo = 0, hi = kWinCoarse - 1;   // largest coarse bin with prefix <= b
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pc[mid] <= b) lo = mid; else hi = mid - 1;
        }
        const uint4 *hf = reinterpret_cast<const uint4 *>(H + (size_t)lo * kWinFinePerCoarse + lane * 32);
        uint32_t hv[32];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const uint4 x = hf[e];
            hv[4 * e] = x.x; hv[4 * e + 1] = x.y; hv[4 * e + 2] = x.z; hv[4 * e + 3] = x.w;
        }
        uint32_t sum = 0;
#pragma unroll
        for (int e = 0; e < 32; ++e) sum += hv[e];
        uint32_t inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(NR_FULL, inc, o);
            if (lane >= o) inc += y;
        }
        const uint32_t lex = pc[lo] + inc - sum;   // rank of the first item of this lane's bins
        if (lex <= b && b < lex + sum) {
            uint32_t r = lex;
            int e = 0;
            for (; e < 31; ++e) {
                if (b < r + hv[e]) break;
                r += hv[e];
            }
            sbin[j] = (uint32_t)lo * kWinFinePerCoarse + lane * 32 + e;
            sP[j] = r;
        }
    }
    __syncthreads();
    // a bin is split if some boundary lies strictly inside it; the boundaries of one
    // bin are consecutive in j.  Group g = the g-th split bin (leader: its first
    // boundary), its list at the exclusive sum of the earlier groups' counts.
    const int j = threadIdx.x;
    bool leader = false;
    uint32_t cntb = 0;
    if (j >= 1 && j < m) {
        const uint32_t bn = sbin[j];
        int j0 = j, j1 = j;
        while (j0 > 1 && sbin[j0 - 1] == bn) --j0;
        while (j1 + 1 < m && sbin[j1 + 1] == bn) ++j1;
        bool split = false;
        for (int jj = j0; jj <= j1; ++jj)
            split |= sP[jj] < (uint32_t)(((int64_t)jj * n + m - 1) / m);
        leader = split && j == j0;
        sg[j] = split ? -2 - j0 : -1;   // (resolved to the leader's group below)
        if (leader) cntb = H[bn];
    }
    uint32_t ng;
    const uint32_t gi = block_excl_scan(leader ? 1u : 0u, ws, &ng);
    uint32_t off_tot;
    const uint32_t go = block_excl_scan(cntb, ws, &off_tot);
    if (leader) {
        groups[gi].bin = sbin[j];
        groups[gi].count = cntb;
        groups[gi].base = sP[j];
        groups[gi].cand_off = go;
        sP[j] = gi;   // (this boundary's rank is no longer needed: hand over the group)
    }
    __syncthreads();
    if (j >= 1 && j < m) {
        bt[j - 1] = sbin[j];
        btg[j - 1] = sg[j] <= -2 ? (int32_t)sP[-2 - sg[j]] : -1;
    }
    if (j == 0) {
        meta[0] = ng;
        meta[1] = off_tot;
    }
}

// Items of split bins go to their group's list; every other item's sub-dataset is the
// number of boundaries whose bin is <= its bin (those all rank at or before it).
__global__ void __launch_bounds__(256) win_classify(const double *__restrict__ norm2, int64_t n, int m,
                                                    const unsigned long long *__restrict__ mm,
                                                    const uint32_t *__restrict__ bt,
                                                    const int32_t *__restrict__ btg,
                                                    const SelGroup *__restrict__ groups,
                                                    uint32_t *__restrict__ fill,
                                                    uint64_t *__restrict__ out_keys,
                                                    uint32_t *__restrict__ out_ids,
                                                    uint8_t *__restrict__ part) {
    __shared__ uint32_t sbt[kMaxParts];
    __shared__ int32_t sbg[kMaxParts];
    __shared__ int64_t goff[kMaxParts];
    const int nb = m - 1;
    for (int t = threadIdx.x; t < nb; t += blockDim.x) {
        sbt[t] = bt[t];
        const int g = btg[t];
        sbg[t] = g;
        if (g >= 0) goff[g] = groups[g].cand_off;
    }
    int shift;
    unsigned long long base;
    win_params(mm, shift, base);
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t key = (uint64_t)__double_as_longlong(norm2[i]);
        const uint32_t b = win_bin(key, shift, base);
        int lo = 0, hi = nb;   // number of boundary bins <= b
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sbt[mid] <= b) lo = mid + 1; else hi = mid;
        }
        const int g = (lo > 0 && sbt[lo - 1] == b) ? sbg[lo - 1] : -1;
        // (an item of a split bin gets its exact sub-dataset from the group sort; the
        // provisional lo keeps part[] in range if that sort is left to the host's
        // multi-level select — the scatter still runs on it before the redo)
        part[i] = (uint8_t)lo;
        if (g >= 0) {
            const uint32_t slot = atomicAdd(&fill[g], 1u);
            out_keys[goff[g] + slot] = key;
            out_ids[goff[g] + slot] = (uint32_t)i;
        }
    }
}

// One level of the exact multi-select, decided on the device: the first digit's
// histogram, the boundary groups, direct assignment outside them and an in-smem sort
// of each group (<= kSmallGroup items; continuous norms — every BASELINE config —
// leave only such groups).  No host synchronisation; *large (device) is set when a
// group is larger, and the caller then runs partition_percentile.
int partition_percentile_fast(const double *norm2, int64_t n, int m, uint8_t *part,
                              unsigned int *large, cudaStream_t s, std::string *err,
                              const unsigned long long *mm_in) {
    if (m == 1) {
        cudaMemsetAsync(part, 0, (size_t)n, s);
        return 0;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // zeroed scratch: [mm 16 B | Hc | fill | bt | btg | H]
    const size_t hdr = 16 + (size_t)kWinCoarse * 4 + (size_t)kMaxGroups * 4 + 2 * (size_t)kMaxParts * 4;
    const size_t zbytes = hdr + ((size_t)1 << kWinBits) * 4;
    DevBuf Z(s), G(s), META(s), KB(s), IB(s);
    if (Z.alloc(zbytes) || G.alloc(sizeof(SelGroup) * kMaxGroups) || META.alloc(16) ||
        KB.alloc((size_t)n * 8) || IB.alloc((size_t)n * 4)) {
        *err = "partition: cudaMalloc failed";
        return NRLSH_ENOMEM;
    }
    uint8_t *z = Z.get<uint8_t>();
    unsigned long long *mm = (unsigned long long *)z;
    uint32_t *Hc = (uint32_t *)(z + 16);
    uint32_t *fill = Hc + kWinCoarse;
    uint32_t *bt = fill + kMaxGroups;
    int32_t *btg = (int32_t *)(bt + kMaxParts);
    uint32_t *H = (uint32_t *)(z + hdr);
    cudaMemsetAsync(z, 0, zbytes, s);
    cudaMemsetAsync(z, 0xff, 8, s);
    if (mm_in) mm = const_cast<unsigned long long *>(mm_in);   // (the norms pass's min / max)
    else win_minmax<<<sms * 4, 256, 0, s>>>(norm2, n, mm);
    const int grid = grid_for(n, 256, sms * 8);
    win_hist<<<grid, 256, 0, s>>>(norm2, n, mm, H);
    win_coarse<<<kWinCoarse, kWinFinePerCoarse / 4, 0, s>>>(H, Hc);
    win_locate<<<1, 1024, 0, s>>>(H, Hc, n, m, G.get<SelGroup>(), META.get<int64_t>(), bt, btg);
    win_classify<<<grid, 256, 0, s>>>(norm2, n, m, mm, bt, btg, G.get<SelGroup>(), fill,
                                      KB.get<uint64_t>(), IB.get<uint32_t>(), part);
    sel_resolve_dev<<<kMaxGroups, 1024, 0, s>>>(G.get<SelGroup>(), META.get<int64_t>(), KB.get<uint64_t>(),
                                               IB.get<uint32_t>(), n, m, part, large);
    note_launch(mm_in ? 5 : 6);
    return 0;
}

int partition_percentile(const double *norm2, int64_t n, int m, uint8_t *part, cudaStream_t s,
                         std::string *err) {
    if (m == 1) {
        cudaMemsetAsync(part, 0, (size_t)n, s);
        return 0;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int64_t maxbins = 1ll << 24;
    DevBuf H(s), P(s), TS(s), G(s), META(s), FILL(s);
    if (H.alloc(maxbins * 4) || P.alloc(maxbins * 4) || TS.alloc(4096 * 4) ||
        G.alloc(sizeof(SelGroup) * kMaxGroups) || META.alloc(16) || FILL.alloc(kMaxGroups * 4)) {
        *err = "partition: cudaMalloc failed";
        return NRLSH_ENOMEM;
    }
    struct Problem {
        const uint64_t *keys;  // nullptr => implicit (all items)
        const uint32_t *ids;
        int64_t count, base;
        int level;
        std::shared_ptr<DevBuf> kbuf, ibuf;  // keep parent lists alive
    };
    std::vector<Problem> stack;
    stack.push_back({nullptr, nullptr, n, 0, 0, nullptr, nullptr});
    std::vector<SelGroup> hg(kMaxGroups);
    while (!stack.empty()) {
        Problem pb = stack.back();
        stack.pop_back();
        if (pb.level >= kNumLevels) {
            *err = "partition: exhausted key digits";
            return NRLSH_ECUDA;
        }
        const SelLevel lv = kLevels[pb.level];
        const int64_t nbins = 1ll << lv.width;
        cudaMemsetAsync(H.p, 0, nbins * 4, s);
        const int grid = grid_for(pb.count, 256, sms * 16);
        if (pb.keys == nullptr)
            sel_hist<true><<<grid, 256, 0, s>>>(norm2, nullptr, nullptr, pb.count, lv.shift,
                                                lv.width, H.get<uint32_t>());
        else
            sel_hist<false><<<grid, 256, 0, s>>>(nullptr, pb.keys, pb.ids, pb.count, lv.shift,
                                                 lv.width, H.get<uint32_t>());
        scan_excl(H.get<uint32_t>(), P.get<uint32_t>(), nbins, TS.get<uint32_t>(), s);
        note_launch(nbins > 4096 ? 5 : 3);
        sel_locate<<<1, kMaxParts, 0, s>>>(H.get<uint32_t>(), P.get<uint32_t>(), nbins, pb.base,
                                           pb.count, n, m, G.get<SelGroup>(), META.get<int64_t>());
        int64_t meta[2];
        cudaMemcpyAsync(meta, META.p, 16, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(hg.data(), G.p, sizeof(SelGroup) * kMaxGroups, cudaMemcpyDeviceToHost, s);
        cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            *err = std::string("partition: ") + cudaGetErrorString(e);
            return NRLSH_ECUDA;
        }
        const int ng = (int)meta[0];
        const int64_t tot = meta[1];
        auto kb = std::make_shared<DevBuf>(s);
        auto ib = std::make_shared<DevBuf>(s);
        if (kb->alloc(tot * 8) || ib->alloc(tot * 4)) {
            *err = "partition: cudaMalloc failed (candidates)";
            return NRLSH_ENOMEM;
        }
        cudaMemsetAsync(FILL.p, 0, kMaxGroups * 4, s);
        if (pb.keys == nullptr)
            sel_classify<true><<<grid, 256, 0, s>>>(
                norm2, nullptr, nullptr, pb.count, lv.shift, lv.width, P.get<uint32_t>(), pb.base,
                n, m, G.get<SelGroup>(), META.get<int64_t>(), FILL.get<uint32_t>(),
                kb->get<uint64_t>(), ib->get<uint32_t>(), part);
        else
            sel_classify<false><<<grid, 256, 0, s>>>(
                nullptr, pb.keys, pb.ids, pb.count, lv.shift, lv.width, P.get<uint32_t>(), pb.base,
                n, m, G.get<SelGroup>(), META.get<int64_t>(), FILL.get<uint32_t>(),
                kb->get<uint64_t>(), ib->get<uint32_t>(), part);
        if (ng == 0) continue;
        std::vector<int> small;
        for (int g = 0; g < ng; ++g) {
            if (hg[g].count <= (uint32_t)kSmallGroup) {
                small.push_back(g);
            } else {
                Problem ch;
                ch.keys = kb->get<uint64_t>() + hg[g].cand_off;
                ch.ids = ib->get<uint32_t>() + hg[g].cand_off;
                ch.count = hg[g].count;
                ch.base = hg[g].base;
                ch.level = pb.level + 1;
                ch.kbuf = kb;
                ch.ibuf = ib;
                stack.push_back(ch);
            }
        }
        if (!small.empty()) {
            // per-launch argument block: this level's group table + the small-group list
            DevBuf gi(s);
            const size_t gbytes = sizeof(SelGroup) * ng;
            if (gi.alloc(gbytes + small.size() * 4)) {
                *err = "partition: cudaMallocAsync failed";
                return NRLSH_ENOMEM;
            }
            cudaMemcpyAsync(gi.p, G.p, gbytes, cudaMemcpyDeviceToDevice, s);
            cudaMemcpyAsync((uint8_t *)gi.p + gbytes, small.data(), small.size() * 4,
                            cudaMemcpyHostToDevice, s);
            note_launch();
            sel_resolve_small<<<(int)small.size(), 1024, 0, s>>>(
                gi.get<SelGroup>(), (const int *)((uint8_t *)gi.p + gbytes), kb->get<uint64_t>(),
                ib->get<uint32_t>(), n, m, part);
            // (pageable H2D copies are staged before cudaMemcpyAsync returns)
        }
    }
    return 0;
}

// ------------------------------------------------------------- k-th of non-negative floats
// One CTA: 4 radix passes of 8 bits over the IEEE bit patterns (monotone for x >= 0).
__global__ void __launch_bounds__(1024) select_kth_float(const float *__restrict__ v, int64_t nt, int64_t r,
                                                         float *__restrict__ out) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_prefix, s_r;
    if (threadIdx.x == 0) { s_prefix = 0u; s_r = (uint32_t)r; }
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        const uint32_t pmask = pass == 0 ? 0u : (0xFFFFFFFFu << (shift + 8));
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0u;
        __syncthreads();
        const uint32_t prefix = s_prefix;
        for (int64_t i = threadIdx.x; i < nt; i += blockDim.x) {
            const uint32_t b = __float_as_uint(v[i]);
            if ((b & pmask) == prefix) atomicAdd(&hist[(b >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t rr = s_r, d = 0;
            while (d < 255 && hist[d] <= rr) { rr -= hist[d]; ++d; }
            s_r = rr;
            s_prefix = prefix | (d << shift);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = __uint_as_float(s_prefix);
}

void launch_select_kth_float(const float *v, int64_t nt, int64_t r, float *out, cudaStream_t s) {
    select_kth_float<<<1, 1024, 0, s>>>(v, nt, r, out);
    note_launch();
}

// ------------------------------------------------------------- uniform (NEXT-2)
__global__ void minmax_bits(const double *__restrict__ norm2, int64_t n,
                            unsigned long long *__restrict__ mm) {
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long b = (unsigned long long)__double_as_longlong(norm2[i]);
        lo = b < lo ? b : lo;
        hi = b > hi ? b : hi;
    }
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long l2 = __shfl_xor_sync(NR_FULL, lo, o);
        unsigned long long h2 = __shfl_xor_sync(NR_FULL, hi, o);
        lo = l2 < lo ? l2 : lo;
        hi = h2 > hi ? h2 : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&mm[0], lo);
        atomicMax(&mm[1], hi);
    }
}

// Sub-dataset j holds norms in the j-th of m equal-width intervals of
// [min ||x||, max ||x||] (Fig. 3(a)).  sqrt is monotone, so the
// interval ends are sqrt(min norm2), sqrt(max norm2).
__global__ void uniform_assign(const double *__restrict__ norm2, int64_t n, int m,
                               const unsigned long long *__restrict__ mm,
                               uint8_t *__restrict__ part) {
    const double lo = sqrt(__longlong_as_double((long long)mm[0]));
    const double hi = sqrt(__longlong_as_double((long long)mm[1]));
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double r = sqrt(norm2[i]);
        long long j = 0;
        if (hi > lo) {
            j = (long long)floor(__dmul_rn(__ddiv_rn(__dsub_rn(r, lo), __dsub_rn(hi, lo)), (double)m));
            if (j >= m) j = m - 1;
            if (j < 0) j = 0;
        }
        part[i] = (uint8_t)j;
    }
}

int partition_uniform(const double *norm2, int64_t n, int m, uint8_t *part, cudaStream_t s,
                      std::string *err) {
    DevBuf mm(s);
    if (mm.alloc(16)) {
        *err = "partition: cudaMalloc failed";
        return NRLSH_ENOMEM;
    }
    unsigned long long init[2] = {~0ull, 0ull};
    cudaMemcpyAsync(mm.p, init, 16, cudaMemcpyHostToDevice, s);
    minmax_bits<<<grid_for(n, 256, 1024), 256, 0, s>>>(norm2, n, mm.get<unsigned long long>());
    note_launch(2);
    uniform_assign<<<grid_for(n, 256, 4096), 256, 0, s>>>(norm2, n, m,
                                                         mm.get<unsigned long long>(), part);
    return 0;
}

// ------------------------------------------------------------ stable scatter
constexpr int kScatTile = 4096;   // items per tile (16 rounds of 256)

__global__ void __launch_bounds__(256) scat_hist(const double *__restrict__ norm2,
                                                 const uint8_t *__restrict__ part, int64_t n,
                                                 int m, uint32_t *__restrict__ tile_cnt,
                                                 unsigned long long *__restrict__ vmax) {
    __shared__ uint32_t c[kMaxParts];
    __shared__ unsigned long long v[kMaxParts];
    for (int j = threadIdx.x; j < m; j += blockDim.x) { c[j] = 0; v[j] = 0; }
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kScatTile;
    for (int t = threadIdx.x; t < kScatTile; t += blockDim.x) {
        const int64_t i = base + t;
        if (i < n) {
            const int j = part[i];
            atomicAdd(&c[j], 1u);
            atomicMax(&v[j], (unsigned long long)__double_as_longlong(norm2[i]));
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        tile_cnt[(int64_t)blockIdx.x * m + j] = c[j];
        if (c[j]) atomicMax(&vmax[j], v[j]);
    }
}

// CTA j: per-tile bases of sub-dataset j (exclusive over tiles, relative to the
// sub-dataset's start), its size tot[j] and V_j
__global__ void __launch_bounds__(1024) scat_colscan(uint32_t *__restrict__ tile_cnt, int ntiles, int m,
                                                     uint32_t *__restrict__ tot,
                                                     const unsigned long long *__restrict__ vmax,
                                                     double *__restrict__ V) {
    __shared__ uint32_t ws[32];
    const int j = blockIdx.x;
    uint32_t run = 0;
    for (int t0 = 0; t0 < ntiles; t0 += 4 * (int)blockDim.x) {
        uint32_t v[4], loc = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int t = t0 + threadIdx.x * 4 + e;
            v[e] = t < ntiles ? tile_cnt[(int64_t)t * m + j] : 0u;
            loc += v[e];
        }
        uint32_t all;
        uint32_t ex = run + block_excl_scan(loc, ws, &all);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int t = t0 + threadIdx.x * 4 + e;
            if (t < ntiles) tile_cnt[(int64_t)t * m + j] = ex;
            ex += v[e];
        }
        run += all;
    }
    if (threadIdx.x == 0) {
        tot[j] = run;
        V[j] = __longlong_as_double((long long)vmax[j]);
    }
}

__global__ void __launch_bounds__(256) scat_write(const uint8_t *__restrict__ part, int64_t n,
                                                  int m, const uint32_t *__restrict__ tile_base,
                                                  const uint32_t *__restrict__ tot,
                                                  int64_t *__restrict__ offsets,
                                                  int32_t *__restrict__ perm,
                                                  int32_t *__restrict__ pos_of_id,
                                                  uint8_t *__restrict__ part_of_pos) {
    __shared__ uint32_t run[kMaxParts];
    __shared__ uint32_t wc[8][kMaxParts];
    __shared__ uint32_t ws[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    {   // offsets: exclusive over the sub-dataset sizes (m <= 256 = blockDim)
        const uint32_t c = (int)threadIdx.x < m ? tot[threadIdx.x] : 0u;
        uint32_t all;
        const uint32_t off = block_excl_scan(c, ws, &all);
        if ((int)threadIdx.x < m) {
            run[threadIdx.x] = off + tile_base[(int64_t)blockIdx.x * m + threadIdx.x];
            if (blockIdx.x == 0) offsets[threadIdx.x] = off;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) offsets[m] = all;
    }
    const int64_t base = (int64_t)blockIdx.x * kScatTile;
    for (int round = 0; round < kScatTile / 256; ++round) {
        for (int e = threadIdx.x; e < 8 * kMaxParts; e += blockDim.x) (&wc[0][0])[e] = 0;
        __syncthreads();
        const int64_t i = base + round * 256 + threadIdx.x;
        const bool valid = i < n;
        const int j = valid ? part[i] : 0x7fffffff;
        const unsigned peers = __match_any_sync(NR_FULL, j);
        const int rank = __popc(peers & lanemask_lt());
        if (valid && rank == 0) wc[warp][j] = __popc(peers);
        __syncthreads();
        if (valid) {
            uint32_t off = run[j];
            for (int w = 0; w < warp; ++w) off += wc[w][j];
            const uint32_t pos = off + rank;
            perm[pos] = (int32_t)i;
            pos_of_id[i] = (int32_t)pos;
            part_of_pos[pos] = (uint8_t)j;
        }
        __syncthreads();
        for (int jj = threadIdx.x; jj < m; jj += blockDim.x) {
            uint32_t add = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) add += wc[w][jj];
            run[jj] += add;
        }
        __syncthreads();
    }
    (void)lane;
}

int partition_scatter(const double *norm2, const uint8_t *part, int64_t n, int m, int32_t *perm,
                      int32_t *pos_of_id, uint8_t *part_of_pos, int64_t *offsets_d, double *V_d,
                      cudaStream_t s, std::string *err) {
    const int ntiles = (int)((n + kScatTile - 1) / kScatTile);
    DevBuf tc(s), vm(s), tt(s);
    if (tc.alloc((size_t)ntiles * m * 4) || vm.alloc((size_t)m * 8) || tt.alloc((size_t)m * 4)) {
        *err = "partition: cudaMalloc failed";
        return NRLSH_ENOMEM;
    }
    cudaMemsetAsync(vm.p, 0, (size_t)m * 8, s);
    scat_hist<<<ntiles, 256, 0, s>>>(norm2, part, n, m, tc.get<uint32_t>(),
                                     vm.get<unsigned long long>());
    scat_colscan<<<m, 1024, 0, s>>>(tc.get<uint32_t>(), ntiles, m, tt.get<uint32_t>(),
                                    vm.get<unsigned long long>(), V_d);
    scat_write<<<ntiles, 256, 0, s>>>(part, n, m, tc.get<uint32_t>(), tt.get<uint32_t>(), offsets_d,
                                      perm, pos_of_id, part_of_pos);
    note_launch(3);
    return 0;
}

// =========================================================================== K3
// SIMT fp32 reference path for the projection (kept for d/L shapes the tensor
// core kernel does not cover).  CTA tile: 64 items x 32W columns, k-chunks of 32.
template <int W>
__global__ void __launch_bounds__(256) k3_codes_simt(
    const float *__restrict__ X, int64_t n, int d, const double *__restrict__ norm2,
    const uint8_t *__restrict__ part, const double *__restrict__ V,
    const float *__restrict__ Apad, int L, const int32_t *__restrict__ pos_of_id,
    uint32_t *__restrict__ codes) {
    constexpr int TB = 32 * W;         // columns
    constexpr int CPT = TB / 16;       // columns per thread
    __shared__ float Xs[32][65];
    __shared__ float As[32][TB];
    __shared__ uint32_t sw[64][W];
    __shared__ float st[64];
    const int tid = threadIdx.x;
    const int tb = tid & 15, ti = tid >> 4;
    for (int64_t i0 = (int64_t)blockIdx.x * 64; i0 < n; i0 += (int64_t)gridDim.x * 64) {
        float acc[4][CPT];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < CPT; ++c) acc[a][c] = 0.f;
        if (tid < 64) {
            const int64_t i = i0 + tid;
            float t = 0.f;
            if (i < n) {
                const double Vj = V[part[i]];
                if (Vj == 0.0) t = 1.f;
                else {
                    const double df = Vj - norm2[i];
                    t = (float)sqrt(df > 0.0 ? df : 0.0);
                }
            }
            st[tid] = t;
        }
        for (int k0 = 0; k0 < d; k0 += 32) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int idx = tid + 256 * e;
                const int r = idx >> 5, k = idx & 31;
                const int64_t i = i0 + r;
                Xs[k][r] = (i < n && k0 + k < d) ? __ldg(X + i * (int64_t)d + k0 + k) : 0.f;
            }
            for (int idx = tid; idx < 32 * TB; idx += 256) {
                const int k = idx / TB, b = idx % TB;
                As[k][b] = (k0 + k < d) ? Apad[(int64_t)(k0 + k) * TB + b] : 0.f;
            }
            __syncthreads();
#pragma unroll 8
            for (int kk = 0; kk < 32; ++kk) {
                float a[4], bb[CPT];
#pragma unroll
                for (int u = 0; u < 4; ++u) a[u] = Xs[kk][ti * 4 + u];
#pragma unroll
                for (int c = 0; c < CPT; ++c) bb[c] = As[kk][tb * CPT + c];
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int c = 0; c < CPT; ++c) acc[u][c] = fmaf(a[u], bb[c], acc[u][c]);
            }
            __syncthreads();
        }
        for (int e = tid; e < 64 * W; e += 256) (&sw[0][0])[e] = 0u;
        __syncthreads();
        const float *Ad = Apad + (int64_t)d * TB;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int r = ti * 4 + u;
            uint32_t mask = 0;
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                const int b = tb * CPT + c;
                const float y = fmaf(__ldg(Ad + b), st[r], acc[u][c]);
                if (b < L && y >= 0.f) mask |= 1u << (b & 31);
            }
            atomicOr(&sw[r][(tb * CPT) >> 5], mask);
        }
        __syncthreads();
        for (int e = tid; e < 64 * W; e += 256) {
            const int r = e / W, w = e % W;
            const int64_t i = i0 + r;
            if (i < n) codes[(int64_t)pos_of_id[i] * W + w] = sw[r][w];
        }
        __syncthreads();
    }
}

void launch_item_codes(const float *X, int64_t n, int d, const double *norm2,
                       const uint8_t *part, const double *V, const float *Apad, int L, int W,
                       const int32_t *pos_of_id, uint32_t *codes, void *Xb, int dpb,
                       float *xnorm, float *Xpad, int dpad, cudaStream_t s,
                       const int32_t *perm, int m) {
    if (codes_tc_supported(d, W)) {
        launch_item_codes_tc(X, n, d, norm2, part, V, Apad, L, W, pos_of_id, codes, Xb, dpb, Xpad,
                             dpad, s, nullptr, 0, nullptr, m);
        return;
    }
    // SIMT path: the row copies in separate passes
    if (Xb) launch_bf16_prep(X, n, d, dpb, Xb, nullptr, s, perm);
    if (Xpad) {
        cudaMemcpy2DAsync(Xpad, (size_t)dpad * 4, X, (size_t)d * 4, (size_t)d * 4, (size_t)n,
                          cudaMemcpyDeviceToDevice, s);
        cudaMemset2DAsync(Xpad + d, (size_t)dpad * 4, 0, (size_t)(dpad - d) * 4, (size_t)n, s);
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = grid_for(n, 64, sms * 8);
    switch (W) {
        case 1: k3_codes_simt<1><<<grid, 256, 0, s>>>(X, n, d, norm2, part, V, Apad, L, pos_of_id, codes); break;
        case 2: k3_codes_simt<2><<<grid, 256, 0, s>>>(X, n, d, norm2, part, V, Apad, L, pos_of_id, codes); break;
        case 3: k3_codes_simt<3><<<grid, 256, 0, s>>>(X, n, d, norm2, part, V, Apad, L, pos_of_id, codes); break;
        default: k3_codes_simt<4><<<grid, 256, 0, s>>>(X, n, d, norm2, part, V, Apad, L, pos_of_id, codes); break;
    }
    note_launch();
}

}  // namespace nrlsh
