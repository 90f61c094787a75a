// gt_kernels.cu — exact brute-force MIPS ground truth (Eq. (1)).
//
// Certified filter: a pilot over a strided item sample gives, per query, a
// lower bound LB_q on the true k-th best inner product (the k-th largest of
// fl(q.x) - e(q,x) over real items, e = a rigorous bound on the fp error).  The
// filter GEMM then keeps every item with fl(q.x) + e(q,x) >= LB_q — a superset of
// the exact top-k — and the survivors are re-scored exactly (fp32) and top-k'd.
#include <algorithm>

#include "common.cuh"
#include "internal.h"

namespace nrlsh {

// |x| in fp32 from a sequential fp64 sum of squares (one warp per row).
__global__ void vec_norms(const float *__restrict__ X, int64_t n, int d,
                          float *__restrict__ xnorm) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n;
         i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        double s = 0.0;
        for (int k = lane; k < d; k += 32) {
            const double v = (double)__ldg(X + i * (int64_t)d + k);
            s += v * v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(NR_FULL, s, o);
        if (lane == 0) xnorm[i] = __double2float_ru(sqrt(s));
    }
}

void launch_vec_norms(const float *X, int64_t n, int d, float *xnorm, cudaStream_t s) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    vec_norms<<<grid_for(n * 32, 256, sms * 16), 256, 0, s>>>(X, n, d, xnorm);
    note_launch();
}

// SIMT fp32 filter GEMM.  CTA tile 64 queries x 128 items, k-chunks of 32;
// thread (tq, ti) owns queries tq + 16v (v < 4) and items ti + 16u (u < 8).
__global__ void __launch_bounds__(256) gt_filter_simt(
    const float *__restrict__ X, int64_t n, int d, const float *__restrict__ Q, int Qb,
    const float *__restrict__ xnorm, const float *__restrict__ qnorm,
    const float *__restrict__ lb, float eps_rel, int32_t *__restrict__ cand,
    uint32_t *__restrict__ cnt, int64_t C) {
    __shared__ float Qs[64][33];
    __shared__ float Xs[128][33];
    const int tid = threadIdx.x;
    const int ti = tid & 15, tq = tid >> 4;
    const int q0 = blockIdx.y * 64;
    for (int64_t i0 = (int64_t)blockIdx.x * 128; i0 < n; i0 += (int64_t)gridDim.x * 128) {
        float acc[4][8];
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[v][u] = 0.f;
        for (int k0 = 0; k0 < d; k0 += 32) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {   // Q chunk: 64 x 32
                const int idx = tid + 256 * e;
                const int r = idx >> 5, k = idx & 31;
                if (e < 8 && r < 64) {
                    const int q = q0 + r;
                    Qs[r][k] = (q < Qb && k0 + k < d) ? Q[(int64_t)q * d + k0 + k] : 0.f;
                }
            }
#pragma unroll
            for (int e = 0; e < 16; ++e) {  // X chunk: 128 x 32
                const int idx = tid + 256 * e;
                const int r = idx >> 5, k = idx & 31;
                const int64_t i = i0 + r;
                Xs[r][k] = (i < n && k0 + k < d) ? __ldg(X + i * (int64_t)d + k0 + k) : 0.f;
            }
            __syncthreads();
#pragma unroll 4
            for (int kk = 0; kk < 32; ++kk) {
                float a[4], b[8];
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = Qs[tq + 16 * v][kk];
#pragma unroll
                for (int u = 0; u < 8; ++u) b[u] = Xs[ti + 16 * u][kk];
#pragma unroll
                for (int v = 0; v < 4; ++v)
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc[v][u] = fmaf(a[v], b[u], acc[v][u]);
            }
            __syncthreads();
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int q = q0 + tq + 16 * v;
            if (q >= Qb) continue;
            const float L0 = lb[q], qn = qnorm[q] * eps_rel;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int64_t i = i0 + ti + 16 * u;
                if (i >= n) continue;
                const float up = __fadd_ru(acc[v][u], __fmul_ru(qn, xnorm[i]));
                if (up >= L0) {
                    const uint32_t slot = atomicAdd(&cnt[q], 1u);
                    if (slot < C) cand[(int64_t)q * C + slot] = (int32_t)i;
                }
            }
        }
    }
}

void launch_gt_filter(const float *X, int64_t n, int d, const float *Q, int Qb,
                      const float *xnorm, const float *qnorm, const float *lb, float eps_rel,
                      int32_t *cand, uint32_t *cnt, int64_t C, cudaStream_t s) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int gy = (Qb + 63) / 64;
    const int gx = std::max(1, std::min<int>((int)((n + 127) / 128), (sms * 8 + gy - 1) / gy * 4));
    gt_filter_simt<<<dim3(gx, gy), 256, 0, s>>>(X, n, d, Q, Qb, xnorm, qnorm, lb, eps_rel, cand,
                                                 cnt, C);
    note_launch();
}


// Certified warm start of the filter threshold from caller-supplied item ids
// (any ids: typically the LSH answers).  Every seed's exact-product score is
// recomputed here: lb = fl(q.x) - eps |q| |x| (rounded down) is a lower bound of
// its true score, so the k-th largest lb over k distinct seeds is a lower bound of
// the true k-th best score (theta_glob[q]; 0 = no bound).  The result of the
// ground truth does not depend on the seeds, only its speed does.
__global__ void __launch_bounds__(256) gt_seed_theta(const float *__restrict__ X, int64_t n, int d,
                                                     const float *__restrict__ Q,
                                                     const float *__restrict__ qnorm,
                                                     const int64_t *__restrict__ seeds, int ks,
                                                     int k, float eps_rel,
                                                     uint32_t *__restrict__ theta_glob,
                                                     uint32_t *__restrict__ zero_cnt) {
    pdl_wait();
    __shared__ float lbs[1024];
    __shared__ int64_t sid[1024];
    const int q = blockIdx.x;
    const float *qp = Q + (int64_t)q * d;
    const int np2 = ks <= 1 ? 1 : 1 << (32 - __clz(ks - 1));
    // a warp per seed, lanes over the dimensions (32 partial FMA chains and a 5-level
    // tree: an error bound below the sequential chain's, which eps_rel covers)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int t = warp; t < np2; t += nw) {
        int64_t id = t < ks ? seeds[(int64_t)q * ks + t] : -1;
        if (id >= n) id = -1;
        // duplicates count once: keep the first occurrence only
        bool dup = false;
        for (int u = lane; u < t && id >= 0; u += 32) dup |= seeds[(int64_t)q * ks + u] == id;
        if (__any_sync(0xffffffffu, dup)) id = -1;
        float lb = -INFINITY;
        if (id >= 0) {   // (warp-uniform)
            const float *xp = X + id * d;
            float acc = 0.f;
            double xx = 0.0;
            for (int j = lane; j < d; j += 32) {
                const float xv = __ldg(xp + j);
                acc = fmaf(__ldg(qp + j), xv, acc);
                xx += (double)xv * (double)xv;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                acc += __shfl_xor_sync(0xffffffffu, acc, o);
                xx += __shfl_xor_sync(0xffffffffu, xx, o);
            }
            const float xn = __double2float_ru(sqrt(xx) * (1.0 + 0x1p-50));
            lb = __fsub_rd(acc, __fmul_ru(__fmul_ru(eps_rel, qnorm[q]), xn));
        }
        if (lane == 0) {
            lbs[t] = lb;
            sid[t] = id;
        }
    }
    __syncthreads();
    // sort descending
    for (int size = 2; size <= np2; size <<= 1) {
        for (int st = size >> 1; st > 0; st >>= 1) {
            for (int t = threadIdx.x; t < np2; t += blockDim.x) {
                const int o = t ^ st;
                if (o > t) {
                    const bool up = (t & size) == 0;
                    if ((lbs[t] < lbs[o]) == up) { const float x = lbs[t]; lbs[t] = lbs[o]; lbs[o] = x; }
                }
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) {
        const float th = (k <= np2) ? lbs[k - 1] : -INFINITY;
        theta_glob[q] = (th > -INFINITY) ? float_order(th) : 0u;
        if (zero_cnt) zero_cnt[q] = 0u;   // (the survivor count, instead of a memset node)
    }
}

void launch_gt_seed_theta(const float *X, int64_t n, int d, const float *Q, int Qb,
                          const float *qnorm, const int64_t *seeds, int ks, int k, float eps_rel,
                          uint32_t *theta_glob, cudaStream_t s, uint32_t *zero_cnt) {
    launch_pdl(gt_seed_theta, dim3(Qb), dim3(256), 0, s, X, n, d, Q, qnorm, seeds, ks, k, eps_rel, theta_glob,
               zero_cnt);
    note_launch();
}

}  // namespace nrlsh
