// ubench_mma.cu — tcgen05.mma issue-rate microbenchmark (sm_100a).
// One CTA per SM; one thread issues `iters` x 4 MMAs (kind::f16 bf16 or kind::tf32,
// M=128, N in {64,128,256}, K=16/8 per instruction) on fixed smem operands,
// optionally committing to an mbarrier and waiting every `sync_every` groups.
// Prints MAC/clk/SM.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I paper_1809_08782_b200/csrc tools/ubench_mma.cu -o tools/ubench_mma -lcuda
#include <cstdio>
#include <cstdlib>

#include "tc_sm100.cuh"

using namespace nrlsh;

__global__ void __launch_bounds__(128, 1) mma_loop(int N, int kind, int iters, int sync_every, int warpwide,
                                                   unsigned long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
    uint8_t *A = smem, *B = smem + 16384;
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0;
    tc::fence_async_shared();
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar, 1);
        tc::fence_mbar_init();
    }
    if (warp == 0) tc::tmem_alloc(&slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tbase = slot;
    if (warpwide && warp == 1) {
        const uint32_t idesc = tc::umma_idesc(kind == 0 ? 1 : 2, 128, N);
        const uint32_t idesc_i8 = tc::umma_idesc_i8(128, N);
        const uint32_t a = tc::smem_u32(A), b = tc::smem_u32(B);
        uint32_t ph = 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (kind == 2)
                    tc::mma_i8_warp(tbase + (it & 1) * 256, tc::umma_desc_sw128(a + kk * 32),
                                    tc::umma_desc_sw128(b + kk * 32), idesc_i8, 1);
                else if (kind == 0)
                    tc::mma_f16_warp(tbase + (it & 1) * 256, tc::umma_desc_sw128(a + kk * 32),
                                     tc::umma_desc_sw128(b + kk * 32), idesc, 1);
                else
                    tc::mma_tf32_warp(tbase + (it & 1) * 256, tc::umma_desc_sw128(a + kk * 32),
                                      tc::umma_desc_sw128(b + kk * 32), idesc, 1);
            }
            if (sync_every > 0 && (it + 1) % sync_every == 0) {
                tc::mma_commit_warp(&bar);
                tc::mbar_wait(&bar, ph);
                ph ^= 1;
            }
        }
        tc::mma_commit_warp(&bar);
        tc::mbar_wait(&bar, ph);
        const long long t1 = clock64();
        if (threadIdx.x == 32) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
    } else if (!warpwide && threadIdx.x == 32) {
        const uint32_t idesc = tc::umma_idesc(kind == 0 ? 1 : 2, 128, N);
        const uint32_t a = tc::smem_u32(A), b = tc::smem_u32(B);
        uint32_t ph = 0;
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            for (int kk = 0; kk < 4; ++kk) {
                if (kind == 0)
                    tc::mma_f16(tbase + (it & 1) * 256, tc::umma_desc_sw128(a + kk * 32),
                                tc::umma_desc_sw128(b + kk * 32), idesc, 1);
                else
                    tc::mma_tf32(tbase + (it & 1) * 256, tc::umma_desc_sw128(a + kk * 32),
                                 tc::umma_desc_sw128(b + kk * 32), idesc, 1);
            }
            if (sync_every > 0 && (it + 1) % sync_every == 0) {
                tc::mma_commit(&bar);
                tc::mbar_wait(&bar, ph);
                ph ^= 1;
            }
        }
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, ph);
        const long long t1 = clock64();
        cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
    }
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tbase, 512);
}


// TMEM read throughput: `nw` warps (warp w reads lane quadrant w % 4) each issue
// `iters` x (2 x tcgen05.ld.32x32b.x32 + wait)
__global__ void __launch_bounds__(512, 1) tmem_ld_loop(int nw, int iters, unsigned long long *cycles,
                                                       float *sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc::tmem_alloc(&slot, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tbase = slot;
    float acc = 0.f;
    long long t0 = clock64();
    if (warp < nw) {
        const uint32_t ta = tbase + ((uint32_t)((warp & 3) * 32) << 16);
        for (int it = 0; it < iters; ++it) {
            uint32_t r0[32], r1[32];
            tc::tmem_ld_32x32b_x32(ta + ((it * 64) & 511), r0);
            tc::tmem_ld_32x32b_x32(ta + ((it * 64 + 32) & 511), r1);
            tc::tmem_ld_wait();
            acc += __uint_as_float(r0[5]) + __uint_as_float(r1[17]);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
    if (acc == 1.2345f) sink[threadIdx.x] = acc;
    if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

int main(int argc, char **argv) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *cyc;
    cudaMalloc(&cyc, sms * 8);
    const int smem = 16384 + 32768 + 1024;
    cudaFuncSetAttribute(mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 20000;
    for (int ww = 1; ww < 2; ++ww)
    for (int kind = 0; kind < 3; ++kind)
        for (int N : {64, 128, 256})
            for (int se : {0, 1, 4}) {
                mma_loop<<<sms, 128, smem>>>(N, kind, iters, se, ww, cyc);
                cudaDeviceSynchronize();
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                mma_loop<<<sms, 128, smem>>>(N, kind, iters, se, ww, cyc);
                cudaEventRecord(e1);
                cudaError_t err = cudaDeviceSynchronize();
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                unsigned long long h[1];
                cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
                const double k_per = kind == 0 ? 16 : (kind == 2 ? 32 : 8);
                const double macs = 128.0 * N * k_per * 4 * iters;
                printf("%s %s N=%3d sync_every=%d: %.1f cyc/MMA, %.0f MAC/clk/SM, %.1f TFLOP/s chip (%s)\n",
                       ww ? "warp  " : "thread", kind == 0 ? "bf16" : (kind == 2 ? "i8  " : "tf32"), N, se, (double)h[0] / (4.0 * iters),
                       macs / (double)h[0], 2.0 * macs * sms / (ms * 1e-3) / 1e12,
                       cudaGetErrorString(err));
            }
    float *sink;
    cudaMalloc(&sink, 4096);
    for (int nw : {4, 8, 16}) {
        const int it = 20000;
        tmem_ld_loop<<<sms, 512>>>(nw, it, cyc, sink);
        cudaError_t err = cudaDeviceSynchronize();
        unsigned long long h[1];
        cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        const double bytes = (double)nw * it * 2 * 32 * 32 * 4;
        printf("tmem ld: %2d warps: %.1f B/clk/SM (%s)\n", nw, bytes / (double)h[0], cudaGetErrorString(err));
    }
    return 0;
}
