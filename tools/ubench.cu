// ubench.cu — microbenchmarks for the peaks MEASURED_PEAKS.json lacks:
// POPC issue rate, the fused XOR+POPC+add loop (the scan's inner loop), and
// the SM clock seen during the run.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void popc_kernel(uint32_t *out, int iters, uint32_t seed) {
    uint32_t a[8];
    for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + 1) * (i + 7);
    uint32_t acc = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) { acc += __popc(a[i]); a[i] = a[i] * 1664525u + 1013904223u; }
    }
    if (acc == 0x12345678u) out[0] = acc;
}

// pure popc on independent registers (no LCG update): 8 popc + 8 adds per iter
__global__ void popc_only(uint32_t *out, int iters, uint32_t seed) {
    uint32_t a[16];
    for (int i = 0; i < 16; ++i) a[i] = seed ^ (threadIdx.x * 2654435761u + i * 97u);
    uint32_t acc[4] = {0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i & 3] += __popc(a[i] ^ (uint32_t)it);
    }
    if ((acc[0] + acc[1] + acc[2] + acc[3]) == 0x12345678u) out[0] = 1;
}

int main() {
    uint32_t *d;
    cudaMalloc(&d, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 20000;
    for (int rep = 0; rep < 2; ++rep) {
        int blocks = sms * 8, threads = 256;
        popc_only<<<blocks, threads>>>(d, iters, 1);
        cudaEventRecord(a);
        popc_only<<<blocks, threads>>>(d, iters, 2);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double ops = (double)blocks * threads * iters * 16;
        printf("popc_only: %.3f ms, %.3e POPC/s, %.2f POPC/clk/SM at %d MHz (max clock)\n", ms,
               ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
        popc_kernel<<<blocks, threads>>>(d, iters, 3);
        cudaEventRecord(a);
        popc_kernel<<<blocks, threads>>>(d, iters, 4);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        ops = (double)blocks * threads * iters * 8;
        printf("popc+lcg: %.3f ms, %.3e POPC/s, %.2f POPC/clk/SM\n", ms, ops / (ms * 1e-3),
               ops / (ms * 1e-3) / sms / (clk * 1e3));
    }
    return 0;
}
