// ubench_imma.cu — legacy mma.sync int8 (m16n8k32) throughput on sm_100a, and POPC for
// reference.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ubench_imma.cu -o tools/ubench_imma
#include <cstdio>
#include <cstdint>
__global__ void imma_loop(int iters, int *out) {
    uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    int c[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(c[u][0]), "+r"(c[u][1]), "+r"(c[u][2]), "+r"(c[u][3])
                         : "r"(a0 + u), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    int s = 0;
    for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void popc_loop(int iters, int *out) {
    uint32_t x = threadIdx.x * 0x9E3779B9u, acc = 0;
    uint32_t v[8];
    for (int u = 0; u < 8; ++u) v[u] = x ^ (u * 0x85EBCA6Bu);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) { acc += __popc(v[u] ^ it); }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int *out; cudaMalloc(&out, sms * 8 * 1024 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int warps : {4, 8, 16, 32}) {
        const int iters = 4000;
        imma_loop<<<sms, warps * 32>>>(iters, out);
        cudaEventRecord(e0);
        imma_loop<<<sms, warps * 32>>>(iters, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double macs = (double)sms * warps * iters * 8 * 16 * 8 * 32;
        printf("IMMA m16n8k32 s8: %2d warps/SM: %.1f TOPS (int8 MAC x2), %.0f MAC/clk/SM @1.965GHz\n", warps,
               2 * macs / (ms * 1e-3) / 1e12, macs / (ms * 1e-3) / 1.965e9 / sms);
        popc_loop<<<sms, warps * 32>>>(iters * 4, out);
        cudaEventRecord(e0);
        popc_loop<<<sms, warps * 32>>>(iters * 4, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double pops = (double)sms * warps * 32 * iters * 4 * 8;
        printf("POPC: %2d warps/SM: %.2f TPOPC/s, %.1f/clk/SM\n", warps, pops / (ms * 1e-3) / 1e12,
               pops / (ms * 1e-3) / 1.965e9 / sms);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
