// common.cuh — shared device/host helpers of libnrlsh (CUDA path only).
// Nothing here is shared with oracle/ (the CPU reference).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#define NR_FULL 0xffffffffu

namespace nrlsh {

// Programmatic dependent launch: a kernel launched with launch_pdl may start (its
// CTAs scheduled, prologue run) while the previous kernel on the stream drains;
// it must call pdl_wait() before touching anything that kernel wrote (the wait
// returns once the predecessor has completed and its writes are visible).
// NRLSH_NO_PDL=1 launches plainly (A/B experiments).
__device__ __forceinline__ void pdl_wait() {
#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ >= 900)
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}


constexpr int kMaxParts = 256;     // uint8 partition ids
constexpr int kMaxWords = 4;       // code_bits <= 128

// ---------------------------------------------------------------- errors
struct Error {
    int status;
    std::string msg;
};

// ---------------------------------------------------------------- device utils
__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Ascending-orderable uint32 image of an fp32 value (total order, -0 < +0).
__device__ __forceinline__ uint32_t float_order(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float float_unorder(uint32_t o) {
    uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(u);
}

// Block-wide exclusive scan of one uint32 per thread (blockDim.x <= 1024,
// multiple of 32).  `ws` must hold 32 words.  Returns the exclusive prefix;
// *total receives the block sum.
// The radius delta_j(q) is stored as int8 with -1 = "sub-dataset skipped"; a radius of
// 128 (L = 128, every cell of j within the bound) wraps to -128 and is read back here.
__device__ __forceinline__ int radius_of(int8_t v) { return v == (int8_t)-1 ? -1 : (int)(uint8_t)v; }

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *ws, uint32_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(NR_FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < nw ? ws[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(NR_FULL, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nw) ws[lane] = w;  // inclusive warp prefix
    }
    __syncthreads();
    uint32_t base = warp > 0 ? ws[warp - 1] : 0u;
    uint32_t tot = ws[nw - 1];
    __syncthreads();
    if (total) *total = tot;
    return base + x - v;
}

template <int W>
__device__ __forceinline__ int hamming(const uint32_t (&a)[W], const uint32_t (&b)[W]) {
    int h = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) h += __popc(a[w] ^ b[w]);
    return h;
}

inline int grid_for(int64_t work, int per_block, int max_blocks) {
    int64_t g = (work + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > max_blocks) g = max_blocks;
    return (int)g;
}

}  // namespace nrlsh
