// Microbenchmark: throughput of __match_any_sync, POPC, ATOMS on sm_100a (tuning aid).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_match(uint32_t* out, int iters, uint32_t seed) {
    uint32_t x = seed ^ (threadIdx.x * 2654435761u), acc = 0;
    for (int i = 0; i < iters; ++i) {
        #pragma unroll
        for (int u = 0; u < 8; ++u) {
            x = x * 1664525u + 1013904223u;
            uint32_t d = (x >> 24);
            uint32_t m = __match_any_sync(0xffffffffu, d);
            acc += m;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_alu(uint32_t* out, int iters, uint32_t seed) {
    uint32_t x = seed ^ (threadIdx.x * 2654435761u), acc = 0;
    for (int i = 0; i < iters; ++i) {
        #pragma unroll
        for (int u = 0; u < 8; ++u) {
            x = x * 1664525u + 1013904223u;
            uint32_t d = (x >> 24);
            acc += d;
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_atoms(uint32_t* out, int iters, uint32_t seed) {
    __shared__ uint32_t h[32][256];
    for (int i = threadIdx.x; i < 32 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    uint32_t x = seed ^ (threadIdx.x * 2654435761u), acc = 0;
    const int w = threadIdx.x >> 5;
    for (int i = 0; i < iters; ++i) {
        #pragma unroll
        for (int u = 0; u < 8; ++u) {
            x = x * 1664525u + 1013904223u;
            uint32_t d = (x >> 24);
            acc += atomicAdd(&h[w][d], 1u);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
    uint32_t* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
      for (int kind = 0; kind < 3; ++kind) {
        cudaEventRecord(a);
        if (kind == 0) k_match<<<148 * 2, 1024>>>(o, iters, 1);
        if (kind == 1) k_alu<<<148 * 2, 1024>>>(o, iters, 1);
        if (kind == 2) k_atoms<<<148 * 2, 1024>>>(o, iters, 1);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = 148.0 * 2 * 1024 * iters * 8;
        int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        printf("%s: %.3f ms, %.1f G ops/s, %.2f lane-ops/clk/SM (@%d MHz)\n", kind == 0 ? "match_any" : kind == 1 ? "alu-baseline" : "atoms(smem,256 bins/warp)",
               ms, ops / ms / 1e6, ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
      }
    }
    return 0;
}
