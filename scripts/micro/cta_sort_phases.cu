// Per-phase cycle counts of the CTA merge sort (tuning aid): network + each merge level.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_1002_4464_b200/csrc/cta_sort.cuh"
using namespace gbs;
#ifndef BLK
#define BLK 1024
#define ITM 32
#endif
constexpr int BLOCK = BLK, ITEMS = ITM;
using CS = CtaSort<uint32_t, BLOCK, ITEMS, 1>;
__global__ void __launch_bounds__(BLOCK, 1) k(uint32_t* data, long long* phases, int v) {
    extern __shared__ uint32_t sm[];
    uint32_t* src = data + (size_t)blockIdx.x * CS::TILE;
    uint32_t x[ITEMS];
    const int p0 = CS::load_pos(0), rem = v - p0;
    #pragma unroll
    for (int q = 0; q < ITEMS; ++q) x[q] = 32 * q < rem ? src[p0 + 32 * q] : 0xFFFFFFFFu;
    __syncthreads();
    long long t0 = clock64();
    const int t = threadIdx.x, wspan0 = (t >> 5) * CS::WARP_SPAN;
    if (wspan0 < v) reg_sort<uint32_t, ITEMS>(x);
    __syncthreads();
    long long t1 = clock64();
    if (t == 0) phases[blockIdx.x * 20 + 0] = t1 - t0;
    const int start = t * ITEMS;
    int lvl = 1;
    for (int w = ITEMS; w < CS::TILE; w *= 2, ++lvl) {
        long long a = clock64();
        #pragma unroll
        for (int q = 0; q < ITEMS; ++q) sm[CS::phys(start + q)] = x[q];
        __syncthreads();
        const bool active = start < v;
        if (active) CS::merge_thread(x, sm, start, w);
        __syncthreads();
        long long b = clock64();
        if (t == 0) phases[blockIdx.x * 20 + lvl] = b - a;
    }
    #pragma unroll
    for (int q = 0; q < ITEMS; ++q) sm[CS::phys(start + q)] = x[q];
    __syncthreads();
    for (int q = t; q < v; q += BLOCK) src[q] = sm[CS::phys(q)];
}
int main() {
    const int ctas = 148 * 4, v = CS::TILE;
    std::vector<uint32_t> h((size_t)ctas * CS::TILE);
    uint64_t z = 1; for (auto& e : h) { z = z * 6364136223846793005ull + 1442695040888963407ull; e = (uint32_t)(z >> 32); }
    uint32_t* d; long long* ph; cudaMalloc(&d, h.size() * 4); cudaMalloc(&ph, ctas * 20 * 8); cudaMemset(ph, 0, ctas * 20 * 8);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    size_t smb = CS::SMEM_ELEMS * 4;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    k<<<ctas, BLOCK, smb>>>(d, ph, v);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaEventRecord(a); k<<<ctas, BLOCK, smb>>>(d, ph, v); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    std::vector<long long> hp(ctas * 20); cudaMemcpy(hp.data(), ph, hp.size() * 8, cudaMemcpyDeviceToHost);
    std::vector<uint32_t> o(CS::TILE); cudaMemcpy(o.data(), d, CS::TILE * 4, cudaMemcpyDeviceToHost);
    bool ok = true; for (int i = 1; i < CS::TILE; ++i) ok &= o[i - 1] <= o[i];
    printf("BLOCK %d ITEMS %d: %d CTAs x %d keys: %.3f ms = %.2f Gkeys/s, sorted=%d\n", BLOCK, ITEMS, ctas, CS::TILE, ms, (double)ctas * CS::TILE / ms / 1e6, ok);
    long long tot = 0;
    for (int l = 0; l < 20; ++l) { long long s = 0; for (int c = 0; c < ctas; ++c) s += hp[c * 20 + l]; if (s) { printf("  phase %2d: %8lld cycles\n", l, s / ctas); tot += s / ctas; } }
    printf("  total %lld cycles per CTA\n", tot);
    return 0;
}
