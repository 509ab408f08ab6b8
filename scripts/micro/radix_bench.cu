// Tile-sort A/B (tuning aid): CTA merge sort (cta_sort.cuh) vs CTA LSD radix sort
// (cta_radix.cuh) on 2^25 keys / 2^24 pairs in independent tiles, HBM -> sort -> HBM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo radix_bench.cu
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_1002_4464_b200/csrc/gbs_kernels.cuh"
#include "cta_radix.cuh"
using namespace gbs;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK, 1) k_merge_keys(const uint32_t* in, uint32_t* out, int ntiles)
{
    using S = Seg<KIND_KEYS, BLOCK, ITEMS>;
    extern __shared__ __align__(16) unsigned char smem[];
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        uint32_t x[ITEMS];
        S::load_regs(x, in, nullptr, (uint64_t)t * S::TILE, S::TILE, smem);
        S::CS::sort(x, reinterpret_cast<uint32_t*>(smem), S::TILE);
        S::store(out, nullptr, (uint64_t)t * S::TILE, S::TILE, smem);
        __syncthreads();
    }
}

template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK, 1) k_merge_pairs(const uint32_t* in, const uint32_t* vin, uint32_t* out,
                                                          uint32_t* vout, int ntiles)
{
    using S = Seg<KIND_PAIRS, BLOCK, ITEMS>;
    extern __shared__ __align__(16) unsigned char smem[];
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        unsigned long long x[ITEMS];
        S::load_regs(x, in, vin, (uint64_t)t * S::TILE, S::TILE, smem);
        S::CS::sort(x, reinterpret_cast<unsigned long long*>(smem), S::TILE);
        S::store(out, vout, (uint64_t)t * S::TILE, S::TILE, smem);
        __syncthreads();
    }
}

template <int BLOCK, int ITEMS, bool PAIRS, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) k_radixT(const uint32_t* in, const uint32_t* vin, uint32_t* out,
                                                        uint32_t* vout, int ntiles, int valid)
{
    using R = CtaRadixT<BLOCK, ITEMS>;
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* kb = sm;
    uint32_t* vb = kb + R::KW;
    uint32_t* cnt = vb + (PAIRS ? R::KW : 0);
    uint32_t* ws = cnt + R::CW;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        uint32_t x[ITEMS], y[ITEMS];
        const uint64_t base = (uint64_t)t * R::TILE;
        for (int p = threadIdx.x; p < valid; p += BLOCK) {
            kb[R::phys(p)] = __ldg(in + base + p);
            if (PAIRS) vb[R::phys(p)] = __ldg(vin + base + p);
        }
        __syncthreads();
        const int p0 = threadIdx.x * ITEMS;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            x[k] = p0 + k < valid ? kb[R::phys(p0 + k)] : 0u;
            if (PAIRS) y[k] = p0 + k < valid ? vb[R::phys(p0 + k)] : 0u;
        }
        __syncthreads();
        R::template sort<PAIRS>(x, y, kb, vb, cnt, ws, valid);
        for (int p = threadIdx.x; p < valid; p += BLOCK) {
            out[base + p] = kb[R::phys(p)];
            if (PAIRS) vout[base + p] = vb[R::phys(p)];
        }
        __syncthreads();
    }
}

template <int BLOCK, int ITEMS, bool PAIRS, int MINB, bool MATCH>
__global__ void __launch_bounds__(BLOCK, MINB) k_radix(const uint32_t* in, const uint32_t* vin, uint32_t* out,
                                                       uint32_t* vout, int ntiles, int valid)
{
    using R = CtaRadix<BLOCK, ITEMS, MATCH>;
    extern __shared__ __align__(16) uint32_t sm[];
    uint32_t* kb = sm;
    uint32_t* vb = kb + R::TILE;
    uint32_t* h0 = vb + (PAIRS ? R::TILE : 0);
    uint32_t* h1 = h0 + R::HIST;
    uint32_t* ws = h1 + R::HIST;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        uint32_t x[ITEMS], y[ITEMS];
        const uint64_t base = (uint64_t)t * R::TILE;
        const int p0 = w * 32 * ITEMS + lane;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const int p = p0 + 32 * k;
            x[k] = p < valid ? __ldg(in + base + p) : 0xFFFFFFFFu;
            if (PAIRS) y[k] = p < valid ? __ldg(vin + base + p) : 0u;
        }
        R::template sort<PAIRS>(x, y, kb, vb, h0, h1, ws, valid);
        // 128-bit write-back
        const uint4* k4 = reinterpret_cast<const uint4*>(kb);
        uint4* o4 = reinterpret_cast<uint4*>(out + base);
        for (int q = threadIdx.x; q < valid / 4; q += BLOCK) o4[q] = k4[q];
        if (PAIRS) {
            const uint4* v4 = reinterpret_cast<const uint4*>(vb);
            uint4* ov = reinterpret_cast<uint4*>(vout + base);
            for (int q = threadIdx.x; q < valid / 4; q += BLOCK) ov[q] = v4[q];
        }
        __syncthreads();
    }
}

static uint64_t sm64(uint64_t& z) { z += 0x9E3779B97F4A7C15ull; uint64_t r = z; r = (r ^ (r >> 30)) * 0xBF58476D1CE4E5B9ull; r = (r ^ (r >> 27)) * 0x94D049BB133111EBull; return r ^ (r >> 31); }

template <typename F>
static float timeit(F f, int reps)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    f();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

static bool check_tiles(const std::vector<uint32_t>& in, const std::vector<uint32_t>& out, const std::vector<uint32_t>* vout,
                        int tile, int ntiles, int valid)
{
    for (int t = 0; t < ntiles; t += std::max(1, ntiles / 16)) {
        std::vector<std::pair<uint32_t, uint32_t>> e;
        for (int p = 0; p < valid; ++p) e.push_back({in[(size_t)t * tile + p], (uint32_t)((size_t)t * tile + p)});
        std::stable_sort(e.begin(), e.end(), [](auto& a, auto& b) { return a.first < b.first; });
        for (int p = 0; p < valid; ++p) {
            if (out[(size_t)t * tile + p] != e[p].first) { printf("  key mismatch tile %d pos %d\n", t, p); return false; }
            if (vout && (*vout)[(size_t)t * tile + p] != e[p].second) { printf("  val mismatch tile %d pos %d\n", t, p); return false; }
        }
    }
    return true;
}

int main()
{
    const size_t N = 1u << 25;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    std::vector<uint32_t> h(N), hv(N), hd(N);
    uint64_t z = 7;
    for (size_t i = 0; i < N; ++i) { h[i] = (uint32_t)(sm64(z) >> 32); hv[i] = (uint32_t)i; hd[i] = h[i] % 1000; }
    uint32_t *din, *dout, *dvin, *dvout;
    CK(cudaMalloc(&din, N * 4)); CK(cudaMalloc(&dout, N * 4)); CK(cudaMalloc(&dvin, N * 4)); CK(cudaMalloc(&dvout, N * 4));
    CK(cudaMemcpy(dvin, hv.data(), N * 4, cudaMemcpyHostToDevice));
    std::vector<uint32_t> ho(N), hvo(N);
    for (int dist = 0; dist < 3; ++dist) {
        const std::vector<uint32_t>& src = dist == 0 ? h : dist == 1 ? hd : std::vector<uint32_t>(N, 5u);
        CK(cudaMemcpy(din, src.data(), N * 4, cudaMemcpyHostToDevice));
        printf("== keys distribution %s\n", dist == 0 ? "uniform" : dist == 1 ? "mod1000" : "zero");
        {   // merge 1024x32
            constexpr int B = 1024, I = 32;
            using S = Seg<KIND_KEYS, B, I>;
            size_t smb = S::smem_bytes();
            CK(cudaFuncSetAttribute(k_merge_keys<B, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
            int nt = (int)(N / S::TILE);
            float ms = timeit([&] { k_merge_keys<B, I><<<nsm, B, smb>>>(din, dout, nt); }, 10);
            CK(cudaMemcpy(ho.data(), dout, N * 4, cudaMemcpyDeviceToHost));
            printf("merge  keys %4dx%2d: %.4f ms  %.1f Gkeys/s  ok=%d\n", B, I, ms, N / ms / 1e6, check_tiles(src, ho, nullptr, S::TILE, nt, S::TILE));
        }
        auto radix_keys = [&](auto bt, auto it, auto mb, int valid) {
            constexpr int B = decltype(bt)::value, I = decltype(it)::value, MB = decltype(mb)::value;
            for (int var = 0; var < 2; ++var) {
                auto kern = var == 0 ? k_radix<B, I, false, MB, false> : k_radixT<B, I, false, MB>;
                const int TILE = B * I;
                size_t smb = (var == 0 ? CtaRadix<B, I>::smem_words(false) : CtaRadixT<B, I>::smem_words(false)) * 4;
                if (smb > 227 * 1024) continue;
                CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
                int occ = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, B, smb);
                if (!occ) continue;
                int nt = (int)(N / TILE);
                float ms = timeit([&] { kern<<<nsm * occ, B, smb>>>(din, nullptr, dout, nullptr, nt, valid); }, 10);
                CK(cudaGetLastError());
                CK(cudaMemcpy(ho.data(), dout, N * 4, cudaMemcpyDeviceToHost));
                const double nk = (double)nt * valid;
                printf("%s keys %4dx%2d (occ %d, valid %d): %.4f ms  %.1f Gkeys/s  ok=%d\n", var ? "radixT " : "radixB8", B, I, occ, valid, ms, nk / ms / 1e6,
                       check_tiles(src, ho, nullptr, TILE, nt, valid));
            }
        };
        radix_keys(std::integral_constant<int, 1024>{}, std::integral_constant<int, 32>{}, std::integral_constant<int, 1>{}, 32768);
        radix_keys(std::integral_constant<int, 1024>{}, std::integral_constant<int, 32>{}, std::integral_constant<int, 1>{}, 16384);
        radix_keys(std::integral_constant<int, 512>{}, std::integral_constant<int, 32>{}, std::integral_constant<int, 2>{}, 16384);
        radix_keys(std::integral_constant<int, 512>{}, std::integral_constant<int, 32>{}, std::integral_constant<int, 2>{}, 12000);
        radix_keys(std::integral_constant<int, 256>{}, std::integral_constant<int, 32>{}, std::integral_constant<int, 4>{}, 8192);
    }
    // pairs (keys mod 1000: many ties -> stability is checked)
    for (int dist = 0; dist < 2; ++dist) {
        const std::vector<uint32_t>& src = dist == 0 ? h : hd;
        CK(cudaMemcpy(din, src.data(), N * 4, cudaMemcpyHostToDevice));
        printf("== pairs distribution %s\n", dist == 0 ? "uniform" : "mod1000");
        {
            constexpr int B = 1024, I = 16;
            using S = Seg<KIND_PAIRS, B, I>;
            size_t smb = S::smem_bytes();
            CK(cudaFuncSetAttribute(k_merge_pairs<B, I>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
            int nt = (int)(N / S::TILE);
            float ms = timeit([&] { k_merge_pairs<B, I><<<nsm, B, smb>>>(din, dvin, dout, dvout, nt); }, 10);
            CK(cudaMemcpy(ho.data(), dout, N * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(hvo.data(), dvout, N * 4, cudaMemcpyDeviceToHost));
            printf("merge  pairs %4dx%2d: %.4f ms  %.1f Gpairs/s  ok=%d\n", B, I, ms, N / ms / 1e6, check_tiles(src, ho, &hvo, S::TILE, nt, S::TILE));
        }
        auto radix_pairs = [&](auto bt, auto it, auto mb) {
            constexpr int B = decltype(bt)::value, I = decltype(it)::value, MB = decltype(mb)::value;
            for (int var = 0; var < 2; ++var) {
                auto kern = var == 0 ? k_radix<B, I, true, MB, false> : k_radixT<B, I, true, MB>;
                const int TILE = B * I;
                size_t smb = (var == 0 ? CtaRadix<B, I>::smem_words(true) : CtaRadixT<B, I>::smem_words(true)) * 4;
                if (smb > 227 * 1024) continue;
                CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
                int occ = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, B, smb);
                if (!occ) continue;
                int nt = (int)(N / TILE);
                float ms = timeit([&] { kern<<<nsm * occ, B, smb>>>(din, dvin, dout, dvout, nt, TILE); }, 10);
                CK(cudaGetLastError());
                CK(cudaMemcpy(ho.data(), dout, N * 4, cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(hvo.data(), dvout, N * 4, cudaMemcpyDeviceToHost));
                printf("%s pairs %4dx%2d (occ %d): %.4f ms  %.1f Gpairs/s  ok=%d\n", var ? "radixT " : "radixB8", B, I, occ, ms, N / ms / 1e6,
                       check_tiles(src, ho, &hvo, TILE, nt, TILE));
            }
        };
        radix_pairs(std::integral_constant<int, 1024>{}, std::integral_constant<int, 16>{}, std::integral_constant<int, 1>{});
        radix_pairs(std::integral_constant<int, 512>{}, std::integral_constant<int, 32>{}, std::integral_constant<int, 1>{});
        radix_pairs(std::integral_constant<int, 512>{}, std::integral_constant<int, 16>{}, std::integral_constant<int, 2>{});
    }
    return 0;
}
