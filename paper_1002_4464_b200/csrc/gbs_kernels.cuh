// gbs_kernels.cuh -- the sm_100a kernels of GPU Bucket Sort (Dehne & Zaboli,
// arXiv 1002.4464, Algorithm 1), one per step of the paper.
//
// A "level" applies Alg. 1 to a batch of B independent problems of static capacity N
// (items [off_b, off_b + len_b), len_b <= N).  The top level is B = 1; Step 4 of a
// level is a level on the B sample arrays (u64 composites); a nested Step 9 is a level
// on the B*s buckets.  Positions len_b..m*L-1 of a problem are virtual sentinels
// (R8): they are never loaded or stored, but they take part in sampling.
//
// Item kinds:  KEYS  u32 keys (tag = post-local-sort position, never stored; R3)
//              PAIRS u32 keys + u32 values; on chip an item is (key << 32 | position)
//                    so the local sort is stable, values are gathered by position
//              U64   u64 composites (samples of a lower level), all distinct
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <type_traits>

#include "cta_sort.cuh"

namespace gbs {

typedef unsigned long long u64;
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

enum Kind { KIND_KEYS = 0, KIND_PAIRS = 1, KIND_U64 = 2 };

struct Probs {
    const u64* off;        // device array or nullptr -> b * stride
    const uint32_t* len;   // device array or nullptr -> len_c
    uint64_t stride;
    uint32_t len_c;
    uint32_t presorted;    // inputs are sorted runs of this length (host-side; copied to LevelDev)
    __device__ __forceinline__ uint64_t offset(uint32_t b) const { return off ? off[b] : (uint64_t)b * stride; }
    __device__ __forceinline__ uint32_t length(uint32_t b) const { return len ? len[b] : len_c; }
};

struct LevelDev {
    Probs pr;
    uint32_t B, L, s, d, m;
    uint32_t N;          // static problem capacity
    uint32_t pad_base;   // KIND_U64: tag base of the virtual sentinels (R8)
    void* in;            // Step 2 in place; Step 8 source; leaf source
    void* reloc;         // Step 8 destination = Step 9 source
    void* out;           // Step 9 / leaf destination
    uint32_t* in_v;
    uint32_t* reloc_v;
    uint32_t* out_v;
    u64* samples;          // [B][m][s]
    u64* splitters;        // [B][s]
    uint32_t* a;           // [B][m][s]   bucket sizes a_ij (real items)
    uint32_t* l;           // [B][m][s]   offsets l_ij (problem-relative)
    unsigned long long* state;  // [B][ceil(s/32)] decoupled look-back words
    u64* child_off;        // [B*s] nested Step 9 problems
    uint32_t* child_len;
    uint32_t pf_stride;    // co-resident CTAs (SMs x CTAs/SM): CTA b prefetches CTA b + pf_stride
    uint32_t presorted;    // input consists of sorted runs of this length (Step 4 levels), 0 = none
};

// L2 prefetch of a byte range (cp.async.bulk.prefetch: a TMA bulk operation, no
// registers or shared memory): the CTA of the next wave finds its tile in L2.
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes)
{
    if (bytes == 0) return;
    const uintptr_t a = (uintptr_t)p & ~uintptr_t(15);
    const uintptr_t e = ((uintptr_t)p + bytes + 15) & ~uintptr_t(15);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a)) : "memory");
}

// Copy `bytes` (multiple of 4) from global to shared memory with all threads of the
// CTA: 16-byte vector loads, 8 in flight per thread, when both sides are 16-byte
// aligned (warp-uniform check); 4-byte loads otherwise.  Caller synchronises.
template <int BLOCK>
__device__ __forceinline__ void stage_to_smem(void* dst, const void* src, size_t bytes)
{
    const bool vec = (((uintptr_t)src | (uintptr_t)dst) & 15) == 0;
    if (vec) {
        const size_t n16 = bytes / 16;
        const uint4* s = reinterpret_cast<const uint4*>(src);
        uint4* d = reinterpret_cast<uint4*>(dst);
        for (size_t q0 = threadIdx.x; q0 < n16; q0 += 8 * BLOCK) {
            uint4 r[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (q0 + u * BLOCK < n16) r[u] = __ldg(s + q0 + u * BLOCK);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (q0 + u * BLOCK < n16) d[q0 + u * BLOCK] = r[u];
        }
        for (size_t q = n16 * 4 + threadIdx.x; q < bytes / 4; q += BLOCK)
            reinterpret_cast<uint32_t*>(dst)[q] = __ldg(reinterpret_cast<const uint32_t*>(src) + q);
    } else {
        const size_t n4 = bytes / 4;
        const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
        uint32_t* d = reinterpret_cast<uint32_t*>(dst);
        for (size_t q0 = threadIdx.x; q0 < n4; q0 += 8 * BLOCK) {
            uint32_t r[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (q0 + u * BLOCK < n4) r[u] = __ldg(s + q0 + u * BLOCK);
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (q0 + u * BLOCK < n4) d[q0 + u * BLOCK] = r[u];
        }
    }
}

// Tile (sublist) of CTA `cta` of a per-sublist kernel: problem offset + i*L, length.
__device__ __forceinline__ void sublist_of(const LevelDev& lv, uint32_t cta, uint64_t& start, int& v)
{
    const uint32_t b = cta / lv.m, i = cta % lv.m;
    const uint32_t len = lv.pr.length(b);
    const uint64_t i0 = (uint64_t)i * lv.L;
    start = lv.pr.offset(b) + i0;
    v = len > i0 ? (int)(len - i0 < lv.L ? len - i0 : lv.L) : 0;
}

#ifndef GBS_KEYS_CHAINS
#define GBS_KEYS_CHAINS 1   // merge chains per thread (0 = automatic); 1 measured best at 1024x32
#endif
#ifndef GBS_WIDE_CHAINS
#define GBS_WIDE_CHAINS 1
#endif
#ifndef GBS_PRESORTED
#define GBS_PRESORTED 1     // Step 4 local sort merges the presorted sample runs only
#endif
#ifndef GBS_ADAPT_DEPTH
#define GBS_ADAPT_DEPTH 2   // Step 9 tile halvings for small buckets
#endif

template <int KIND> struct ItemT { using T = unsigned long long; };
template <> struct ItemT<KIND_KEYS> { using T = uint32_t; };

// Virtual sentinel of a U64 problem at position p >= N: key 0xFFFFFFFF with a tag
// above every tag of the level below, increasing in p (R8).
__device__ __forceinline__ unsigned long long pad64(uint32_t pad_base, uint64_t p_minus_N)
{
    return (0xFFFFFFFFull << 32) | (unsigned long long)(pad_base + (uint32_t)p_minus_N);
}

// ------------------------------------------------------------------ segment I/O
// Sort `v` items starting at element offset `src_off` of lv.in-like buffer `src`
// and leave the sorted tile in shared memory (pairs: values staged in vsm).
template <int KIND, int BLOCK, int ITEMS>
struct Seg {
    using T = typename ItemT<KIND>::T;
    using CS = CtaSort<T, BLOCK, ITEMS, (KIND == KIND_KEYS ? GBS_KEYS_CHAINS : GBS_WIDE_CHAINS)>;
    using KeyT = typename std::conditional<KIND == KIND_U64, unsigned long long, uint32_t>::type;  // in HBM
    static constexpr int TILE = CS::TILE;
    static constexpr size_t smem_bytes()
    {
        return sizeof(T) * CS::SMEM_ELEMS + (KIND == KIND_PAIRS ? sizeof(uint32_t) * TILE : 0);
    }

    static __device__ __forceinline__ void load_sort(const void* src, const uint32_t* src_v, uint64_t src_off,
                                                     int v, T* sm, uint32_t* vsm)
    {
        T x[ITEMS];
        if constexpr (KIND == KIND_KEYS) {
            const int p0 = CS::load_pos(0), rem = v - p0;    // load_pos(k) = p0 + 32k
            const uint32_t* s = reinterpret_cast<const uint32_t*>(src) + src_off + p0;
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) x[k] = 32 * k < rem ? (T)__ldg(s + 32 * k) : (T)0xFFFFFFFFu;
        } else if constexpr (KIND == KIND_PAIRS) {
            const int p0 = CS::load_pos(0), rem = v - p0;
            const uint32_t* s = reinterpret_cast<const uint32_t*>(src) + src_off + p0;
            const uint32_t* sv = src_v + src_off;
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) {
                const uint32_t key = 32 * k < rem ? __ldg(s + 32 * k) : 0xFFFFFFFFu;
                x[k] = ((T)key << 32) | (T)(uint32_t)(p0 + 32 * k);     // stable: ties by position
            }
            for (int p = threadIdx.x; p < v; p += BLOCK) vsm[p] = __ldg(sv + p);
        } else {
            const int p0 = CS::load_pos(0), rem = v - p0;
            const unsigned long long* s = reinterpret_cast<const unsigned long long*>(src) + src_off + p0;
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) x[k] = 32 * k < rem ? (T)__ldg(s + 32 * k) : (T)~0ull;
        }
        CS::sort(x, sm, v);
    }

    static __device__ __forceinline__ void store(void* dst, uint32_t* dst_v, uint64_t dst_off, int v,
                                                 const T* sm, const uint32_t* vsm)
    {
        if constexpr (KIND == KIND_KEYS) {
            uint32_t* d = reinterpret_cast<uint32_t*>(dst) + dst_off;
            for (int p = threadIdx.x; p < v; p += BLOCK) d[p] = (uint32_t)sm[CS::phys(p)];
        } else if constexpr (KIND == KIND_PAIRS) {
            uint32_t* d = reinterpret_cast<uint32_t*>(dst) + dst_off;
            uint32_t* dv = dst_v + dst_off;
            for (int p = threadIdx.x; p < v; p += BLOCK) {
                const T c = sm[CS::phys(p)];
                d[p] = (uint32_t)(c >> 32);
                dv[p] = vsm[(uint32_t)c];
            }
        } else {
            unsigned long long* d = reinterpret_cast<unsigned long long*>(dst) + dst_off;
            for (int p = threadIdx.x; p < v; p += BLOCK) d[p] = sm[CS::phys(p)];
        }
    }
};

// ------------------------------------------------------------ Steps 2 + 3
// Step 2: sort sublist A_i of problem b in place.  Step 3,
// fused into the write-back as the paper does: s samples at sorted
// positions (k+1)d - 1 (R2), as composites (key << 32 | tag), tag = iL + r (R3).
template <int KIND, int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK, 1) k_local_sort(LevelDev lv)
{
    using S = Seg<KIND, BLOCK, ITEMS>;
    using T = typename S::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    uint32_t* vsm = reinterpret_cast<uint32_t*>(sm + S::CS::SMEM_ELEMS);

    const uint32_t b = blockIdx.x / lv.m, i = blockIdx.x % lv.m;
    const uint64_t off = lv.pr.offset(b);
    const uint32_t len = lv.pr.length(b);
    const uint64_t i0 = (uint64_t)i * lv.L;
    const int v = len > i0 ? (int)umin64(len - i0, lv.L) : 0;

    if (threadIdx.x == 0 && blockIdx.x + lv.pf_stride < lv.B * lv.m) {
        uint64_t ps;
        int pv;
        sublist_of(lv, blockIdx.x + lv.pf_stride, ps, pv);
        prefetch_l2(reinterpret_cast<const char*>(lv.in) + ps * sizeof(typename S::KeyT), (size_t)pv * sizeof(typename S::KeyT));
        if (KIND == KIND_PAIRS) prefetch_l2(lv.in_v + ps, (size_t)pv * 4);
    }
    if (v > 0) {
        bool done = false;
        if constexpr (KIND == KIND_U64) {
            if (GBS_PRESORTED && lv.presorted >= (uint32_t)ITEMS) {
                const unsigned long long* src = reinterpret_cast<const unsigned long long*>(lv.in) + off + i0;
                S::CS::sort_presorted(src, sm, v, (int)lv.presorted);
                done = true;
            }
        }
        if (!done) S::load_sort(lv.in, lv.in_v, off + i0, v, sm, vsm);
        S::store(lv.in, lv.in_v, off + i0, v, sm, vsm);
    }
    u64* smp = lv.samples + ((uint64_t)b * lv.m + i) * lv.s;
    for (uint32_t k = threadIdx.x; k < lv.s; k += BLOCK) {
        const uint32_t r = (k + 1) * lv.d - 1;
        const uint32_t tag = (uint32_t)i0 + r;
        unsigned long long c;
        if (KIND == KIND_U64) {
            c = (int)r < v ? (unsigned long long)sm[S::CS::phys(r)] : pad64(lv.pad_base, i0 + r - len);
        } else {
            uint32_t key = 0xFFFFFFFFu;
            if ((int)r < v) key = KIND == KIND_KEYS ? (uint32_t)sm[S::CS::phys(r)]
                                                    : (uint32_t)((unsigned long long)sm[S::CS::phys(r)] >> 32);
            c = ((unsigned long long)key << 32) | tag;
        }
        smp[k] = c;
    }
}

// ------------------------------------------------------------ Step 5
// Global sampling: g_k = sorted_samples[(k+1)m - 1] (R2).
__global__ void k_global_samples(LevelDev lv)
{
    const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (uint64_t)lv.B * lv.s) return;
    const uint32_t b = (uint32_t)(idx / lv.s), k = (uint32_t)(idx % lv.s);
    lv.splitters[idx] = lv.samples[((uint64_t)b * lv.m) * lv.s + (uint64_t)(k + 1) * lv.m - 1];
}

// ------------------------------------------------------------ Step 6
// Sample indexing: for sorted sublist A_i and every global
// sample g_j, Q_ij = #{real r : (A_i[r], iL + r) <= g_j}; a_ij = Q_ij - Q_i,j-1
// (bucket j = (g_{j-1}, g_j], R4).  The sublist's keys are staged in shared memory
// (the paper loads the s global samples into shared memory); each thread
// bisects for its splitters -- the paper's staged schedule only avoided
// GT200 bank contention and does not change the result (R10).
template <int KIND, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_sample_index(LevelDev lv)
{
    using KT = typename std::conditional<KIND == KIND_U64, unsigned long long, uint32_t>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned long long* gs = reinterpret_cast<unsigned long long*>(smem_raw);
    uint32_t* Q = reinterpret_cast<uint32_t*>(gs + lv.s);
    KT* ks = reinterpret_cast<KT*>(Q + lv.s + (lv.s & 1));

    const uint32_t b = blockIdx.x / lv.m, i = blockIdx.x % lv.m;
    const uint64_t off = lv.pr.offset(b);
    const uint32_t len = lv.pr.length(b);
    const uint64_t i0 = (uint64_t)i * lv.L;
    const int v = len > i0 ? (int)umin64(len - i0, lv.L) : 0;

    const KT* src = reinterpret_cast<const KT*>(lv.in) + off + i0;
    if (threadIdx.x == 0 && blockIdx.x + lv.pf_stride < lv.B * lv.m) {
        uint64_t ps;
        int pv;
        sublist_of(lv, blockIdx.x + lv.pf_stride, ps, pv);
        prefetch_l2(reinterpret_cast<const KT*>(lv.in) + ps, (size_t)pv * sizeof(KT));
    }
    stage_to_smem<BLOCK>(ks, src, (size_t)v * sizeof(KT));
    const unsigned long long* g = lv.splitters + (uint64_t)b * lv.s;
    for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) gs[j] = g[j];
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) {
        const unsigned long long gj = gs[j];
        int lo = 0, hi = v;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            unsigned long long rk;
            if (KIND == KIND_U64) rk = (unsigned long long)ks[mid];
            else rk = ((unsigned long long)ks[mid] << 32) | (uint32_t)(i0 + mid);
            if (rk <= gj) lo = mid + 1; else hi = mid;
        }
        Q[j] = (uint32_t)lo;
    }
    __syncthreads();
    uint32_t* arow = lv.a + ((uint64_t)b * lv.m + i) * lv.s;
    for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) arow[j] = Q[j] - (j ? Q[j - 1] : 0u);
}

// ------------------------------------------------------------ Step 7
// Prefix sum: l = exclusive scan of a in the order
// a_11..a_m1, a_12, ... (column-major, R5) over row-major storage.  One CTA per block
// of 32 columns: pass 1 column sums (the paper's "parallel column sum"), one
// decoupled look-back across column blocks replaces the single-SM scan of column
// sums, pass 2 writes l (the paper's "final update").  Integer sums: deterministic.
static constexpr int SCAN_BLOCK = 512;
static constexpr unsigned long long LB_AGG = 1ull << 62, LB_INC = 2ull << 62, LB_VAL = (1ull << 62) - 1;

__global__ void __launch_bounds__(SCAN_BLOCK) k_scan(LevelDev lv)
{
    constexpr int NW = SCAN_BLOCK / 32;
    __shared__ uint32_t wsum[NW][33];
    __shared__ uint32_t colpre[32];
    __shared__ unsigned long long blk_prefix;
    const uint32_t nblk = (lv.s + 31) / 32;
    const uint32_t b = blockIdx.x / nblk, jb = blockIdx.x % nblk;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t c = jb * 32 + lane;
    const bool col_ok = c < lv.s;
    const uint64_t rows_per = (lv.m + NW - 1) / NW;
    const uint64_t r0 = (uint64_t)w * rows_per, r1 = umin64(r0 + rows_per, lv.m);
    const uint32_t* A = lv.a + (uint64_t)b * lv.m * lv.s;
    uint32_t* Lo = lv.l + (uint64_t)b * lv.m * lv.s;

    uint32_t sum = 0;
    if (col_ok) {
        uint64_t r = r0;
        for (; r + 4 <= r1; r += 4) {
            const uint32_t x0 = A[(r + 0) * lv.s + c], x1 = A[(r + 1) * lv.s + c];
            const uint32_t x2 = A[(r + 2) * lv.s + c], x3 = A[(r + 3) * lv.s + c];
            sum += x0 + x1 + x2 + x3;
        }
        for (; r < r1; ++r) sum += A[r * lv.s + c];
    }
    wsum[w][lane] = sum;
    __syncthreads();
    if (w == 0) {
        // per column: exclusive prefix over warps; column total
        uint32_t run = 0;
        for (int q = 0; q < NW; ++q) { const uint32_t x = wsum[q][lane]; wsum[q][lane] = run; run += x; }
        // exclusive scan of column totals across the 32 lanes
        uint32_t incl = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        colpre[lane] = incl - run;
        const unsigned long long agg = __shfl_sync(0xffffffffu, incl, 31);
        if (lane == 0) {
            unsigned long long* st = lv.state + (uint64_t)b * nblk;
            unsigned long long prefix = 0;
            if (jb == 0) {
                atomicExch(st + 0, LB_INC | agg);
            } else {
                atomicExch(st + jb, LB_AGG | agg);
                int q = (int)jb - 1;
                while (q >= 0) {
                    unsigned long long word;
                    do { word = atomicAdd(st + q, 0ull); } while ((word >> 62) == 0);
                    prefix += word & LB_VAL;
                    if ((word >> 62) == 2) break;
                    --q;
                }
                atomicExch(st + jb, LB_INC | (prefix + agg));
            }
            blk_prefix = prefix;
        }
    }
    __syncthreads();
    if (col_ok) {
        uint32_t run = (uint32_t)blk_prefix + colpre[lane] + wsum[w][lane];
        for (uint64_t r = r0; r < r1; ++r) {
            const uint32_t x = A[r * lv.s + c];
            Lo[r * lv.s + c] = run;
            run += x;
        }
    }
}

// ------------------------------------------------------------ Step 8
// Data relocation: R[l_ij + q] = A_i[start_ij + q], q < a_ij.
// Each thread maps a contiguous slice of positions to destinations (bucket of r =
// last j with start_j <= r), then the block copies position-ordered (coalesced:
// consecutive positions of one run go to consecutive addresses).
template <int BLOCK>
__device__ __forceinline__ void block_excl_scan(uint32_t* arr, int n, uint32_t* wtmp)
{
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int per = (n + BLOCK - 1) / BLOCK;
    const int c0 = min(n, t * per), c1 = min(n, c0 + per);
    uint32_t sum = 0;
    for (int q = c0; q < c1; ++q) sum += arr[q];
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wtmp[w] = incl;
    __syncthreads();
    if (w == 0) {
        uint32_t x = lane < BLOCK / 32 ? wtmp[lane] : 0, xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += y;
        }
        if (lane < BLOCK / 32) wtmp[lane] = xi - x;
    }
    __syncthreads();
    uint32_t run = wtmp[w] + incl - sum;
    for (int q = c0; q < c1; ++q) { const uint32_t x = arr[q]; arr[q] = run; run += x; }
    __syncthreads();
}

__device__ __forceinline__ int upper_bound_u32(const uint32_t* a, int lo, int hi, uint32_t x)
{
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// MAXPER = max items per thread (L / BLOCK): the sublist is prefetched into registers
// (striped, coalesced) while the destination map is built, then stored.
template <int KIND, int BLOCK, int MAXPER>
__global__ void __launch_bounds__(BLOCK, 1) k_relocate(LevelDev lv)
{
    using KT = typename std::conditional<KIND == KIND_U64, unsigned long long, uint32_t>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* starts = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* delta = starts + lv.s;
    uint32_t* dest = delta + lv.s;          // L + BLOCK entries (one pad slot per `per`)
    __shared__ uint32_t wtmp[32];

    const uint32_t b = blockIdx.x / lv.m, i = blockIdx.x % lv.m;
    const uint64_t off = lv.pr.offset(b);
    const uint32_t len = lv.pr.length(b);
    const uint64_t i0 = (uint64_t)i * lv.L;
    const int v = len > i0 ? (int)umin64(len - i0, lv.L) : 0;
    if (v == 0) return;

    // prefetch the sublist (striped: r = t + k*BLOCK) -- latency overlaps the map build
    const KT* src = reinterpret_cast<const KT*>(lv.in) + off + i0;
    if (threadIdx.x == 0 && blockIdx.x + lv.pf_stride < lv.B * lv.m) {
        uint64_t ps;
        int pv;
        sublist_of(lv, blockIdx.x + lv.pf_stride, ps, pv);
        prefetch_l2(reinterpret_cast<const KT*>(lv.in) + ps, (size_t)pv * sizeof(KT));
        if (KIND == KIND_PAIRS) prefetch_l2(lv.in_v + ps, (size_t)pv * 4);
    }
    KT x[MAXPER];
    {
        const int rem = v - (int)threadIdx.x;
        const KT* s0 = src + threadIdx.x;
#pragma unroll
        for (int k = 0; k < MAXPER; ++k) x[k] = k * BLOCK < rem ? s0[k * BLOCK] : KT(0);
    }

    const uint64_t row = ((uint64_t)b * lv.m + i) * lv.s;
    for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) starts[j] = lv.a[row + j];
    __syncthreads();
    block_excl_scan<BLOCK>(starts, (int)lv.s, wtmp);
    for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) delta[j] = lv.l[row + j] - starts[j];
    __syncthreads();

    // destination map: thread t walks positions [t*per, t*per + per) (blocked) and
    // writes dest at r + r/per (padding keeps the blocked writes bank-conflict free)
    const int S = (int)lv.s;
    const int per = (int)(lv.L / BLOCK) > 0 ? (int)(lv.L / BLOCK) : 1;   // power of two
    const int lp = 31 - __clz(per);
    const int r0 = threadIdx.x * per, r1 = min(v, r0 + per);
    if (r0 < r1) {
        int j = upper_bound_u32(starts, 0, S, (uint32_t)r0) - 1;
        for (int r = r0; r < r1; ++r) {
            if (j + 1 < S && starts[j + 1] <= (uint32_t)r) {
                ++j;
                if (j + 1 < S && starts[j + 1] <= (uint32_t)r) j = upper_bound_u32(starts, j + 1, S, (uint32_t)r) - 1;
            }
            dest[r + (r >> lp)] = (uint32_t)r + delta[j];
        }
    }
    __syncthreads();
    KT* dst = reinterpret_cast<KT*>(lv.reloc) + off;
#pragma unroll
    for (int k = 0; k < MAXPER; ++k) {
        const int r = threadIdx.x + k * BLOCK;
        if (r < v) dst[dest[r + (r >> lp)]] = x[k];
    }
    if (KIND == KIND_PAIRS) {
        const uint32_t* sv = lv.in_v + off + i0;
        uint32_t* dv = lv.reloc_v + off;
        uint32_t y[8];
        for (int r0v = threadIdx.x; r0v < v; r0v += 8 * BLOCK) {
#pragma unroll
            for (int u = 0; u < 8; ++u) y[u] = r0v + u * BLOCK < v ? sv[r0v + u * BLOCK] : 0u;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int r = r0v + u * BLOCK;
                if (r < v) dv[dest[r + (r >> lp)]] = y[u];
            }
        }
    }
}

// ------------------------------------------------------------ Step 9 (+ leaves)
// Sublist sort: one CTA per bucket B_j = R[l_0j, l_0j+|B_j|),
// |B_j| <= the tight bound <= tile capacity (checked by the planner).  MODE_LEAF:
// one CTA per whole problem (len_b <= tile).
enum SegMode { MODE_BUCKET = 0, MODE_LEAF = 1 };

// Sort v items with the smallest tile (ITEMS, ITEMS/2, ITEMS/4 per thread; same CTA)
// that holds them: every thread stays busy, so a bucket of half the capacity (the
// average, since the bound is ~2n/s) costs about half.  Block-uniform branch.
template <int KIND, int BLOCK, int ITEMS, int DEPTH>
__device__ __forceinline__ void seg_sort_adaptive(const void* src, const uint32_t* src_v, uint64_t off, int v,
                                                  void* dst, uint32_t* dst_v, unsigned char* smem_raw)
{
    if constexpr (DEPTH > 0 && ITEMS >= 8) {
        if (v <= BLOCK * ITEMS / 2) {
            seg_sort_adaptive<KIND, BLOCK, ITEMS / 2, DEPTH - 1>(src, src_v, off, v, dst, dst_v, smem_raw);
            return;
        }
    }
    using S = Seg<KIND, BLOCK, ITEMS>;
    using T = typename S::T;
    T* sm = reinterpret_cast<T*>(smem_raw);
    uint32_t* vsm = reinterpret_cast<uint32_t*>(sm + S::CS::SMEM_ELEMS);
    S::load_sort(src, src_v, off, v, sm, vsm);
    S::store(dst, dst_v, off, v, sm, vsm);
}

template <int KIND, int BLOCK, int ITEMS, int MODE>
__global__ void __launch_bounds__(BLOCK, 1) k_segment_sort(LevelDev lv)
{
    using S = Seg<KIND, BLOCK, ITEMS>;
    using T = typename S::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    uint32_t* vsm = reinterpret_cast<uint32_t*>(sm + S::CS::SMEM_ELEMS);

    uint32_t b;
    uint64_t start;
    int v;
    const void* src;
    const uint32_t* src_v;
    if (MODE == MODE_LEAF) {
        b = blockIdx.x;
        start = 0;
        v = (int)lv.pr.length(b);
        src = lv.in;
        src_v = lv.in_v;
    } else {
        b = blockIdx.x / lv.s;
        const uint32_t j = blockIdx.x % lv.s;
        const uint32_t* l0 = lv.l + (uint64_t)b * lv.m * lv.s;   // row 0 of problem b
        const uint32_t st = l0[j];
        const uint32_t en = j + 1 < lv.s ? l0[j + 1] : lv.pr.length(b);
        start = st;
        v = (int)(en - st);
        src = lv.reloc;
        src_v = lv.reloc_v;
        const uint32_t nxt = blockIdx.x + lv.pf_stride;
        if (threadIdx.x == 0 && nxt < lv.B * lv.s) {
            const uint32_t nb = nxt / lv.s, nj = nxt % lv.s;
            const uint32_t* n0 = lv.l + (uint64_t)nb * lv.m * lv.s;
            const uint32_t ns = n0[nj], ne = nj + 1 < lv.s ? n0[nj + 1] : lv.pr.length(nb);
            const uint64_t po = lv.pr.offset(nb) + ns;
            prefetch_l2(reinterpret_cast<const typename S::KeyT*>(lv.reloc) + po, (size_t)(ne - ns) * sizeof(typename S::KeyT));
            if (KIND == KIND_PAIRS) prefetch_l2(lv.reloc_v + po, (size_t)(ne - ns) * 4);
        }
    }
    if (v <= 0) return;
    const uint64_t off = lv.pr.offset(b) + start;
    (void)sm;
    (void)vsm;
    seg_sort_adaptive<KIND, BLOCK, ITEMS, GBS_ADAPT_DEPTH>(src, src_v, off, v, lv.out, lv.out_v, smem_raw);
}

// Nested Step 9: the buckets of this level become the problems of the next level.
__global__ void k_child_desc(LevelDev lv)
{
    const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (uint64_t)lv.B * lv.s) return;
    const uint32_t b = (uint32_t)(idx / lv.s), j = (uint32_t)(idx % lv.s);
    const uint32_t* l0 = lv.l + (uint64_t)b * lv.m * lv.s;
    const uint32_t st = l0[j];
    const uint32_t en = j + 1 < lv.s ? l0[j + 1] : lv.pr.length(b);
    lv.child_off[idx] = lv.pr.offset(b) + st;
    lv.child_len[idx] = en - st;
}

}  // namespace gbs
