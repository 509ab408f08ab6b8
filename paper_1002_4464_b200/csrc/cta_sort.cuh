// cta_sort.cuh -- on-chip sort of one tile (<= BLOCK*ITEMS items) by one CTA.
//
// Used for Step 2 (local sort of a sublist A_i), Step 9
// (sort of a bucket B_j) and single-tile problems.
// The paper sorted 2K items with a shared-memory bitonic network; any
// on-chip sort yields the same sorted tile, so on sm_100a we keep most of the work in
// registers: Batcher odd-even merge sort of ITEMS items per thread, then log2(BLOCK)
// merge-path levels through padded shared memory (the first five within a warp,
// synchronised with __syncwarp only).
//
// Valid items: the caller loads positions [0, valid) and fills every other slot with
// a sentinel that compares >= every real item.  Work is skipped for warps/threads
// whose output range lies entirely in the sentinel tail, so a half-full bucket costs
// about half a full one (Step 9 buckets average half the tile capacity).
#pragma once
#include <cstdint>
#include <utility>

namespace gbs {

template <int X> struct Log2 { static constexpr int value = 1 + Log2<X / 2>::value; };
template <> struct Log2<1> { static constexpr int value = 0; };

template <typename T>
__device__ __forceinline__ void cas(T& a, T& b)
{
    const bool sw = b < a;
    const T lo = sw ? b : a;
    const T hi = sw ? a : b;
    a = lo;
    b = hi;
}
template <>
__device__ __forceinline__ void cas<uint32_t>(uint32_t& a, uint32_t& b)
{
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

// Batcher odd-even merge sort network over N registers.  The comparator list is
// generated at compile time and applied with a fold expression, so every index is
// a constant and x[] stays in registers (no dynamic indexing -> no local memory).
template <int N>
struct BatcherNet {
    static constexpr int count()
    {
        int c = 0;
        for (int p = 1; p < N; p += p)
            for (int k = p; k > 0; k /= 2)
                for (int j = k % p; j + k < N; j += k + k)
                    for (int i = 0; i < k; ++i)
                        if (i + j + k < N && (i + j) / (p + p) == (i + j + k) / (p + p)) ++c;
        return c;
    }
    static constexpr int C = count();
    int a[C > 0 ? C : 1], b[C > 0 ? C : 1];
    constexpr BatcherNet() : a(), b()
    {
        int c = 0;
        for (int p = 1; p < N; p += p)
            for (int k = p; k > 0; k /= 2)
                for (int j = k % p; j + k < N; j += k + k)
                    for (int i = 0; i < k; ++i)
                        if (i + j + k < N && (i + j) / (p + p) == (i + j + k) / (p + p)) {
                            a[c] = i + j;
                            b[c] = i + j + k;
                            ++c;
                        }
    }
};

template <typename T, int N, size_t... Cs>
__device__ __forceinline__ void apply_net(T (&x)[N], std::index_sequence<Cs...>)
{
    constexpr BatcherNet<N> net{};
    (cas(x[net.a[Cs]], x[net.b[Cs]]), ...);
}

template <typename T, int N>
__device__ __forceinline__ void reg_sort(T (&x)[N])
{
    if constexpr (N > 1) apply_net<T, N>(x, std::make_index_sequence<BatcherNet<N>::C>{});
}

template <typename T, int BLOCK, int ITEMS>
struct CtaSort {
    static constexpr int TILE = BLOCK * ITEMS;
    static constexpr int LOG_ITEMS = Log2<ITEMS>::value;
    static constexpr int WARP_SPAN = 32 * ITEMS;                  // items owned by one warp
    // one pad slot per ITEMS items (bank-conflict-free blocked stores) + 1 overrun slot
    static constexpr int SMEM_ELEMS = TILE + TILE / ITEMS + 1;
    // independent merge chains per thread (ILP) when registers allow
    static constexpr int CHAINS = (ITEMS * sizeof(T) <= 128) ? 2 : 1;

    static __device__ __forceinline__ int phys(int p) { return p + (p >> LOG_ITEMS); }

    // Position of register slot k of the calling thread in the load order: each warp
    // owns a contiguous span of 32*ITEMS positions, read 32 consecutive at a time
    // (coalesced).  Valid positions then form a prefix of every warp span, which is
    // what the skip logic below relies on.
    static __device__ __forceinline__ int load_pos(int k)
    {
        return (threadIdx.x >> 5) * WARP_SPAN + k * 32 + (threadIdx.x & 31);
    }

    // Merge-path split of output diagonal `diag` of the pair (A = [a0, a0+w),
    // B = [a0+w, a0+2w)): number of outputs taken from A (ties: A first -> stable).
    static __device__ __forceinline__ int split(const T* sm, int a0, int w, int diag)
    {
        const int b0 = a0 + w;
        int lo = max(0, diag - w), hi = min(diag, w);
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sm[phys(a0 + mid)] <= sm[phys(b0 + diag - 1 - mid)]) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    }

    // The thread's ITEMS outputs [start, start+ITEMS) of the merge of the pair of
    // sorted runs of width w containing `start`, produced as two independent halves
    // (two merge-path chains interleaved for ILP: each step of a chain waits on one
    // shared-memory load).
    static __device__ __forceinline__ void merge_thread1(T (&x)[ITEMS], const T* sm, int start, int w)
    {
        const int base = start & ~(2 * w - 1);
        const int diag = start - base;
        const int aEnd = base + w, bEnd = base + 2 * w;
        const int s0 = split(sm, base, w, diag);
        int ai = base + s0, bi = aEnd + diag - s0;
        T a = sm[phys(ai)], b = sm[phys(bi)];
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const bool t = (ai < aEnd) && (bi >= bEnd || a <= b);
            x[k] = t ? a : b;
            const int n = (t ? ai : bi) + 1;
            ai += t ? 1 : 0;
            bi += t ? 0 : 1;
            const T v = sm[phys(n)];
            a = t ? v : a;
            b = t ? b : v;
        }
    }

    static __device__ __forceinline__ void merge_thread(T (&x)[ITEMS], const T* sm, int start, int w)
    {
        if constexpr (CHAINS == 1) { merge_thread1(x, sm, start, w); return; }
        constexpr int H = ITEMS / 2;
        const int base = start & ~(2 * w - 1);
        const int diag0 = start - base, diag1 = diag0 + H;
        const int aEnd = base + w, bEnd = base + 2 * w;
        const int s0 = split(sm, base, w, diag0);
        const int s1 = split(sm, base, w, diag1);
        int ai0 = base + s0, bi0 = aEnd + diag0 - s0;
        int ai1 = base + s1, bi1 = aEnd + diag1 - s1;
        T a0 = sm[phys(ai0)], b0 = sm[phys(bi0)];
        T a1 = sm[phys(ai1)], b1 = sm[phys(bi1)];
#pragma unroll
        for (int k = 0; k < H; ++k) {
            const bool t0 = (ai0 < aEnd) && (bi0 >= bEnd || a0 <= b0);
            const bool t1 = (ai1 < aEnd) && (bi1 >= bEnd || a1 <= b1);
            x[k] = t0 ? a0 : b0;
            x[H + k] = t1 ? a1 : b1;
            const int n0 = (t0 ? ai0 : bi0) + 1;
            const int n1 = (t1 ? ai1 : bi1) + 1;
            ai0 += t0 ? 1 : 0;
            bi0 += t0 ? 0 : 1;
            ai1 += t1 ? 1 : 0;
            bi1 += t1 ? 0 : 1;
            const T v0 = sm[phys(n0)];
            const T v1 = sm[phys(n1)];
            a0 = t0 ? v0 : a0;
            b0 = t0 ? b0 : v0;
            a1 = t1 ? v1 : a1;
            b1 = t1 ? b1 : v1;
        }
    }

    // Sort: x[] holds the items of positions load_pos(k) (sentinels at >= valid).
    // On return sm[phys(p)] holds the sorted tile for p < valid (block-synchronised).
    static __device__ __forceinline__ void sort(T (&x)[ITEMS], T* sm, int valid)
    {
        const int t = threadIdx.x;
        const int wspan0 = (t >> 5) * WARP_SPAN;
        if (wspan0 < valid) reg_sort<T, ITEMS>(x);
        const int start = t * ITEMS;
#pragma unroll 1
        for (int w = ITEMS; w < TILE; w *= 2) {
            const bool intra = 2 * w <= WARP_SPAN;
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) sm[phys(start + k)] = x[k];
            if (intra) __syncwarp(); else __syncthreads();
            const bool active = intra ? (wspan0 < valid) : (start < valid);
            if (active) merge_thread(x, sm, start, w);
            if (intra) __syncwarp(); else __syncthreads();
        }
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) sm[phys(start + k)] = x[k];
        __syncthreads();
    }
};

}  // namespace gbs
