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

#include <cooperative_groups.h>

#include "cta_sort.cuh"

namespace gbs {

typedef unsigned long long u64;
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// Programmatic dependent launch (sm_90+): every kernel of a sort lets its successor's
// CTAs launch as soon as all of its own CTAs are resident, and waits for its
// predecessor's completion (and memory) before touching global memory.  The successor
// thus fills the SMs the predecessor's last wave frees instead of waiting for the
// launch after the grid drains.  No-ops for a normal launch.
#ifndef GBS_GROUP_MAX_RUN
#define GBS_GROUP_MAX_RUN 256   // grouped Step 8 only when every run a_ij is at most this long
#endif

__device__ __forceinline__ void pdl_entry()
{
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

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
    uint32_t seg_min, seg_max;   // k_segment_sort: this launch sorts segments of seg_min < v <= seg_max
    // k_segment_sort over a size tier: the tier's bucket list (k_bucket_tiers) and its
    // length; null = one CTA per segment of the level
    const uint32_t* tier_list;
    const uint32_t* tier_len;
    // where Step 2 writes the sorted sublists (Steps 3, 6, 8 and the fused Step 8+9 read
    // them): `in` itself, or -- for the fused path when in == out -- the reloc buffer
    void* srt;
    uint32_t* srt_v;
    uint32_t* pex;        // fused Step 8+9: P_i,j-1 (run start in sublist i), row-major like a
    // host-pipelined calls (gbs_sort_keys_host): k_local_sort sorts tiles [tile_lo,
    // tile_hi) and k_segment_sort the segments [seg_lo, seg_hi) of the level (0, 0 = all)
    uint32_t tile_lo, tile_hi, seg_lo, seg_hi;
    // Step 7 records the longest run max a_ij here (zeroed with the look-back words);
    // Step 8 picks the grouped relocation only when runs are short (R21)
    uint32_t* maxrun;
    // typed keys: the transform applied where keys enter (Step 2 / leaf loads from `in`)
    // and leave (the last level's Step 9 / leaf stores to `out`); 0 = none
    int xf_in, xf_out;
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

#ifndef GBS_VEC_IO
#define GBS_VEC_IO 1        // keys tiles: 16-byte global loads / stores (A/B switch)
#endif
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

// Typed keys (NEXT-4): an order-preserving bijection of int32 / binary32 bit patterns onto
// u32 (xf = 1: int32, x ^ 2^31; xf = 2: float, negatives -> ~x, others -> x ^ 2^31) and its
// inverse.  Applied where keys enter the sort (Step 2's load, a leaf's load) and where they
// leave it (the last level's Step 9 store, a leaf's store): every intermediate array is in
// the u32 image, and no extra pass touches the keys (xf = 0: plain u32 keys).
__device__ __forceinline__ uint32_t key_fwd(uint32_t x, int type)
{
    if (type == 1) return x ^ 0x80000000u;
    return x ^ ((x >> 31) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ uint32_t key_inv(uint32_t x, int type)
{
    if (type == 1) return x ^ 0x80000000u;
    return x ^ ((x >> 31) ? 0x80000000u : 0xFFFFFFFFu);
}
__device__ __forceinline__ uint32_t xf_in(uint32_t x, int xf) { return xf ? key_fwd(x, xf) : x; }
__device__ __forceinline__ uint32_t xf_out(uint32_t x, int xf) { return xf ? key_inv(x, xf) : x; }

// ------------------------------------------------------------------ segment I/O
// One tile of `v` items at element offset `off` of an HBM buffer: registers <- HBM
// (load_regs), on-chip sort (sort: CS::sort, result in shared memory), HBM <- shared
// memory (store).  Keys and u64 composites; pairs are the specialisation below.
template <int KIND, int BLOCK, int ITEMS>
struct Seg {
    using T = typename ItemT<KIND>::T;
    using CS = CtaSort<T, BLOCK, ITEMS, (KIND == KIND_KEYS ? GBS_KEYS_CHAINS : GBS_WIDE_CHAINS)>;
    using KeyT = typename std::conditional<KIND == KIND_U64, unsigned long long, uint32_t>::type;  // in HBM
    static constexpr int TILE = CS::TILE;
    __host__ __device__ static constexpr size_t smem_bytes() { return sizeof(T) * CS::SMEM_ELEMS; }

    template <int M>
    static __device__ __forceinline__ void sort(T (&x)[M], unsigned char* smem, int v)
    {
        CS::sort(x, reinterpret_cast<T*>(smem), v);
    }
    // sorted item r (keys: the key; u64: the composite) after sort()
    static __device__ __forceinline__ T item_at(const unsigned char* smem, int r)
    {
        return reinterpret_cast<const T*>(smem)[CS::phys(r)];
    }

    // Registers <- the tile's v items; returns the count the CTA sort is to treat as valid
    // (items sit in a prefix of every warp span; sentinels elsewhere).  Keys load 16-byte
    // vectors: the tile is read from the 16-byte boundary at or below its start, slot
    // (j, c) of lane l in warp w holding position 128 j + 4 l + c + w 32 ITEMS - mis, so the
    // first mis slots are sentinels and the sort sees v + mis slots (one vector per 4 keys;
    // scalar loads only at the two ends).
    template <int M>
    static __device__ __forceinline__ int load_regs(T (&x)[M], const void* src, const uint32_t* src_v,
                                                    uint64_t off, int v, unsigned char* smem, int xf = 0)
    {
        if constexpr (KIND == KIND_KEYS) {
            const uint32_t* s = reinterpret_cast<const uint32_t*>(src) + off;
            const int mis = (int)(((uintptr_t)s >> 2) & 3);
            if (GBS_VEC_IO && ITEMS % 4 == 0 && v + mis <= TILE) {
                const uint32_t* a = s - mis;                  // 16-byte aligned
                const int q0 = (int)(threadIdx.x >> 5) * CS::WARP_SPAN + 4 * (int)(threadIdx.x & 31);
#pragma unroll
                for (int j = 0; j < ITEMS / 4; ++j) {
                    const int q = q0 + 128 * j, p = q - mis;
                    if (p >= 0 && p + 3 < v) {
                        const uint4 u = __ldg(reinterpret_cast<const uint4*>(a + q));
                        x[4 * j] = xf_in(u.x, xf);
                        x[4 * j + 1] = xf_in(u.y, xf);
                        x[4 * j + 2] = xf_in(u.z, xf);
                        x[4 * j + 3] = xf_in(u.w, xf);
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            x[4 * j + c] = (p + c >= 0 && p + c < v) ? xf_in(__ldg(a + q + c), xf) : CS::TMAX;
                    }
                }
                return v + mis;
            }
            const int p0 = CS::load_pos(0), rem = v - p0;     // load_pos(k) = p0 + 32k
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) x[k] = 32 * k < rem ? xf_in(s[p0 + 32 * k], xf) : CS::TMAX;
        } else {
            CS::load(x, reinterpret_cast<const KeyT*>(src) + off, v);
        }
        return v;
    }

    // Fused Step 8+9: register slot k holds bucket position load_pos(k) (32 consecutive
    // positions per warp instruction, as for a relocated bucket, so the reads stay
    // coalesced inside each run).  Each lane finds the run of its first position by
    // binary search over the run table, then walks forward (positions only grow).
    template <int M, typename G>
    static __device__ __forceinline__ void load_gather(T (&x)[M], const G& g, int v, unsigned char* smem)
    {
        const int pbase = CS::load_pos(0);            // + 32 k
        int i = 0;
        if (pbase < v) {
            int lo = 0, hi = g.m - 1;                 // last run i with start_i <= pbase
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if ((int)g.run[mid].x <= pbase) lo = mid;
                else hi = mid - 1;
            }
            i = lo;
        }
        uint32_t base = g.run[i].y;
        uint2 nx = g.run[i + 1];
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const int p = pbase + 32 * k;
            if (p < v) {
                while (p >= (int)nx.x) {              // next non-empty run
                    base = nx.y;
                    ++i;
                    nx = g.run[i + 1];
                }
                const uint32_t q = base + (uint32_t)p;
                x[k] = (T)__ldg(reinterpret_cast<const KeyT*>(g.src) + q);
            } else {
                x[k] = CS::TMAX;
            }
        }
    }

    static __device__ __forceinline__ void store(void* dst, uint32_t* dst_v, uint64_t dst_off, int v,
                                                 unsigned char* smem, int xf = 0)
    {
        const T* sm = reinterpret_cast<const T*>(smem);
        if constexpr (KIND == KIND_KEYS) {
            uint32_t* d = reinterpret_cast<uint32_t*>(dst) + dst_off;
            if (GBS_VEC_IO) {
                // 16-byte stores: group g = positions 4g - mis .. 4g - mis + 3 lands on the
                // g-th 16-byte word at or after the boundary below d (scalar at the ends);
                // the four shared-memory reads of a group are conflict-free across a warp
                const int mis = (int)(((uintptr_t)d >> 2) & 3);
                uint32_t* a = d - mis;
                const int ng = (v + mis + 3) >> 2;
                for (int g = threadIdx.x; g < ng; g += BLOCK) {
                    const int p = 4 * g - mis;
                    if (p >= 0 && p + 3 < v) {
                        uint4 u;
                        u.x = xf_out((uint32_t)sm[CS::phys(p)], xf);
                        u.y = xf_out((uint32_t)sm[CS::phys(p + 1)], xf);
                        u.z = xf_out((uint32_t)sm[CS::phys(p + 2)], xf);
                        u.w = xf_out((uint32_t)sm[CS::phys(p + 3)], xf);
                        *reinterpret_cast<uint4*>(a + 4 * g) = u;
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; ++c)
                            if (p + c >= 0 && p + c < v) a[4 * g + c] = xf_out((uint32_t)sm[CS::phys(p + c)], xf);
                    }
                }
            } else if constexpr (BLOCK % (1 << CS::PAD) == 0) {
                // position tid + k BLOCK sits at phys(tid) + k (BLOCK + BLOCK >> PAD): one
                // address, constant offsets (BLOCK is a multiple of the pad group)
                const int t = threadIdx.x;
                const T* s0 = sm + CS::phys(t);
                uint32_t* d0 = d + t;
#pragma unroll
                for (int k = 0; k < ITEMS; ++k)
                    if (t + k * BLOCK < v) d0[k * BLOCK] = xf_out((uint32_t)s0[k * (BLOCK + (BLOCK >> CS::PAD))], xf);
            } else {
                for (int p = threadIdx.x; p < v; p += BLOCK) d[p] = xf_out((uint32_t)sm[CS::phys(p)], xf);
            }
        } else {
            unsigned long long* d = reinterpret_cast<unsigned long long*>(dst) + dst_off;
            for (int p = threadIdx.x; p < v; p += BLOCK) d[p] = sm[CS::phys(p)];
        }
    }
};

// Pairs (u32 key -> u32 value, stable by key; R7).  Sorting (key << 32 | position)
// composites moves 8 bytes per item through every shared-memory merge level; the tile
// instead sorts 4-byte packed items P = (prefix << POSB) | position, prefix = the top
// 32 - POSB bits of key - min (the tile's key range shifted into 32 - POSB bits), on the
// keys' CtaSort, then restores the exact order (key, position):
//   - prefix is monotone in key, so only items of equal prefix can be out of key order,
//     and inside such a group the sort left them in position order;
//   - with the keys gathered by position, odd-even transposition sort restricted to
//     neighbours of equal prefix (swap iff the later key is strictly smaller) sorts every
//     group by key with equal keys kept in position order -- the stable order.  It stops
//     after the first round pair with no swap (one round pair when the keys never
//     collide in their prefix: a key range below 2^(32-POSB), equal keys, presorted runs).
// Uniform keys over a tile of 2^14 give groups of 1-4 items (2-3 round pairs).  A tile
// whose key range fits the prefix (shift 0: the prefix is key - min itself) needs neither
// the gather nor the fix-up, and its keys are read back from P (MODE_EXACT).  A tile
// whose groups need more than PK_MAX_ITERS round pairs (a long unsorted run of keys
// sharing a prefix) is sorted as (key << 32 | position) composites instead, in the same
// shared memory: the result is identical either way (the stable sort), only the cost
// differs.  Values are parked at their positions and gathered at the write-back.
#ifndef GBS_PAIRS_SHFL_LEVELS
#define GBS_PAIRS_SHFL_LEVELS 5   // packed pairs tiles of 32 items per thread: 5 warp-shuffle merge levels (C4 57.6 / 57.3 / 57.0 ms with 3 / 4 / 5)
#endif
#ifndef GBS_PAIRS_SHFL_LEVELS_SMALL
#define GBS_PAIRS_SHFL_LEVELS_SMALL 3   // ... of 16 or fewer (Step 9 tiers: 4 measured +0.06 ms)
#endif
#ifndef GBS_PK_MAX_ITERS
#define GBS_PK_MAX_ITERS 16
#endif
template <int BLOCK, int ITEMS>
struct Seg<KIND_PAIRS, BLOCK, ITEMS> {
    using T = uint32_t;                                   // register items: keys, then P
    using KeyT = uint32_t;                                // in HBM
    using CS = CtaSort<uint32_t, BLOCK, ITEMS, GBS_KEYS_CHAINS,
                       (ITEMS >= 32 ? GBS_PAIRS_SHFL_LEVELS : GBS_PAIRS_SHFL_LEVELS_SMALL)>;
    using CS64 = CtaSort<unsigned long long, BLOCK, ITEMS, GBS_WIDE_CHAINS>;   // fallback
    static constexpr int TILE = CS::TILE;
    static constexpr int NW = BLOCK / 32;
    static constexpr int POSB = Log2<TILE>::value + ((TILE & (TILE - 1)) ? 1 : 0);   // position bits
    static constexpr uint32_t PMASK = (1u << POSB) - 1;
    static_assert(POSB <= 16 && ITEMS % 2 == 0 && BLOCK % 32 == 0, "packed pairs tile");
    static_assert(CS::SMEM_ELEMS == CS64::SMEM_ELEMS, "one padded layout for both sorts");
    struct Ctrl {
        uint32_t mn[NW], mx[NW];          // key range reduction
        uint32_t fP[NW], fK[NW], lP[NW], lK[NW];   // first / last item of every warp
        int mode;                         // MODE_FIXED, MODE_EXACT or MODE_COMPOSITE
        uint32_t klo;                     // MODE_EXACT: key = klo + (P >> POSB)
    };
    // MODE_EXACT: the key range fits the prefix (shift 0), so the prefix is key - min
    // itself and the packed sort alone is the stable order (no gather, no fix-up);
    // MODE_FIXED: sorted keys in ksm after the fix-up; MODE_COMPOSITE: the fallback
    enum { MODE_FIXED = 0, MODE_EXACT = 1, MODE_COMPOSITE = 2 };
    // shared memory: [ psm u32 | ksm u32 ] (or the fallback's u64 array) | vsm u32 | Ctrl
    __host__ __device__ static constexpr size_t region_bytes() { return 8 * (size_t)CS::SMEM_ELEMS; }
    __host__ __device__ static constexpr size_t smem_bytes()
    {
        return region_bytes() + 4 * (size_t)TILE + sizeof(Ctrl);
    }
    static __device__ __forceinline__ uint32_t* psm_of(unsigned char* smem) { return reinterpret_cast<uint32_t*>(smem); }
    static __device__ __forceinline__ uint32_t* ksm_of(unsigned char* smem)
    {
        return reinterpret_cast<uint32_t*>(smem) + CS::SMEM_ELEMS;
    }
    static __device__ __forceinline__ uint32_t* vsm_of(unsigned char* smem)
    {
        return reinterpret_cast<uint32_t*>(smem + region_bytes());
    }
    static __device__ __forceinline__ Ctrl* ctrl_of(unsigned char* smem)
    {
        return reinterpret_cast<Ctrl*>(smem + region_bytes() + 4 * (size_t)TILE);
    }

    // the keys of positions load_pos(k) (0xFFFFFFFF beyond v; registers only, so it may
    // run while the previous tile is written back)
    template <int M>
    static __device__ __forceinline__ void load_keys(uint32_t (&x)[M], const void* src, uint64_t off, int v, int xf = 0)
    {
        const int p0 = CS::load_pos(0), rem = v - p0;
        const uint32_t* s = reinterpret_cast<const uint32_t*>(src) + off + p0;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) x[k] = 32 * k < rem ? xf_in(__ldg(s + 32 * k), xf) : 0xFFFFFFFFu;
    }
    // the values parked in shared memory at their positions: every load of the thread in
    // flight before the stores
    static __device__ __forceinline__ void load_vals(const uint32_t* src_v, uint64_t off, int v, unsigned char* smem)
    {
        uint32_t* vsm = vsm_of(smem);
        const uint32_t* sv = src_v + off;
        constexpr int PER = (TILE + BLOCK - 1) / BLOCK;
        uint32_t t[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int p = (int)threadIdx.x + k * BLOCK;
            t[k] = p < v ? __ldg(sv + p) : 0u;
        }
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int p = (int)threadIdx.x + k * BLOCK;
            if (p < v) vsm[p] = t[k];
        }
    }
    template <int M>
    static __device__ __forceinline__ int load_regs(uint32_t (&x)[M], const void* src, const uint32_t* src_v,
                                                    uint64_t off, int v, unsigned char* smem, int xf = 0)
    {
        load_keys(x, src, off, v, xf);
        load_vals(src_v, off, v, smem);
        return v;
    }
    // fused Step 8+9: bucket position load_pos(k) gathered through the run table (see the
    // primary template); the value parked at its position
    template <int M, typename G>
    static __device__ __forceinline__ void load_gather(uint32_t (&x)[M], const G& g, int v, unsigned char* smem)
    {
        const int pbase = CS::load_pos(0);
        int i = 0;
        if (pbase < v) {
            int lo = 0, hi = g.m - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if ((int)g.run[mid].x <= pbase) lo = mid;
                else hi = mid - 1;
            }
            i = lo;
        }
        uint32_t base = g.run[i].y;
        uint2 nx = g.run[i + 1];
        uint32_t* vsm = vsm_of(smem);
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const int p = pbase + 32 * k;
            if (p < v) {
                while (p >= (int)nx.x) {
                    base = nx.y;
                    ++i;
                    nx = g.run[i + 1];
                }
                const uint32_t q = base + (uint32_t)p;
                x[k] = __ldg(reinterpret_cast<const uint32_t*>(g.src) + q);
                vsm[p] = __ldg(g.src_v + q);
            } else {
                x[k] = 0xFFFFFFFFu;
            }
        }
    }

    // compare-exchange of neighbours a (earlier) and b inside one prefix group
    static __device__ __forceinline__ void cx(bool eq, uint32_t& pa, uint32_t& ka, uint32_t& pb, uint32_t& kb, bool& sw)
    {
        const bool s = eq && kb < ka;
        const uint32_t p0 = s ? pb : pa, p1 = s ? pa : pb, k0 = s ? kb : ka, k1 = s ? ka : kb;
        pa = p0; pb = p1; ka = k0; kb = k1;
        sw |= s;
    }

    // x[k] = the key of position load_pos(k) (0xFFFFFFFF beyond v).  On return the
    // tile's stable order is in shared memory (key_at / store).  Block-synchronised.
    template <int M>
    static __device__ __forceinline__ void sort(uint32_t (&x)[M], unsigned char* smem, int v)
    {
        uint32_t* psm = psm_of(smem);
        uint32_t* ksm = ksm_of(smem);
        Ctrl* c = ctrl_of(smem);
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        const int p0 = CS::load_pos(0);
        // keys parked at their positions (the fix-up gathers them); the tile's key range
        uint32_t lo = 0xFFFFFFFFu, hi = 0;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            if (p0 + 32 * k < v) {
                ksm[CS::phys(p0 + 32 * k)] = x[k];
                lo = min(lo, x[k]);
                hi = max(hi, x[k]);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
            c->mn[w] = lo;
            c->mx[w] = hi;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            lo = min(lo, c->mn[q]);
            hi = max(hi, c->mx[q]);
        }
        const int bits = hi > lo ? 32 - __clz((int)(hi - lo)) : 0;
        const int shift = max(0, bits - (32 - POSB));
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const int p = p0 + 32 * k;
            x[k] = p < v ? (((x[k] - lo) >> shift) << POSB) | (uint32_t)p : 0xFFFFFFFFu;
        }
        if (threadIdx.x == 0) {   // read by key_at / store after the sort's barriers
            c->mode = shift ? MODE_FIXED : MODE_EXACT;
            c->klo = lo;
        }
        CS::sort(x, psm, v);     // x: the thread's sorted outputs [start, start + ITEMS)
        if (shift == 0) return;  // (the sort ends on a barrier)

        // exact order inside prefix groups: odd-even transposition on (prefix, key)
        const int start = threadIdx.x * ITEMS;
        uint32_t K[ITEMS];
        uint32_t eqm = 0;        // bit i: items i and i+1 share a prefix (invariant under swaps)
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) K[i] = start + i < v ? ksm[CS::phys(x[i] & PMASK)] : 0xFFFFFFFFu;
#pragma unroll   // (sentinels past v never move: they take no part in any group)
        for (int i = 0; i + 1 < ITEMS; ++i)
            eqm |= (start + i + 1 < v && (x[i] >> POSB) == (x[i + 1] >> POSB) ? 1u : 0u) << i;
        // Odd-even transposition sorts a group of g items in g rounds (any starting
        // parity), and groups never change (the prefixes are invariant), so when every
        // group is known to be short the rounds run a fixed count with no convergence
        // vote: g_max = the largest group, from the runs of eqm and the groups crossing a
        // thread boundary (tail of t + head of t + 1); a group that may span three threads
        // (a thread whose items all share one prefix) takes the voting loop instead.
        constexpr uint32_t FULL = (ITEMS >= 33) ? 0xFFFFFFFFu : ((1u << (ITEMS - 1)) - 1u);
        const bool full = eqm == FULL;
        int rounds = -1;   // -1: vote until a round pair swaps nothing
        {
            uint32_t m = eqm;
            int rint = 0;
            while (m) {
                m &= m >> 1;
                ++rint;
            }
            const int lead = full ? ITEMS - 1 : __ffs(~eqm) - 1;            // leading ones of eqm
            const int tail = full ? ITEMS - 1 : (eqm & (1u << (ITEMS - 2))) ? (ITEMS - 1 - (32 - __clz(~eqm & FULL))) : 0;
            const uint32_t info = (uint32_t)lead | (full ? 0x10000u : 0u);
            uint32_t nP = __shfl_down_sync(0xffffffffu, x[0], 1), nI = __shfl_down_sync(0xffffffffu, info, 1);
            if (lane == 0) {
                c->fP[w] = x[0];
                c->fK[w] = info;
            }
            __syncthreads();
            const bool has_next = threadIdx.x + 1 < BLOCK;
            if (lane == 31 && has_next) {
                nP = c->fP[w + 1];
                nI = c->fK[w + 1];
            }
            int g = rint + 1;
            bool lng = false;
            if (has_next && start + ITEMS < v && (x[ITEMS - 1] >> POSB) == (nP >> POSB)) {
                g = max(g, tail + 1 + (int)(nI & 0xFFFFu) + 1);
                lng = full || (nI >> 16);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                g = max(g, __shfl_xor_sync(0xffffffffu, g, o));
                lng |= __shfl_xor_sync(0xffffffffu, lng ? 1 : 0, o) != 0;
            }
            if (lane == 0) {
                c->mx[w] = (uint32_t)g;
                c->mn[w] = lng ? 1u : 0u;
            }
            __syncthreads();
            uint32_t gm = 0, lm = 0;
#pragma unroll
            for (int q = 0; q < NW; ++q) {
                gm = max(gm, c->mx[q]);
                lm |= c->mn[q];
            }
            if (!lm && gm <= 2 * GBS_PK_MAX_ITERS) rounds = gm <= 1 ? 0 : (int)gm;
        }
        int iter = 0, fb = 0;
        for (; rounds != 0;) {
            bool sw = false;
            if (eqm) {
#pragma unroll
                for (int i = 0; i + 1 < ITEMS; i += 2) cx((eqm >> i) & 1, x[i], K[i], x[i + 1], K[i + 1], sw);
#pragma unroll
                for (int i = 1; i + 1 < ITEMS; i += 2) cx((eqm >> i) & 1, x[i], K[i], x[i + 1], K[i + 1], sw);
            }
            // odd pair across threads: (last of t, first of t + 1)
            uint32_t fP = __shfl_down_sync(0xffffffffu, x[0], 1), fK = __shfl_down_sync(0xffffffffu, K[0], 1);
            uint32_t lP = __shfl_up_sync(0xffffffffu, x[ITEMS - 1], 1), lK = __shfl_up_sync(0xffffffffu, K[ITEMS - 1], 1);
            if (lane == 0) {
                c->fP[w] = x[0];
                c->fK[w] = K[0];
            }
            if (lane == 31) {
                c->lP[w] = x[ITEMS - 1];
                c->lK[w] = K[ITEMS - 1];
            }
            __syncthreads();
            const bool has_next = threadIdx.x + 1 < BLOCK, has_prev = threadIdx.x > 0;
            if (lane == 31 && has_next) {
                fP = c->fP[w + 1];
                fK = c->fK[w + 1];
            }
            if (lane == 0 && has_prev) {
                lP = c->lP[w - 1];
                lK = c->lK[w - 1];
            }
            if (has_next && (x[ITEMS - 1] >> POSB) == (fP >> POSB) && fK < K[ITEMS - 1]) {
                x[ITEMS - 1] = fP;
                K[ITEMS - 1] = fK;
                sw = true;
            }
            if (has_prev && (lP >> POSB) == (x[0] >> POSB) && K[0] < lK) {
                x[0] = lP;
                K[0] = lK;
                sw = true;
            }
            if (rounds > 0) {    // a fixed number of round pairs
                __syncthreads(); // (c->fP / lP reused by the next round pair)
                rounds -= 2;
                if (rounds < 0) rounds = 0;
                continue;
            }
            if (!__syncthreads_or(sw)) break;
            if (++iter == GBS_PK_MAX_ITERS) {
                fb = 1;
                break;
            }
        }
        if (!fb) {
            // every gather is done (the loop ends on a barrier): sorted keys and P in place
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                ksm[CS::phys(start + i)] = K[i];
                psm[CS::phys(start + i)] = x[i];
            }
            __syncthreads();
            return;
        }
        composite_sort(smem, v);
    }

    // fallback (cold, out of line so that its 64-bit registers do not weigh on the packed
    // path): the stable sort of (key << 32 | position) composites of the parked keys
    static __device__ __noinline__ void composite_sort(unsigned char* smem, int v)
    {
        Ctrl* c = ctrl_of(smem);
        const uint32_t* ksm = ksm_of(smem);
        const int p0 = CS::load_pos(0);
        if (threadIdx.x == 0) c->mode = MODE_COMPOSITE;
        unsigned long long xx[ITEMS];
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const int p = p0 + 32 * k;
            xx[k] = p < v ? ((unsigned long long)ksm[CS::phys(p)] << 32) | (unsigned)p : ~0ull;
        }
        __syncthreads();         // ksm read before the composites overwrite it
        CS64::sort(xx, reinterpret_cast<unsigned long long*>(smem), v);
    }

    // key of sorted item r (after sort)
    static __device__ __forceinline__ uint32_t key_at(unsigned char* smem, int r)
    {
        const Ctrl* c = ctrl_of(smem);
        if (c->mode == MODE_EXACT) return c->klo + (psm_of(smem)[CS::phys(r)] >> POSB);
        if (c->mode == MODE_COMPOSITE)
            return (uint32_t)(reinterpret_cast<const unsigned long long*>(smem)[CS::phys(r)] >> 32);
        return ksm_of(smem)[CS::phys(r)];
    }
    static __device__ __forceinline__ uint32_t item_at(unsigned char* smem, int r) { return key_at(smem, r); }

    static __device__ __forceinline__ void store(void* dst, uint32_t* dst_v, uint64_t dst_off, int v,
                                                 unsigned char* smem, int xf = 0)
    {
        const uint32_t* vsm = vsm_of(smem);
        uint32_t* d = reinterpret_cast<uint32_t*>(dst) + dst_off;
        uint32_t* dv = dst_v + dst_off;
        const Ctrl* c = ctrl_of(smem);
        const uint32_t* psm = psm_of(smem);
        if (c->mode == MODE_EXACT) {
            const uint32_t klo = c->klo;
            for (int p = threadIdx.x; p < v; p += BLOCK) {
                const uint32_t P = psm[CS::phys(p)];
                d[p] = xf_out(klo + (P >> POSB), xf);
                dv[p] = vsm[P & PMASK];
            }
            return;
        }
        if (c->mode == MODE_COMPOSITE) {
            const unsigned long long* sm = reinterpret_cast<const unsigned long long*>(smem);
            for (int p = threadIdx.x; p < v; p += BLOCK) {
                const unsigned long long cc = sm[CS::phys(p)];
                d[p] = xf_out((uint32_t)(cc >> 32), xf);
                dv[p] = vsm[(uint32_t)cc];
            }
            return;
        }
        const uint32_t* ksm = ksm_of(smem);
        for (int p = threadIdx.x; p < v; p += BLOCK) {
            d[p] = xf_out(ksm[CS::phys(p)], xf);
            dv[p] = vsm[psm[CS::phys(p)] & PMASK];
        }
    }
};

// Fused Step 8+9: where bucket j's items come from.  Relocation (Step 8,
// P:235-239) would copy run (i, j) -- the a_ij items of sorted sublist i starting at
// P_i,j-1 -- to R[l_ij + q]; the bucket's CTA instead reads position p of B_j (in R's
// order) straight from the sorted sublists: run i covers positions [lrel_i, lrel_i+1)
// with lrel_i = l_ij - l_0j, and position p is sorted-sublist item i*L + P_i,j-1 +
// (p - lrel_i).  The run table is staged in shared memory behind the tile.
struct GatherSrc {
    const void* src;          // sorted sublists of the bucket's problem (item 0 of sublist 0)
    const uint32_t* src_v;
    // run table in shared memory, m + 1 entries: x = lrel_i (run i's first bucket
    // position; x of entry m = |B_j|), y = i*L + P_i,j-1 - lrel_i, so that bucket position
    // p of run i is item y + p of the problem (32-bit modular: a problem has < 2^32 items)
    const uint2* run;
    int m;
};

// The same CTA sorts a tile of v items with ITEMS, ITEMS/2 or ITEMS/4 items per thread
// -- the smallest that holds v (block-uniform choice) -- so every thread stays busy: a
// bucket of half the capacity (the average, the bound being ~2n/s) costs about half.
// One register array of ITEMS entries serves every size.
template <int KIND, int BLOCK, int ITEMS, int DEPTH>
struct Adapt {
    using S = Seg<KIND, BLOCK, ITEMS>;
    using T = typename S::T;
    static constexpr bool HALF = DEPTH > 0 && ITEMS >= 8;
    using Sub = Adapt<KIND, BLOCK, (HALF ? ITEMS / 2 : ITEMS), (HALF ? DEPTH - 1 : 0)>;

    template <int M>
    static __device__ __forceinline__ int load(T (&x)[M], const void* src, const uint32_t* src_v, uint64_t off,
                                               int v, unsigned char* smem, int xf = 0)
    {
        if constexpr (HALF) {
            if (v <= S::TILE / 2) return Sub::load(x, src, src_v, off, v, smem, xf);
        }
        return S::load_regs(x, src, src_v, off, v, smem, xf);
    }
    template <int M>
    static __device__ __forceinline__ void sort(T (&x)[M], unsigned char* smem, int v)
    {
        if constexpr (HALF) {
            if (v <= S::TILE / 2) { Sub::sort(x, smem, v); return; }
        }
        S::sort(x, smem, v);
    }
    static __device__ __forceinline__ void store(void* dst, uint32_t* dst_v, uint64_t off, int v, unsigned char* smem,
                                                 int xf = 0)
    {
        if constexpr (HALF) {
            if (v <= S::TILE / 2) { Sub::store(dst, dst_v, off, v, smem, xf); return; }
        }
        S::store(dst, dst_v, off, v, smem, xf);
    }
    // fused Step 8+9: gather + sort + store, register array sized for the chosen tile
    template <typename G>
    static __device__ __forceinline__ void run_gather(const G& g, int v, void* dst, uint32_t* dst_v, uint64_t off,
                                                      unsigned char* smem, int xf_o = 0)
    {
        if constexpr (HALF) {
            if (v <= S::TILE / 2) { Sub::run_gather(g, v, dst, dst_v, off, smem, xf_o); return; }
        }
        T x[ITEMS];
        S::load_gather(x, g, v, smem);
        S::sort(x, smem, v);
        S::store(dst, dst_v, off, v, smem, xf_o);
    }
    // load + sort + store with a register array sized for the chosen tile
    static __device__ __forceinline__ void run(const void* src, const uint32_t* src_v, uint64_t off, int v,
                                               void* dst, uint32_t* dst_v, unsigned char* smem, int xf_i = 0,
                                               int xf_o = 0)
    {
        if constexpr (HALF) {
            if (v <= S::TILE / 2) { Sub::run(src, src_v, off, v, dst, dst_v, smem, xf_i, xf_o); return; }
        }
        T x[ITEMS];
        const int vs = S::load_regs(x, src, src_v, off, v, smem, xf_i);
        S::sort(x, smem, vs);
        S::store(dst, dst_v, off, v, smem, xf_o);
    }
};

// ------------------------------------------------------------ Steps 2 + 3
// Step 2: sort sublist A_i of problem b in place.  Step 3,
// fused into the write-back as the paper does: s samples at sorted
// positions (k+1)d - 1 (R2), as composites (key << 32 | tag), tag = iL + r (R3).
// Persistent CTAs (grid = SMs x CTAs/SM) walk the sublists; for keys and u64 the next
// sublist is loaded into registers while the current one is written back (software
// pipelining: the HBM load latency hides behind the store phase), and it is
// prefetched into L2 one sublist ahead.
template <int KIND, int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK, 1) k_local_sort(LevelDev lv)
{
    pdl_entry();
    using S = Seg<KIND, BLOCK, ITEMS>;
    using T = typename S::T;
    using KeyT = typename S::KeyT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);

    const uint32_t ntiles = lv.tile_hi ? lv.tile_hi : lv.B * lv.m;
    const bool presorted = KIND == KIND_U64 && GBS_PRESORTED && lv.presorted >= (uint32_t)ITEMS;
    // the next sublist's items (pairs: keys) are loaded into the free registers while the
    // current one is written back; pairs load their values before the sort (parked in
    // shared memory, their latency overlaps the register phase of the sort)
    const bool pipe = !presorted;
    T x[ITEMS];
    uint32_t tile = lv.tile_lo + blockIdx.x;
    uint64_t start = 0;
    int v = 0;
    auto load_next = [&](uint64_t st, int vv) -> int {   // into registers (pairs: the keys)
        if constexpr (KIND == KIND_PAIRS) {
            S::load_keys(x, lv.in, st, vv, lv.xf_in);
            return vv;
        } else {
            return S::load_regs(x, lv.in, lv.in_v, st, vv, smem_raw, lv.xf_in);
        }
    };
    int vs = 0;                      // the count the CTA sort treats as valid (load_regs)
    if (tile < ntiles) {
        sublist_of(lv, tile, start, v);
        if (pipe) vs = load_next(start, v);
    }
    for (; tile < ntiles; tile += gridDim.x) {
        const uint32_t b = tile / lv.m, i = tile % lv.m;
        const uint32_t len = lv.pr.length(b);
        const uint64_t i0 = (uint64_t)i * lv.L;
        const uint32_t nxt = tile + gridDim.x;
        uint64_t nstart = 0;
        int nv = 0;
        if (nxt < ntiles) {
            sublist_of(lv, nxt, nstart, nv);
            if (threadIdx.x == 0) {
                prefetch_l2(reinterpret_cast<const KeyT*>(lv.in) + nstart, (size_t)nv * sizeof(KeyT));
                if (KIND == KIND_PAIRS) prefetch_l2(lv.in_v + nstart, (size_t)nv * 4);
            }
        }
        if (v > 0) {
            if (presorted) {
                if constexpr (KIND == KIND_U64)
                    S::CS::sort_presorted(x, reinterpret_cast<const unsigned long long*>(lv.in) + start, sm, v,
                                          (int)lv.presorted);
            } else {
                if constexpr (KIND == KIND_PAIRS) S::load_vals(lv.in_v, start, v, smem_raw);
                S::sort(x, smem_raw, vs);
            }
        }
        int nvs = 0;
        if (pipe && nv > 0) nvs = load_next(nstart, nv);   // in flight during the store
        if (v > 0) S::store(lv.srt, lv.srt_v, start, v, smem_raw);
        u64* smp = lv.samples + ((uint64_t)b * lv.m + i) * lv.s;
        for (uint32_t k = threadIdx.x; k < lv.s; k += BLOCK) {
            const uint32_t r = (k + 1) * lv.d - 1;
            const uint32_t tag = (uint32_t)i0 + r;
            unsigned long long c;
            if (KIND == KIND_U64) {
                c = (int)r < v ? (unsigned long long)sm[S::CS::phys(r)] : pad64(lv.pad_base, i0 + r - len);
            } else {
                uint32_t key = 0xFFFFFFFFu;
                if ((int)r < v) key = (uint32_t)S::item_at(smem_raw, (int)r);
                c = ((unsigned long long)key << 32) | tag;
            }
            smp[k] = c;
        }
        __syncthreads();                     // shared memory is reused by the next sublist
        start = nstart;
        v = nv;
        vs = nvs;
    }
}

// ------------------------------------------------------------ Steps 2 + 3 on a CTA pair
// SURVEY NEXT-2 (the B200 reading of "n/m is the shared memory size"): a
// sublist of L = 2 tiles is sorted by a thread-block cluster of two CTAs.  Each CTA sorts
// its half on chip (CtaSort), then the last merge level crosses the pair through
// distributed shared memory: with a* = the number of half-0 items among the first TILE
// outputs (one merge-path split, found by a warp with 32-way probes of both halves),
// CTA 0 outputs merge(A[0, a*), B[0, b*)) and CTA 1 merge(A[a*, T), B[b*, T)), b* = T - a*.
// The two CTAs swap exactly b* items (CTA 0's A[a*, T) against CTA 1's B[0, b*), read
// once over DSMEM), so each then holds its two runs in its own shared memory and runs
// an ordinary uneven merge.  Samples (Step 3) at sublist positions (k+1)d - 1 come from
// the CTA that outputs them.  Keys only.
template <int BLOCK, int ITEMS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(BLOCK, 1) k_local_sort_pair(LevelDev lv)
{
    pdl_entry();
    namespace cg = cooperative_groups;
    using S = Seg<KIND_KEYS, BLOCK, ITEMS>;
    using CS = typename S::CS;
    using T = uint32_t;
    constexpr int H = CS::TILE;                         // items per CTA (half a sublist)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    __shared__ int s_astar;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const uint32_t ntiles = lv.tile_hi ? lv.tile_hi : lv.B * lv.m;
    const uint32_t ncl = gridDim.x / 2;
    T x[ITEMS];
    for (uint32_t tile = lv.tile_lo + blockIdx.x / 2; tile < ntiles; tile += ncl) {   // uniform in the pair
        uint64_t start = 0;
        int v = 0;
        sublist_of(lv, tile, start, v);
        const int vr = max(0, min(v - rank * H, H));
        if (threadIdx.x == 0 && tile + ncl < ntiles) {
            uint64_t ns;
            int nv;
            sublist_of(lv, tile + ncl, ns, nv);
            const int nr = max(0, min(nv - rank * H, H));
            if (nr > 0) prefetch_l2(reinterpret_cast<const T*>(lv.in) + ns + (uint64_t)rank * H, (size_t)nr * 4);
        }
        const int vs = S::load_regs(x, lv.in, nullptr, start + (uint64_t)rank * H, vr, smem_raw, lv.xf_in);
        CS::sort(x, sm, vs);                            // positions >= vr read as TMAX
        cluster.sync();                                 // both halves sorted and visible
        const T* peer = cluster.map_shared_rank(sm, rank ^ 1);
        if (threadIdx.x < 32) {
            const T* A = rank == 0 ? sm : peer;         // half 0's sorted tile
            const T* B = rank == 0 ? peer : sm;         // half 1's
            // a* = first i in [0, H) with A[i] > B[H-1-i] (H if none): the merge-path
            // split of diagonal H.  Invariant: the predicate is false below lo and true
            // from hi on; each round probes 32 evenly spaced points (2 DSMEM-or-local
            // reads per lane) and shrinks [lo, hi] 32-fold.
            const int lane = threadIdx.x;
            int lo = 0, hi = H;
            while (lo < hi) {
                const int step = (hi - lo + 31) / 32;
                const int i = lo + lane * step;
                const bool gt = i >= hi || A[CS::phys(i)] > B[CS::phys(H - 1 - i)];
                const unsigned m = __ballot_sync(0xffffffffu, gt);
                if (m == 0) {
                    lo = lo + 31 * step + 1;
                } else {
                    const int f = __ffs(m) - 1;
                    if (f == 0) hi = lo;
                    else {
                        hi = min(hi, lo + f * step);
                        lo = lo + (f - 1) * step + 1;
                    }
                }
            }
            if (lane == 0) s_astar = lo;
        }
        __syncthreads();
        const int astar = s_astar, bstar = H - astar;
        // swap b* items: CTA 0 fetches B[0, b*), CTA 1 fetches A[a*, H).  Item q + k BLOCK
        // sits at phys(q) + k (BLOCK + BLOCK/32): one base address, constant offsets.
        static_assert(BLOCK % 32 == 0 && CS::PAD == 5, "swap addressing assumes one pad per 32");
        constexpr int KSTEP = BLOCK + BLOCK / 32;
        {
            const int q = (int)threadIdx.x;
            const T* src = peer + CS::phys((rank == 0 ? 0 : astar) + q);
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) x[k] = q + k * BLOCK < bstar ? src[k * KSTEP] : T(0);
            cluster.sync();                             // every remote read done
            T* dst = sm + CS::phys((rank == 0 ? astar : 0) + q);
#pragma unroll
            for (int k = 0; k < ITEMS; ++k)
                if (q + k * BLOCK < bstar) dst[k * KSTEP] = x[k];
        }
        __syncthreads();
        // local runs: rank 0 [A[0,a*) | B[0,b*)], rank 1 [A[a*,H) | B[b*,H)]; A part first
        const int len1 = rank == 0 ? astar : bstar;
        CS::merge_two(x, sm, (int)threadIdx.x * ITEMS, len1);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) sm[CS::phys((int)threadIdx.x * ITEMS + k)] = x[k];
        __syncthreads();
        // (loading the next half into registers during the write-back, as k_local_sort
        // does, measured slower here: it spills)
        if (vr > 0) S::store(lv.srt, nullptr, start + (uint64_t)rank * H, vr, smem_raw);
        // Step 3: samples k whose position (k+1)d - 1 falls in this CTA's half
        const uint32_t i = tile % lv.m, b = tile / lv.m;
        const uint64_t i0 = (uint64_t)i * lv.L;
        u64* smp = lv.samples + ((uint64_t)b * lv.m + i) * lv.s;
        const uint32_t k0 = (uint32_t)rank * (lv.s / 2), k1 = k0 + lv.s / 2;
        for (uint32_t k = k0 + threadIdx.x; k < k1; k += BLOCK) {
            const uint32_t r = (k + 1) * lv.d - 1;
            const uint32_t key = (int)r < v ? sm[CS::phys((int)r - rank * H)] : 0xFFFFFFFFu;
            smp[k] = ((unsigned long long)key << 32) | (uint32_t)(i0 + r);
        }
        __syncthreads();                                // shared memory reused next sublist
    }
}

// ------------------------------------------------------------ Step 4 as a merge tree
// Step 4 sorts the m*s samples, and Step 5 reads s of them:
// g_k = sorted[(k+1)m - 1] (R2).  The samples arrive as m sorted runs of s
// (Step 3 takes them from sorted sublists), so sorting them is a merge of m runs.  For
// one problem whose samples stay L2-resident (R22): k_s4_tile merges the runs inside
// tiles of TILE_U64 on chip, k_s4_merge merges pairs of runs per launch (one CTA per
// output tile, the merge-path split found by a warp), and once two runs are left
// k_s4_select computes only the s order statistics Step 5 reads, each by one merge-path
// split: the d-th output of merge(A, B) is max(A[i-1], B[d-1-i]), i = split(d).

// Merge-path split of diagonal d in merge(A[0, na), B[0, nb)): the number of A items among
// the first d outputs (ties: A first).  One warp, 32 evenly spaced probes per round:
// P(i) = A[i] <= B[d-1-i] is true below the split and false from it on, so the ballot's
// popcount c narrows the interval to the c-th gap (log_32 of the range rounds, each one
// pair of L2 loads per lane).  All lanes return the split.
__device__ __forceinline__ uint32_t warp_split(const u64* A, uint32_t na, const u64* B, uint32_t nb, uint32_t d)
{
    const uint32_t lane = threadIdx.x & 31;
    uint32_t lo = d > nb ? d - nb : 0, hi = min(d, na);   // split in [lo, hi]
    while (lo < hi) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t p = lo + (lane + 1) * step - 1;
        const bool t = p < hi && A[p] <= B[d - 1 - p];
        const uint32_t c = __popc(__ballot_sync(0xffffffffu, t));
        hi = min(hi, lo + (c + 1) * step - 1);   // P false at probe c (when it exists)
        lo += c * step;                          // P true at probe c-1
    }
    return lo;
}

// Runs of R (a power of two, R >= ITEMS: merge levels only; R < ITEMS: full sort) merged
// inside tiles of TILE: src -> dst (may alias: a CTA reads its whole tile first).
template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK, 1) k_s4_tile(const u64* src, u64* dst, uint32_t N, uint32_t R)
{
    pdl_entry();
    using CS = CtaSort<unsigned long long, BLOCK, ITEMS>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned long long* sm = reinterpret_cast<unsigned long long*>(smem_raw);
    const uint64_t t0 = (uint64_t)blockIdx.x * CS::TILE;
    const int v = (int)umin64(CS::TILE, N - t0);
    unsigned long long x[ITEMS];
    if (R >= (uint32_t)ITEMS) {
        CS::sort_presorted(x, src + t0, sm, v, (int)R);
    } else {
        CS::load(x, src + t0, v);
        CS::sort(x, sm, v);
    }
    for (int p = threadIdx.x; p < v; p += BLOCK) dst[t0 + p] = sm[CS::phys(p)];
}

// One merge level: pairs of runs of R (run r = [rR, min((r+1)R, N)); an unpaired last run
// is copied through) -> runs of 2R.  CTA = TO consecutive outputs inside one pair; the
// splits of its first and last diagonals by two warps, both input ranges staged in
// shared memory, a merge-path merge of ITEMS outputs per thread, a padded transpose for
// coalesced stores.  Ties take A first (stable; the composites are distinct anyway).
#ifndef GBS_S4_MERGE_MINB
#define GBS_S4_MERGE_MINB 4   // CTAs per SM (registers): the whole level in one wave
#endif
template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK, GBS_S4_MERGE_MINB) k_s4_merge(const u64* src, u64* dst, uint32_t N, uint32_t R)
{
    pdl_entry();
    constexpr int TO = BLOCK * ITEMS;
    __shared__ u64 sm[TO + TO / ITEMS + ITEMS];
    __shared__ uint32_t s_split[2];
    const uint64_t o0 = (uint64_t)blockIdx.x * TO;
    if (o0 >= N) return;
    const uint64_t base = o0 / (2ull * R) * (2ull * R);
    const uint32_t na = (uint32_t)umin64(R, N - base);
    const uint32_t nb = (uint32_t)(N - base > R ? umin64(R, N - base - R) : 0);
    const u64* A = src + base;
    const u64* Bp = A + na;
    const uint32_t d0 = (uint32_t)(o0 - base), d1 = min(d0 + (uint32_t)TO, na + nb);
    const int warp = threadIdx.x >> 5;
    if (warp < 2) {
        const uint32_t sp = warp_split(A, na, Bp, nb, warp ? d1 : d0);
        if ((threadIdx.x & 31) == 0) s_split[warp] = sp;
    }
    __syncthreads();
    const uint32_t a0 = s_split[0], a1 = s_split[1];
    const int la = (int)(a1 - a0), lb = (int)((d1 - a1) - (d0 - a0)), tot = la + lb;
    const u64* As = A + a0;
    const u64* Bs = Bp + (d0 - a0);
    u64 out[ITEMS];
    // staging: all ITEMS loads of a thread in flight before the shared-memory stores
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        const int i = threadIdx.x + r * BLOCK;
        out[r] = i < la ? __ldg(As + i) : (i < tot ? __ldg(Bs + (i - la)) : 0ull);
    }
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
        const int i = threadIdx.x + r * BLOCK;
        if (i < tot) sm[i] = out[r];
    }
    __syncthreads();
    const int dg = threadIdx.x * ITEMS;
    if (dg < tot) {
        int lo = max(0, dg - lb), hi = min(dg, la);
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sm[mid] <= sm[la + dg - 1 - mid]) lo = mid + 1;
            else hi = mid;
        }
        // one shared-memory load per output: the head of the run just consumed; an
        // exhausted run reads as all-ones (never a composite: tags < 2^32 - 2^20)
        int i = lo, j = dg - lo;
        u64 a = i < la ? sm[i] : ~0ull, b = j < lb ? sm[la + j] : ~0ull;
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
            const bool t = a <= b;
            out[r] = t ? a : b;
            i += t ? 1 : 0;
            j += t ? 0 : 1;
            const bool ok = t ? i < la : j < lb;
            const u64 v = sm[ok ? (t ? i : la + j) : 0];
            a = t ? (ok ? v : ~0ull) : a;
            b = t ? b : (ok ? v : ~0ull);
        }
    }
    __syncthreads();
    if (dg < tot) {
#pragma unroll
        for (int r = 0; r < ITEMS; ++r) {
            const int o = dg + r;
            sm[o + o / ITEMS] = out[r];
        }
    }
    __syncthreads();
    u64* C = dst + o0;
    for (int o = threadIdx.x; o < tot; o += BLOCK) C[o] = sm[o + o / ITEMS];
}

// The last level, selection only: with runs A = src[0, R) and B = src[R, N) (N <= 2R),
// samples[(k+1)m - 1] = the ((k+1)m)-th smallest of A u B, one warp per k < s.
__global__ void k_s4_select(const u64* src, u64* samples, uint32_t N, uint32_t R, uint32_t m, uint32_t s)
{
    pdl_entry();
    const uint32_t k = (uint32_t)(((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (k >= s) return;   // warp-uniform
    const uint32_t d = (k + 1) * m;
    const uint32_t na = min(R, N), nb = N - na;
    const uint32_t i = warp_split(src, na, src + na, nb, d);
    u64 g = i > 0 ? src[i - 1] : 0ull;
    if (d > i) g = max(g, src[na + (d - i - 1)]);
    if ((threadIdx.x & 31) == 0) samples[(uint64_t)d - 1] = g;
}

// ------------------------------------------------------------ Step 5
// Global sampling: g_k = sorted_samples[(k+1)m - 1] (R2).
__global__ void k_global_samples(LevelDev lv)
{
    pdl_entry();
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
#ifndef GBS_IDX_CHUNK_KB
#define GBS_IDX_CHUNK_KB 64
#endif
static constexpr int IDX_CHUNK_BYTES = GBS_IDX_CHUNK_KB * 1024;

// --- TMA bulk copy + mbarrier helpers (sm_90+ PTX; SASS UBLKCP / SYNCS)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase)
{
    asm volatile("{\n\t.reg .pred p;\n\tLAB_WAIT:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra LAB_WAIT;\n\t}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

// Step 6, streaming form: persistent CTAs walk (sublist, 64 KB chunk) work items; one
// thread keeps the next chunk's TMA bulk copy in flight (double buffer) while all
// threads bisect the current one; per-splitter counts accumulate in registers.  A bulk
// copy needs 16-byte aligned addresses: a chunk that starts `lead` items past a 16-byte
// boundary (nested problems start at bucket offsets) is copied from that boundary and
// read at buffer + lead (the items copied before it are ignored; the last partial
// 16 bytes are loaded by the threads).
template <int KIND, int BLOCK, int MAXQ>
__global__ void __launch_bounds__(BLOCK, (GBS_IDX_CHUNK_KB <= 32 ? 2 : 1)) k_sample_index_tma(LevelDev lv)
{
    pdl_entry();
    using KT = typename std::conditional<KIND == KIND_U64, unsigned long long, uint32_t>::type;
    constexpr int CH = IDX_CHUNK_BYTES / sizeof(KT);
    constexpr int LEAD = 16 / sizeof(KT);            // room for a misaligned chunk start
    extern __shared__ __align__(16) unsigned char smem_raw[];
    KT* buf0 = reinterpret_cast<KT*>(smem_raw);
    KT* buf1 = buf0 + CH + LEAD;
    unsigned long long* gs = reinterpret_cast<unsigned long long*>(buf1 + CH + LEAD);
    uint32_t* Q = reinterpret_cast<uint32_t*>(gs + lv.s);
    __shared__ __align__(8) unsigned long long bars[2];

    const uint32_t ntiles = lv.B * lv.m;
    // chunks of tile t: ceil(v / CH); work items in order (tile, chunk)
    auto tile_v = [&](uint32_t t) -> int {
        const uint32_t b = t / lv.m, i = t % lv.m;
        const uint32_t len = lv.pr.length(b);
        const uint64_t i0 = (uint64_t)i * lv.L;
        return len > i0 ? (int)umin64(len - i0, lv.L) : 0;
    };
    // first item of work item (tile t, chunk c) in HBM
    auto chunk_src = [&](uint32_t t, int c) -> const KT* {
        return reinterpret_cast<const KT*>(lv.srt) + lv.pr.offset(t / lv.m) + (uint64_t)(t % lv.m) * lv.L +
               (uint64_t)c * CH;
    };
    auto lead_of = [&](const KT* src) -> int { return (int)(((uintptr_t)src & 15) / sizeof(KT)); };
    auto issue = [&](uint32_t t, int c, int slot) {   // thread 0 only
        const int v = tile_v(t);
        const int cl = min(CH, v - c * CH);
        const KT* src = chunk_src(t, c);
        const int ld = lead_of(src);
        const unsigned bytes = (unsigned)((size_t)(ld + cl) * sizeof(KT)) & ~15u;
        unsigned long long* bar = &bars[slot];
        mbar_expect_tx(bar, bytes);
        if (bytes) tma_load_1d(slot ? buf1 : buf0, src - ld, bytes, bar);
    };
    if (threadIdx.x == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    uint32_t tile = blockIdx.x;
    // first work item: skip empty tiles
    while (tile < ntiles && tile_v(tile) == 0) {
        // an empty sublist still owns a row of zeros
        uint32_t* arow = lv.a + (uint64_t)tile * lv.s;
        for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) arow[j] = 0;
        tile += gridDim.x;
    }
    if (tile >= ntiles) return;
    int chunk = 0;
    if (threadIdx.x == 0) issue(tile, 0, 0);
    uint32_t loaded_b = 0xFFFFFFFFu;
    uint32_t q[MAXQ];
#pragma unroll
    for (int k = 0; k < MAXQ; ++k) q[k] = 0;
    unsigned phase = 0;   // bit k: parity of the next completion of bars[k]
    int slot = 0;
    while (true) {
        const uint32_t b = tile / lv.m, i = tile % lv.m;
        const int v = tile_v(tile);
        const int nch = (v + CH - 1) / CH;
        const uint64_t i0 = (uint64_t)i * lv.L;
        // next work item (same tile's next chunk, else the next non-empty tile)
        uint32_t ntile = tile;
        int nchunk = chunk + 1;
        if (nchunk >= nch) {
            nchunk = 0;
            ntile = tile + gridDim.x;
            while (ntile < ntiles && tile_v(ntile) == 0) ntile += gridDim.x;   // rows zeroed below
        }
        if (threadIdx.x == 0 && ntile < ntiles) issue(ntile, nchunk, slot ^ 1);
        if (b != loaded_b) {          // splitters of problem b (Step 5 fused)
            const u64* srt = lv.samples + (uint64_t)b * lv.m * lv.s;
            for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) {
                const u64 gj = srt[(uint64_t)(j + 1) * lv.m - 1];
                gs[j] = gj;
                if (i == 0) lv.splitters[(uint64_t)b * lv.s + j] = gj;
            }
            loaded_b = b;
        }
        const KT* csrc = chunk_src(tile, chunk);
        const int ld = lead_of(csrc);
        KT* ks = (slot ? buf1 : buf0) + ld;
        mbar_wait(&bars[slot], (phase >> slot) & 1u);
        phase ^= 1u << slot;
        const int c0 = chunk * CH;
        const int cl = min(CH, v - c0);
        {   // keys past the last 16-byte boundary of the chunk (tail of the sublist)
            const int full = (int)(((unsigned)((size_t)(ld + cl) * sizeof(KT)) & ~15u) / sizeof(KT)) - ld;
            for (int p = max(full, 0) + threadIdx.x; p < cl; p += BLOCK) ks[p] = csrc[p];
        }
        __syncthreads();
        auto rank_key = [&](int p) -> unsigned long long {
            if (KIND == KIND_U64) return (unsigned long long)ks[p];
            return ((unsigned long long)ks[p] << 32) | (uint32_t)(i0 + c0 + p);
        };
        const unsigned long long first = rank_key(0), last = rank_key(cl - 1);
#pragma unroll
        for (int k = 0; k < MAXQ; ++k) {
            const uint32_t j = threadIdx.x + k * BLOCK;
            if (j < lv.s) {
                const unsigned long long gj = gs[j];
                int lo = 0, hi = cl;
                if (gj < first) hi = 0;
                else if (gj >= last) lo = cl;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (rank_key(mid) <= gj) lo = mid + 1; else hi = mid;
                }
                q[k] += (uint32_t)lo;
            }
        }
        if (chunk + 1 >= nch) {       // sublist done: a_ij = Q_ij - Q_i,j-1
#pragma unroll
            for (int k = 0; k < MAXQ; ++k) {
                const uint32_t j = threadIdx.x + k * BLOCK;
                if (j < lv.s) Q[j] = q[k];
                q[k] = 0;
            }
            __syncthreads();
            uint32_t* arow = lv.a + ((uint64_t)b * lv.m + i) * lv.s;
            for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) arow[j] = Q[j] - (j ? Q[j - 1] : 0u);
            if (lv.pex) {             // fused Step 8+9: run (i, j) starts at P_i,j-1
                uint32_t* prow = lv.pex + ((uint64_t)b * lv.m + i) * lv.s;
                for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) prow[j] = j ? Q[j - 1] : 0u;
            }
            // empty sublists skipped on the way to the next tile get rows of zeros
            for (uint32_t t2 = tile + gridDim.x; t2 < ntile && t2 < ntiles; t2 += gridDim.x) {
                uint32_t* zrow = lv.a + (uint64_t)t2 * lv.s;
                for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) zrow[j] = 0;
            }
        }
        __syncthreads();              // buffer `slot` free; Q / gs reusable
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (ntile >= ntiles) break;
        tile = ntile;
        chunk = nchunk;
        slot ^= 1;
    }
}

template <int KIND, int BLOCK>
__global__ void __launch_bounds__(BLOCK, 2) k_sample_index(LevelDev lv)
{
    pdl_entry();
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

    const KT* src = reinterpret_cast<const KT*>(lv.srt) + off + i0;
    if (threadIdx.x == 0 && blockIdx.x + lv.pf_stride < lv.B * lv.m) {
        uint64_t ps;
        int pv;
        sublist_of(lv, blockIdx.x + lv.pf_stride, ps, pv);
        prefetch_l2(reinterpret_cast<const KT*>(lv.srt) + ps, (size_t)pv * sizeof(KT));
    }
    // Step 5 fused into the prologue (the paper loads the s global samples into shared
    // memory here): g_j = sorted_samples[(j+1)m - 1]; sublist 0 of each
    // problem also records them (the splitters array, for stage parity).
    const u64* srt = lv.samples + (uint64_t)b * lv.m * lv.s;
    for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) {
        const u64 gj = srt[(uint64_t)(j + 1) * lv.m - 1];
        gs[j] = gj;
        Q[j] = 0;
        if (i == 0) lv.splitters[(uint64_t)b * lv.s + j] = gj;
    }
    // The sublist is searched in chunks of IDX_CHUNK bytes (64 KB) so the CTA fits
    // twice per SM: one CTA's chunk load overlaps the other's bisections.  The
    // count over the sublist is the sum of the counts over its sorted chunks.
    constexpr int CH = IDX_CHUNK_BYTES / sizeof(KT);
    for (int c0 = 0; c0 < v; c0 += CH) {
        const int cl = min(CH, v - c0);
        stage_to_smem<BLOCK>(ks, src + c0, (size_t)cl * sizeof(KT));
        __syncthreads();
        auto rank_key = [&](int q) -> unsigned long long {
            if (KIND == KIND_U64) return (unsigned long long)ks[q];
            return ((unsigned long long)ks[q] << 32) | (uint32_t)(i0 + c0 + q);
        };
        const unsigned long long first = rank_key(0), last = rank_key(cl - 1);
        for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) {
            const unsigned long long gj = gs[j];
            int lo = 0, hi = cl;
            if (gj < first) hi = 0;                       // whole chunk above g_j
            else if (gj >= last) lo = cl;                 // whole chunk at or below g_j
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                unsigned long long rk;
                if (KIND == KIND_U64) rk = (unsigned long long)ks[mid];
                else rk = ((unsigned long long)ks[mid] << 32) | (uint32_t)(i0 + c0 + mid);
                if (rk <= gj) lo = mid + 1; else hi = mid;
            }
            Q[j] += (uint32_t)lo;
        }
        __syncthreads();
    }
    __syncthreads();   // Q complete (also when v == 0 and the chunk loop never ran)
    uint32_t* arow = lv.a + ((uint64_t)b * lv.m + i) * lv.s;
    for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) arow[j] = Q[j] - (j ? Q[j - 1] : 0u);
    if (lv.pex) {                     // fused Step 8+9: run (i, j) starts at P_i,j-1
        uint32_t* prow = lv.pex + ((uint64_t)b * lv.m + i) * lv.s;
        for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) prow[j] = j ? Q[j - 1] : 0u;
    }
}

// ------------------------------------------------------------ Step 7
// Prefix sum: l = exclusive scan of a in the order
// a_11..a_m1, a_12, ... (column-major, R5) over row-major storage.  One CTA per block
// of 32 columns: pass 1 column sums (the paper's "parallel column sum"), one
// decoupled look-back across column blocks replaces the single-SM scan of column
// sums, pass 2 writes l (the paper's "final update").  Integer sums: deterministic.
#ifndef GBS_SCAN_BLOCK
#define GBS_SCAN_BLOCK 1024
#endif
static constexpr int SCAN_BLOCK = GBS_SCAN_BLOCK;
static constexpr unsigned long long LB_AGG = 1ull << 62, LB_INC = 2ull << 62, LB_VAL = (1ull << 62) - 1;

__global__ void __launch_bounds__(SCAN_BLOCK) k_scan(LevelDev lv)
{
    pdl_entry();
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

    uint32_t sum = 0, mx = 0;
    if (col_ok) {
        uint64_t r = r0;
        for (; r + 8 <= r1; r += 8) {           // 8 independent loads in flight
            uint32_t x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = A[(r + u) * lv.s + c];
#pragma unroll
            for (int u = 0; u < 8; ++u) { sum += x[u]; mx = max(mx, x[u]); }
        }
        for (; r < r1; ++r) { const uint32_t x = A[r * lv.s + c]; sum += x; mx = max(mx, x); }
    }
    if (lv.maxrun) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0 && mx) atomicMax(lv.maxrun, mx);
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
        uint64_t r = r0;
        for (; r + 8 <= r1; r += 8) {           // 8 independent loads in flight
            uint32_t x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) x[u] = A[(r + u) * lv.s + c];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                Lo[(r + u) * lv.s + c] = run;
                run += x[u];
            }
        }
        for (; r < r1; ++r) {
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

// A u16 bucket map (bucket of every position) keeps the CTA at ~100 KB of shared
// memory, so two CTAs share an SM and one's loads overlap the other's map build.
template <int KIND, int BLOCK, int MAXPER>
__global__ void __launch_bounds__(BLOCK, 2) k_relocate(LevelDev lv)
{
    pdl_entry();
    if (lv.maxrun && *lv.maxrun <= GBS_GROUP_MAX_RUN) return;   // short runs: k_relocate_grouped did it
    using KT = typename std::conditional<KIND == KIND_U64, unsigned long long, uint32_t>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint32_t* starts = reinterpret_cast<uint32_t*>(smem_raw);
    uint32_t* delta = starts + lv.s;
    uint16_t* bmap = reinterpret_cast<uint16_t*>(delta + lv.s);   // L + 2L/per + 2 entries
    __shared__ uint32_t wtmp[32];

    const uint32_t b = blockIdx.x / lv.m, i = blockIdx.x % lv.m;
    const uint64_t off = lv.pr.offset(b);
    const uint32_t len = lv.pr.length(b);
    const uint64_t i0 = (uint64_t)i * lv.L;
    const int v = len > i0 ? (int)umin64(len - i0, lv.L) : 0;
    if (v == 0) return;

    // prefetch the sublist (striped: r = t + k*BLOCK) -- latency overlaps the map build
    const KT* src = reinterpret_cast<const KT*>(lv.srt) + off + i0;
    if (threadIdx.x == 0 && blockIdx.x + lv.pf_stride < lv.B * lv.m) {
        uint64_t ps;
        int pv;
        sublist_of(lv, blockIdx.x + lv.pf_stride, ps, pv);
        prefetch_l2(reinterpret_cast<const KT*>(lv.srt) + ps, (size_t)pv * sizeof(KT));
        if (KIND == KIND_PAIRS) prefetch_l2(lv.srt_v + ps, (size_t)pv * 4);
    }

    // the first batch of keys is loaded now; its latency overlaps the map build
    constexpr int U = 8;
    KT y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int r = threadIdx.x + u * BLOCK;
        y[u] = r < v ? src[r] : KT(0);
    }

    const uint64_t row = ((uint64_t)b * lv.m + i) * lv.s;
    for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) starts[j] = lv.a[row + j];
    __syncthreads();
    block_excl_scan<BLOCK>(starts, (int)lv.s, wtmp);
    for (uint32_t j = threadIdx.x; j < lv.s; j += BLOCK) delta[j] = lv.l[row + j] - starts[j];
    __syncthreads();

    // bucket map: thread t walks positions [t*per, t*per + per) (blocked), keeping the
    // next bucket start in a register; the map entry of r lives at r + 2 r/per (u16
    // units: each thread's row is 33 words, so the blocked writes are conflict free)
    const int S = (int)lv.s;
    const int per = (int)(lv.L / BLOCK) > 0 ? (int)(lv.L / BLOCK) : 1;   // power of two
    const int lp = 31 - __clz(per);
    const int r0 = threadIdx.x * per, r1 = min(v, r0 + per);
    if (r0 < r1) {
        int j = upper_bound_u32(starts, 0, S, (uint32_t)r0) - 1;
        uint32_t nxt = j + 1 < S ? starts[j + 1] : 0xFFFFFFFFu;
        for (int r = r0; r < r1; ++r) {
            while ((uint32_t)r >= nxt) {          // crossed a bucket boundary (rare)
                ++j;
                nxt = j + 1 < S ? starts[j + 1] : 0xFFFFFFFFu;
            }
            bmap[r + 2 * (r >> lp)] = (uint16_t)j;
        }
    }
    __syncthreads();
    // position-ordered copy, software-pipelined: batch k+1 is loaded before batch k is
    // stored, so one batch of loads is always in flight (the compiler cannot reorder the
    // loads above the stores itself: src and dst may alias as far as it knows)
    KT* dst = reinterpret_cast<KT*>(lv.reloc) + off;
    for (int q0 = threadIdx.x; q0 < v; q0 += U * BLOCK) {
        KT z[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = q0 + (U + u) * BLOCK;
            z[u] = r < v ? src[r] : KT(0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = q0 + u * BLOCK;
            if (r < v) dst[(uint32_t)r + delta[bmap[r + 2 * (r >> lp)]]] = y[u];
            y[u] = z[u];
        }
    }
    if (KIND == KIND_PAIRS) {
        const uint32_t* sv = lv.srt_v + off + i0;
        uint32_t* dv = lv.reloc_v + off;
        uint32_t w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = threadIdx.x + u * BLOCK;
            w[u] = r < v ? sv[r] : 0u;
        }
        for (int q0 = threadIdx.x; q0 < v; q0 += U * BLOCK) {
            uint32_t z[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int r = q0 + (U + u) * BLOCK;
                z[u] = r < v ? sv[r] : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int r = q0 + u * BLOCK;
                if (r < v) dv[(uint32_t)r + delta[bmap[r + 2 * (r >> lp)]]] = w[u];
                w[u] = z[u];
            }
        }
    }
}

// ------------------------------------------------------------ Step 9 (+ leaves)
// Sublist sort: one CTA per bucket B_j = R[l_0j, l_0j+|B_j|),
// |B_j| <= the tight bound <= tile capacity (checked by the planner).  MODE_LEAF:
// one CTA per whole problem (len_b <= tile).
enum SegMode { MODE_BUCKET = 0, MODE_LEAF = 1, MODE_GATHER = 2 };   // GATHER: fused Step 8+9

// Segment idx of a Step-9 / leaf launch: element offset and length.
template <int MODE>
__device__ __forceinline__ void segment_of(const LevelDev& lv, uint32_t idx, uint64_t& off, int& v)
{
    if (MODE == MODE_LEAF) {
        off = lv.pr.offset(idx);
        v = (int)lv.pr.length(idx);
    } else {
        const uint32_t b = idx / lv.s, j = idx % lv.s;
        const uint32_t* l0 = lv.l + (uint64_t)b * lv.m * lv.s;   // row 0 of problem b
        const uint32_t st = l0[j];
        const uint32_t en = j + 1 < lv.s ? l0[j + 1] : lv.pr.length(b);
        off = lv.pr.offset(b) + st;
        v = (int)(en - st);
    }
}

// Step 8, grouped by destination: a CTA per (group of G consecutive sublists, range of
// JB buckets); a warp per bucket j copies the G runs (i, j) of its group, which are
// adjacent in R (l_{i+1,j} = l_ij + a_ij, R5), as ONE contiguous destination chunk of
// ~G d items.  Relocating sublist by sublist writes runs of ~d items at arbitrary
// alignment whose partial 32-byte sectors each cost HBM a read-modify-write (measured:
// DRAM reads 1.5x the algorithmic bytes at d = 16).  The run starts P_i,j-1 come from
// Step 6 (lv.pex), so no row scan is needed and the grid is fine-grained.  Same R as
// k_relocate, bit for bit.
template <int KIND, int BLOCK, int G, int JB>
__global__ void __launch_bounds__(BLOCK) k_relocate_grouped(LevelDev lv)
{
    pdl_entry();
    if (lv.maxrun && *lv.maxrun > GBS_GROUP_MAX_RUN) return;    // long runs: k_relocate does it
    using KT = typename std::conditional<KIND == KIND_U64, unsigned long long, uint32_t>::type;
    __shared__ uint32_t sa[G][JB], sp[G][JB], sl[JB];
    const uint32_t S = lv.s;
    const uint32_t ng = (lv.m + G - 1) / G, nj = (S + JB - 1) / JB;
    const uint32_t jb = blockIdx.x % nj, rest = blockIdx.x / nj;
    const uint32_t b = rest / ng, i0 = (rest % ng) * G;
    const uint32_t j0 = jb * JB, jn = min((uint32_t)JB, S - j0);
    const int gn = (int)min((uint32_t)G, lv.m - i0);
    const uint64_t row0 = ((uint64_t)b * lv.m + i0) * S + j0;
    for (uint32_t t = threadIdx.x; t < (uint32_t)G * JB; t += BLOCK) {
        const uint32_t r = t / JB, j = t % JB;
        const bool ok = (int)r < gn && j < jn;
        sa[r][j] = ok ? lv.a[row0 + (uint64_t)r * S + j] : 0u;
        sp[r][j] = ok ? lv.pex[row0 + (uint64_t)r * S + j] : 0u;
    }
    for (uint32_t j = threadIdx.x; j < jn; j += BLOCK) sl[j] = lv.l[row0 + j];
    __syncthreads();
    const uint64_t off = lv.pr.offset(b);
    const KT* src = reinterpret_cast<const KT*>(lv.srt) + off;
    KT* dst = reinterpret_cast<KT*>(lv.reloc) + off;
    const int lane = threadIdx.x & 31;
    for (uint32_t j = threadIdx.x >> 5; j < jn; j += BLOCK / 32) {
        // run r covers chunk positions [pre[r], pre[r+1]); position e of run r is problem
        // item dl[r] + e (dl[r] = run start - pre[r], precomputed once per bucket)
        uint32_t pre[G + 1], dl[G];
        pre[0] = 0;
#pragma unroll
        for (int r = 0; r < G; ++r) {
            dl[r] = (uint32_t)(i0 + r) * lv.L + sp[r][j] - pre[r];
            pre[r + 1] = pre[r] + sa[r][j];
        }
        const uint32_t total = pre[G], d0 = sl[j];
        for (uint32_t e0 = 0; e0 < total; e0 += 128) {                  // 4 loads in flight per lane
            KT y[4];
            uint32_t q[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t e = e0 + u * 32 + lane;
                uint32_t base = dl[0];
#pragma unroll
                for (int k = 1; k < G; ++k)
                    if (e >= pre[k]) base = dl[k];
                q[u] = base + e;
                if (e < total) y[u] = src[q[u]];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t e = e0 + u * 32 + lane;
                if (e < total) dst[d0 + e] = y[u];
            }
            if (KIND == KIND_PAIRS) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t e = e0 + u * 32 + lane;
                    if (e < total) lv.reloc_v[off + d0 + e] = lv.srt_v[off + q[u]];
                }
            }
        }
    }
}

// Step 9 size tiers: bucket idx goes to list t (0: 0 < v <= cut0, 1: cut0 < v <= cut1,
// 2: v > cut1); empty buckets are dropped.  Each 256-bucket block appends its buckets in
// index order (ballot compaction; one atomic per tier and block), so neighbouring CTAs
// of a tier read neighbouring runs.  The output never depends on the list order: each
// bucket is sorted on its own.
__global__ void __launch_bounds__(256) k_bucket_tiers(LevelDev lv, uint32_t* lists, uint32_t* lens, uint32_t cut0,
                                                      uint32_t cut1, uint32_t cut2)
{
    pdl_entry();
    constexpr int NT = 4;   // tiers: (0, cut0], (cut0, cut1], (cut1, cut2], > cut2
    __shared__ uint32_t wcnt[NT][8], wbase[NT][8];
    const uint32_t count = lv.B * lv.s;
    const uint32_t idx = blockIdx.x * 256 + threadIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int t = -1;
    if (idx < count) {
        uint64_t off;
        int v;
        segment_of<MODE_BUCKET>(lv, idx, off, v);
        const uint32_t u = (uint32_t)v;
        if (v > 0) t = u <= cut0 ? 0 : (u <= cut1 ? 1 : (u <= cut2 ? 2 : 3));
    }
    uint32_t mine = 0;
#pragma unroll
    for (int q = 0; q < NT; ++q) {
        const uint32_t mask = __ballot_sync(0xffffffffu, t == q);
        if (lane == 0) wcnt[q][w] = __popc(mask);
        if (t == q) mine = __popc(mask & ((1u << lane) - 1u));
    }
    __syncthreads();
    if (threadIdx.x < NT) {
        const int q = threadIdx.x;
        uint32_t tot = 0;
        for (int k = 0; k < 8; ++k) { wbase[q][k] = tot; tot += wcnt[q][k]; }
        const uint32_t base = tot ? atomicAdd(lens + q, tot) : 0u;
        for (int k = 0; k < 8; ++k) wbase[q][k] += base;
    }
    __syncthreads();
    if (t >= 0) lists[(uint64_t)t * count + wbase[t][w] + mine] = idx;
}

// Fused Step 8+9: lrel / pex staging area behind the CTA's largest tile
template <int KIND, int BLOCK, int ITEMS>
__host__ __device__ constexpr size_t gather_smem_offset()
{
    return (Seg<KIND, BLOCK, ITEMS>::smem_bytes() + 15) / 16 * 16;
}
// most sublists per problem the fused path stages (the plan falls back to Step 8 above)
__host__ __device__ constexpr uint32_t gather_max_m(int kind) { return kind == KIND_KEYS ? 2048u : 1024u; }

// Fused Step 8+9 for bucket idx: stage its run table (from l and P_i,j-1) in shared
// memory behind the tile, gather, sort, store.  `bounded`: a launch over every bucket
// that skips those outside [seg_min, seg_max).
template <int KIND, int BLOCK, int ITEMS, typename A>
__device__ __forceinline__ void sort_gathered(const LevelDev& lv, uint32_t idx, unsigned char* smem_raw, bool bounded)
{
    using KeyT = typename A::S::KeyT;
    uint64_t off;
    int v;
    segment_of<MODE_BUCKET>(lv, idx, off, v);
    if (v <= 0 || (bounded && ((uint32_t)v <= lv.seg_min || (uint32_t)v > lv.seg_max))) return;
    // (an L2 prefetch of the next wave's runs measured no gain here)
    const uint32_t b = idx / lv.s, j = idx % lv.s;
    uint2* run = reinterpret_cast<uint2*>(smem_raw + gather_smem_offset<KIND, BLOCK, ITEMS>());
    const uint64_t col0 = (uint64_t)b * lv.m * lv.s + j;          // (row 0, column j) of problem b
    const uint32_t l0 = lv.l[col0];
    for (uint32_t i = threadIdx.x; i < lv.m; i += BLOCK) {
        const uint32_t lr = lv.l[col0 + (uint64_t)i * lv.s] - l0;
        run[i] = make_uint2(lr, i * lv.L + lv.pex[col0 + (uint64_t)i * lv.s] - lr);
    }
    if (threadIdx.x == 0) run[lv.m] = make_uint2((uint32_t)v, 0u);
    __syncthreads();
    const uint64_t pb = lv.pr.offset(b);
    GatherSrc g{reinterpret_cast<const KeyT*>(lv.srt) + pb, KIND == KIND_PAIRS ? lv.srt_v + pb : nullptr, run,
                (int)lv.m};
    A::run_gather(g, v, lv.out, lv.out_v, off, smem_raw, lv.xf_out);
}

// One CTA per segment (bucket or leaf problem), adaptive tile size.  The segment
// pf_stride ahead (the next wave) is prefetched into L2.  (A persistent variant that
// walked segments with a work counter and register prefetch measured ~8% slower: the
// shared register array across tile sizes costs more than the hidden load latency.)
template <int KIND, int BLOCK, int ITEMS, int MODE>
__global__ void __launch_bounds__(BLOCK, (BLOCK <= 576 ? 2 : 1)) k_segment_sort(LevelDev lv)
{
    pdl_entry();
    // the mid tier (ITEMS not a power of two) only sees sizes just above the small tier
    using A = Adapt<KIND, BLOCK, ITEMS, ((ITEMS & (ITEMS - 1)) == 0 ? GBS_ADAPT_DEPTH : 0)>;
    using KeyT = typename A::S::KeyT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if constexpr (MODE == MODE_GATHER) {
        uint32_t idx = blockIdx.x;
        if (lv.tier_list) {
            if (blockIdx.x >= *lv.tier_len) return;
            idx = lv.tier_list[blockIdx.x];
        }
        sort_gathered<KIND, BLOCK, ITEMS, A>(lv, idx, smem_raw, !lv.tier_list);
        return;
    }
    const void* src = MODE == MODE_LEAF ? lv.in : lv.reloc;
    const uint32_t* src_v = MODE == MODE_LEAF ? lv.in_v : lv.reloc_v;
    if (lv.tier_list) {
        // one size tier: CTA q sorts the q-th bucket of the tier's list (k_bucket_tiers);
        // the CTAs past the list's length exit at once -- they are the grid's tail, so
        // the hardware block scheduler still balances the real buckets over the SMs
        const uint32_t len = *lv.tier_len;
        if (blockIdx.x >= len) return;
        if (threadIdx.x == 0 && blockIdx.x + lv.pf_stride < len) {
            uint64_t po;
            int pv;
            segment_of<MODE>(lv, lv.tier_list[blockIdx.x + lv.pf_stride], po, pv);
            prefetch_l2(reinterpret_cast<const KeyT*>(src) + po, (size_t)pv * sizeof(KeyT));
            if (KIND == KIND_PAIRS) prefetch_l2(src_v + po, (size_t)pv * 4);
        }
        uint64_t off;
        int v;
        segment_of<MODE>(lv, lv.tier_list[blockIdx.x], off, v);
        A::run(src, src_v, off, v, lv.out, lv.out_v, smem_raw, MODE == MODE_LEAF ? lv.xf_in : 0, lv.xf_out);
        return;
    }
    const uint32_t count = MODE == MODE_LEAF ? lv.B : lv.B * lv.s;
    const uint32_t seg_end = lv.seg_hi ? lv.seg_hi : count;
    if (threadIdx.x == 0 && lv.seg_lo + blockIdx.x + lv.pf_stride < seg_end) {
        uint64_t po;
        int pv;
        segment_of<MODE>(lv, lv.seg_lo + blockIdx.x + lv.pf_stride, po, pv);
        if (pv > 0 && (uint32_t)pv > lv.seg_min && (uint32_t)pv <= lv.seg_max) {   // this launch's
            prefetch_l2(reinterpret_cast<const KeyT*>(src) + po, (size_t)pv * sizeof(KeyT));
            if (KIND == KIND_PAIRS) prefetch_l2(src_v + po, (size_t)pv * 4);
        }
    }
    uint64_t off;
    int v;
    segment_of<MODE>(lv, lv.seg_lo + blockIdx.x, off, v);
    if (v <= 0 || (uint32_t)v <= lv.seg_min || (uint32_t)v > lv.seg_max) return;
    A::run(src, src_v, off, v, lv.out, lv.out_v, smem_raw, MODE == MODE_LEAF ? lv.xf_in : 0, lv.xf_out);
}

// The sparse size tiers of Step 9 (the full tile; in nested levels, whose buckets
// average a quarter of the bound, the mid tier too) on persistent CTAs walking the
// tier's list: a sparse tier then costs one wave of CTAs instead of one CTA per bucket
// slot (C4 level 2: 262,144 slots of a 165 KB CTA took 4.9 ms for an almost empty tier).
// Relocated buckets (MODE_BUCKET) or gathered ones (MODE_GATHER, fused Step 8+9).
template <int KIND, int BLOCK, int ITEMS, int MODE = MODE_BUCKET>
__global__ void __launch_bounds__(BLOCK, (BLOCK <= 576 ? 2 : 1)) k_segment_sort_rare(LevelDev lv)
{
    pdl_entry();
    using A = Adapt<KIND, BLOCK, ITEMS, ((ITEMS & (ITEMS - 1)) == 0 || KIND == KIND_KEYS ? GBS_ADAPT_DEPTH : 0)>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t len = *lv.tier_len;
    for (uint32_t q = blockIdx.x; q < len; q += gridDim.x) {
        if (q != blockIdx.x) __syncthreads();   // shared memory reused
        if constexpr (MODE == MODE_GATHER) {
            sort_gathered<KIND, BLOCK, ITEMS, A>(lv, lv.tier_list[q], smem_raw, false);
        } else {
            uint64_t off;
            int v;
            segment_of<MODE_BUCKET>(lv, lv.tier_list[q], off, v);
            A::run(lv.reloc, lv.reloc_v, off, v, lv.out, lv.out_v, smem_raw, 0, lv.xf_out);
        }
    }
}

// ------------------------------------------------------------ Step 9 on a CTA pair
// SURVEY NEXT-2 for buckets: a bucket of up to 2 tiles (Step 9) sorted by a
// cluster of two CTAs exactly as k_local_sort_pair sorts a two-tile sublist (each CTA
// sorts half on chip, one merge-path split of the halves over DSMEM, swap, uneven local
// merge), reading the relocated bucket and writing the final output.  Used when one-tile
// buckets would need a nested level.  Keys only.
template <int BLOCK, int ITEMS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(BLOCK, 1) k_segment_sort_pair(LevelDev lv)
{
    pdl_entry();
    namespace cg = cooperative_groups;
    using S = Seg<KIND_KEYS, BLOCK, ITEMS>;
    using CS = typename S::CS;
    using T = uint32_t;
    constexpr int H = CS::TILE;                         // items per CTA (half a bucket)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    __shared__ int s_astar;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    // all buckets [seg_lo, seg_hi) of the level, or a size tier's list (k_bucket_tiers)
    const uint32_t count = lv.tier_list ? *lv.tier_len : (lv.seg_hi ? lv.seg_hi : lv.B * lv.s);
    const uint32_t q0 = lv.tier_list ? 0u : lv.seg_lo;
    auto seg = [&](uint32_t q) { return lv.tier_list ? lv.tier_list[q] : q; };
    const uint32_t ncl = gridDim.x / 2;
    T x[ITEMS];
    for (uint32_t q = q0 + blockIdx.x / 2; q < count; q += ncl) {   // uniform in the pair
        uint64_t off;
        int v;
        segment_of<MODE_BUCKET>(lv, seg(q), off, v);
        if (v <= 0) continue;                           // both CTAs skip
        const int vr = max(0, min(v - rank * H, H));
        if (threadIdx.x == 0 && q + ncl < count) {
            uint64_t no;
            int nv;
            segment_of<MODE_BUCKET>(lv, seg(q + ncl), no, nv);
            const int nr = max(0, min(nv - rank * H, H));
            if (nr > 0) prefetch_l2(reinterpret_cast<const T*>(lv.reloc) + no + (uint64_t)rank * H, (size_t)nr * 4);
        }
        const int vs = S::load_regs(x, lv.reloc, nullptr, off + (uint64_t)rank * H, vr, smem_raw);
        CS::sort(x, sm, vs);
        cluster.sync();                                 // both halves sorted and visible
        const T* peer = cluster.map_shared_rank(sm, rank ^ 1);
        if (threadIdx.x < 32) {                         // a* = merge-path split of diagonal H
            const T* A = rank == 0 ? sm : peer;
            const T* B = rank == 0 ? peer : sm;
            const int lane = threadIdx.x;
            int lo = 0, hi = H;
            while (lo < hi) {
                const int step = (hi - lo + 31) / 32;
                const int i = lo + lane * step;
                const bool gt = i >= hi || A[CS::phys(i)] > B[CS::phys(H - 1 - i)];
                const unsigned m = __ballot_sync(0xffffffffu, gt);
                if (m == 0) {
                    lo = lo + 31 * step + 1;
                } else {
                    const int f = __ffs(m) - 1;
                    if (f == 0) hi = lo;
                    else {
                        hi = min(hi, lo + f * step);
                        lo = lo + (f - 1) * step + 1;
                    }
                }
            }
            if (lane == 0) s_astar = lo;
        }
        __syncthreads();
        const int astar = s_astar, bstar = H - astar;
        static_assert(BLOCK % 32 == 0 && CS::PAD == 5, "swap addressing assumes one pad per 32");
        constexpr int KSTEP = BLOCK + BLOCK / 32;
        {
            const int t = (int)threadIdx.x;
            const T* src = peer + CS::phys((rank == 0 ? 0 : astar) + t);
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) x[k] = t + k * BLOCK < bstar ? src[k * KSTEP] : T(0);
            cluster.sync();                             // every remote read done
            T* dst = sm + CS::phys((rank == 0 ? astar : 0) + t);
#pragma unroll
            for (int k = 0; k < ITEMS; ++k)
                if (t + k * BLOCK < bstar) dst[k * KSTEP] = x[k];
        }
        __syncthreads();
        CS::merge_two(x, sm, (int)threadIdx.x * ITEMS, rank == 0 ? astar : bstar);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) sm[CS::phys((int)threadIdx.x * ITEMS + k)] = x[k];
        __syncthreads();
        if (vr > 0) S::store(lv.out, nullptr, off + (uint64_t)rank * H, vr, smem_raw, lv.xf_out);
        __syncthreads();                                // shared memory reused next bucket
    }
}

// 64-bit keys (gbs_sort_keys64 / gbs_sort_pairs64, NEXT-4): the sort key of a 64-bit
// item is an order-preserving u64 image of its bits -- u64 as is, i64 with the sign bit
// flipped, f64 in IEEE-754 totalOrder (negatives -> ~x, others -> x ^ 2^63) -- sorted as
// the composite (hi, lo) of two u32 halves by two stable passes (lo, then hi).
__device__ __forceinline__ unsigned long long key64_image(unsigned long long x, int type)
{
    if (type == 1) return x ^ (1ull << 63);
    if (type == 2) return x ^ ((x >> 63) ? ~0ull : (1ull << 63));
    return x;
}
// pass 1 input: lo[i] = low half of key i's image, idx[i] = i (the stable sort's values)
__global__ void k_k64_lo(const unsigned long long* keys, uint64_t n, int type, uint32_t* lo, uint32_t* idx)
{
    pdl_entry();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        lo[i] = (uint32_t)key64_image(keys[i], type);
        idx[i] = (uint32_t)i;
    }
}
// pass 2 input: hi[i] = high half of the image of the key pass 1 put at position i
__global__ void k_k64_hi(const unsigned long long* keys, uint64_t n, int type, const uint32_t* idx, uint32_t* hi)
{
    pdl_entry();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        hi[i] = (uint32_t)(key64_image(keys[idx[i]], type) >> 32);
}
// output: out[i] = in[idx[i]] (the original bits), values likewise
__global__ void k_k64_gather(const unsigned long long* in, const uint32_t* idx, uint64_t n, unsigned long long* out,
                             const uint32_t* vin, uint32_t* vout)
{
    pdl_entry();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t j = idx[i];
        out[i] = in[j];
        if (vin) vout[i] = vin[j];
    }
}

// Debug-only invariant checks (GBS_DEBUG_SYNC): *flag |= 1 if some problem's sorted
// samples are out of order, |= 2 if some row of a does not sum to the sublist's
// real item count (conservation).
// With a selection-only Step 4 (k_s4_select) only the splitter positions are checked.
__global__ void k_check_level(LevelDev lv, unsigned* flag, int only_splitters)
{
    pdl_entry();
    const uint64_t ms = (uint64_t)lv.m * lv.s;
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < (uint64_t)lv.B * ms;
         q += (uint64_t)gridDim.x * blockDim.x) {
        if (only_splitters) {
            const uint64_t r = q % ms + 1;
            if (r % lv.m == 0 && r > lv.m && lv.samples[q] <= lv.samples[q - lv.m]) atomicOr(flag, 1u);
        } else if (q % ms != 0 && lv.samples[q] <= lv.samples[q - 1]) {
            atomicOr(flag, 1u);
        }
        if (q % lv.s == 0) {
            const uint64_t row = q / lv.s;
            const uint32_t b = (uint32_t)(row / lv.m), i = (uint32_t)(row % lv.m);
            const uint32_t len = lv.pr.length(b);
            const uint64_t i0 = (uint64_t)i * lv.L;
            const uint64_t v = len > i0 ? umin64(len - i0, lv.L) : 0;
            uint64_t sum = 0;
            for (uint32_t j = 0; j < lv.s; ++j) sum += lv.a[q + j];
            if (sum != v && atomicOr(flag, 2u) == 0) {
                flag[1] = b; flag[2] = i; flag[3] = (unsigned)sum; flag[4] = (unsigned)v; flag[5] = len;
                const u64 g = lv.samples[(uint64_t)b * ms + ms - 1];
                flag[6] = (unsigned)(g >> 32); flag[7] = (unsigned)g;
            }
        }
    }
}

// Nested Step 9: the buckets of this level become the problems of the next level.  Also
// the number of samples the next level's Step 4 must sort per problem: those of its
// non-empty sublists, ceil(len / Lc) * sc.  The samples of empty sublists are virtual
// sentinels (key 0xFFFFFFFF, tags above every real item, R8), already in sorted order
// after every real sample, so they stay where they are.
__global__ void k_child_desc(LevelDev lv, uint32_t* child_scnt, uint32_t Lc, uint32_t sc)
{
    pdl_entry();
    const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (uint64_t)lv.B * lv.s) return;
    const uint32_t b = (uint32_t)(idx / lv.s), j = (uint32_t)(idx % lv.s);
    const uint32_t* l0 = lv.l + (uint64_t)b * lv.m * lv.s;
    const uint32_t st = l0[j];
    const uint32_t en = j + 1 < lv.s ? l0[j + 1] : lv.pr.length(b);
    lv.child_off[idx] = lv.pr.offset(b) + st;
    lv.child_len[idx] = en - st;
    if (child_scnt) child_scnt[idx] = (uint32_t)(((uint64_t)(en - st) + Lc - 1) / Lc * sc);
}

}  // namespace gbs
