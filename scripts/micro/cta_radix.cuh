// cta_radix.cuh (prototype, measured and rejected: profiles/r02/radix_ab.md) -- on-chip LSD radix sort of one tile (<= BLOCK*ITEMS u32 keys, or u32
// key -> u32 value pairs, stable) by one CTA.
//
// Steps 2 and 9 of Alg. 1 sort a sublist / bucket on one SM.  The
// paper sorted 2K items with a shared-memory bitonic network and reports trying
// quicksort and adaptive bitonic sort as well: the on-chip algorithm is free,
// because every correct sort of a tile yields the same bytes (keys: the sorted multiset;
// pairs: the stable order by key, R7).  On sm_100a a comparison merge sort of 2^15 keys
// costs ~207 instructions per key (round-1 ncu); an LSD radix sort over 8-bit digits does
// four data-oblivious passes of ~25 instructions per key:
//
//   phase A  per warp, in processing order (row k, then lane): the lanes holding the same
//            digit find each other with one MATCH.ANY; the lowest of them adds the group
//            size to the warp's counter of that digit (shared-memory atomic, returns the
//            old value) and broadcasts it: every key gets its rank among the warp's keys
//            of its digit (11 bits, two per register);
//   scan     exclusive scan of the NW x 256 counters in (digit, warp) order;
//   phase B  key -> position offset[warp][digit] + rank in the shared-memory buffer;
//   readback every thread reloads its keys in processing order for the next digit.
//
// Stability: the processing order of a pass is the output order of the previous pass
// (the first pass: the load order), and ranks follow it, so each pass is stable and the
// whole sort is stable -- pairs need no position tag (no 64-bit compares).
//
// Layout of the register slots: slot k of thread (warp w, lane) is processing position
// w*32*ITEMS + 32k + lane (the load order of CtaSort::load_pos, coalesced).  Valid items
// are a prefix of that order; rows (32 positions of one warp) beyond it are skipped, the
// partial last row is padded with 0xFFFFFFFF sentinels, which sort after every real key
// (stable: after real 0xFFFFFFFF keys too).  On return kb[0, valid) holds the sorted keys
// (plain layout, 16-byte aligned rows) and vb[0, valid) their values.
#pragma once
#include <cstdint>

namespace gbs {

template <int BLOCK, int ITEMS, bool MATCH = false>
struct CtaRadix {
    static constexpr int TILE = BLOCK * ITEMS;
    static constexpr int NW = BLOCK / 32;
    static constexpr int RADIX_BITS = 8, NB = 1 << RADIX_BITS;
    static constexpr int HS = NB + 1;                 // padded warp row: scan reads conflict-free
    static constexpr int HIST = NW * HS;              // words per counter array
    static constexpr int E = NW * NB / BLOCK;         // counters per thread in the scan (8)
    static constexpr int NRK = (ITEMS + 1) / 2;       // packed 16-bit ranks per thread
    static_assert(BLOCK % 32 == 0 && NW <= 32, "BLOCK: 32..1024 threads");
    static_assert(E * BLOCK == NW * NB && NW % E == 0, "scan split");
    static_assert(32 * ITEMS <= 65535, "ranks are 16-bit");

    // shared memory: keys TILE, values TILE (pairs), two counter arrays, 32 warp sums
    __host__ __device__ static constexpr size_t smem_words(bool pairs) { return (size_t)TILE * (pairs ? 2 : 1) + 2 * HIST + 32; }

    static __device__ __forceinline__ uint32_t lanemask_lt()
    {
        uint32_t m;
        asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
        return m;
    }

    // Exclusive scan of h[w*HS + d] in (d, w) order, in place.  Thread t owns the E
    // counters e = tE .. tE+E-1 (one digit, E consecutive warps).  Two barriers inside.
    static __device__ __forceinline__ void scan(uint32_t* h, uint32_t* wsum)
    {
        const int t = threadIdx.x, lane = t & 31, w = t >> 5;
        const int e0 = t * E, d = e0 / NW, w0 = e0 % NW;
        uint32_t* hp = h + w0 * HS + d;
        // (the counters are read twice rather than held: the caller's keys and ranks
        // occupy most of the registers here)
        uint32_t s = 0;
#pragma unroll
        for (int i = 0; i < E; ++i) s += hp[i * HS];
        uint32_t inc = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        // every warp scans the NW warp totals itself (no second barrier)
        uint32_t ws = lane < NW ? wsum[lane] : 0u, wi = ws;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        const uint32_t wbase = __shfl_sync(0xffffffffu, wi - ws, w);
        uint32_t run = wbase + inc - s;
#pragma unroll
        for (int i = 0; i < E; ++i) {
            const uint32_t v = hp[i * HS];
            hp[i * HS] = run;
            run += v;
        }
    }

    // One pass over digit bits [sh, sh + 8).  rows = valid rows of this warp (uniform).
    // LAST: the keys (values) stay in kb (vb); otherwise they are reloaded into x (y).
    // hc: this pass's counters (zero on entry); hn: the next pass's, zeroed here.
    template <bool PAIRS, bool LAST, int M>
    static __device__ __forceinline__ void pass(uint32_t (&x)[M], uint32_t (&y)[M], uint32_t* kb, uint32_t* vb,
                                                uint32_t* hc, uint32_t* hn, uint32_t* wsum, int sh, int rows)
    {
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        uint32_t* hw = hc + w * HS;
        const uint32_t ltm = lanemask_lt();
        uint32_t rk[NRK];
#pragma unroll
        for (int q = 0; q < NRK; ++q) rk[q] = 0u;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            if (k < rows) {
                const uint32_t d = (x[k] >> sh) & (NB - 1);
                uint32_t peers;
                if (MATCH) {
                    peers = __match_any_sync(0xffffffffu, d);
                } else {   // MATCH.ANY is microcoded on sm_100a: 8 ballots instead
                    peers = 0xffffffffu;
#pragma unroll
                    for (int b = 0; b < RADIX_BITS; ++b) {
                        const bool bit = (d >> b) & 1u;
                        const uint32_t m = __ballot_sync(0xffffffffu, bit);
                        peers &= bit ? m : ~m;
                    }
                }
                const uint32_t lt = __popc(peers & ltm);
                uint32_t old = 0;
                if (lt == 0) old = atomicAdd(hw + d, (uint32_t)__popc(peers));
                old = __shfl_sync(0xffffffffu, old, __ffs(peers) - 1);
                const uint32_t r = old + lt;
                rk[k >> 1] |= r << ((k & 1) * 16);
            }
        }
        if (!LAST) {
            for (int q = threadIdx.x; q < HIST; q += BLOCK) hn[q] = 0u;
        }
        __syncthreads();
        scan(hc, wsum);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            if (k < rows) {
                const uint32_t d = (x[k] >> sh) & (NB - 1);
                const uint32_t pos = hw[d] + ((rk[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu);
                kb[pos] = x[k];
                if (PAIRS) vb[pos] = y[k];
            }
        }
        __syncthreads();
        if (!LAST) {
            const int p0 = w * 32 * ITEMS + lane;
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) {
                if (k < rows) {
                    x[k] = kb[p0 + 32 * k];
                    if (PAIRS) y[k] = vb[p0 + 32 * k];
                }
            }
        }
    }

    // Sort: x (and y) hold processing positions w*32*ITEMS + 32k + lane, sentinels at
    // >= valid.  h0/h1: counter arrays (HIST words each), wsum: 32 words.  On return
    // (block-synchronised) kb[0, valid) / vb[0, valid) hold the sorted tile.
    template <bool PAIRS, int M>
    static __device__ __forceinline__ void sort(uint32_t (&x)[M], uint32_t (&y)[M], uint32_t* kb, uint32_t* vb,
                                                uint32_t* h0, uint32_t* h1, uint32_t* wsum, int valid)
    {
        static_assert(M >= ITEMS, "register array too small");
        const int w = threadIdx.x >> 5;
        const int rem = valid - w * 32 * ITEMS;
        const int rows = rem <= 0 ? 0 : min(ITEMS, (rem + 31) >> 5);
        for (int q = threadIdx.x; q < HIST; q += BLOCK) h0[q] = 0u;
        __syncthreads();
        pass<PAIRS, false>(x, y, kb, vb, h0, h1, wsum, 0, rows);
        pass<PAIRS, false>(x, y, kb, vb, h1, h0, wsum, 8, rows);
        pass<PAIRS, false>(x, y, kb, vb, h0, h1, wsum, 16, rows);
        pass<PAIRS, true>(x, y, kb, vb, h1, h0, wsum, 24, rows);
    }
};


// Thread-private counters (no MATCH, no atomics): 4-bit digits, 8 passes.  Processing
// order is blocked: slot k of thread t is position t*ITEMS + k.  cnt[d][t] (u32, one pad
// word per 32) counts thread t's keys of digit d; the exclusive scan of cnt in (d, t)
// order plus the thread's running count gives every key its stable position.
template <int BLOCK, int ITEMS, int BITS = 4>
struct CtaRadixT {
    static constexpr int TILE = BLOCK * ITEMS;
    static constexpr int NB = 1 << BITS;
    static constexpr int NC = NB * BLOCK;                       // counters
    static constexpr int CW = NC + NC / 32;                     // counter words (padded)
    static constexpr int KW = TILE + TILE / 32;                 // key words (padded)
    static constexpr int NRK = (ITEMS + 1) / 2;
    static constexpr int PASSES = (32 + BITS - 1) / BITS;
    __host__ __device__ static constexpr size_t smem_words(bool pairs) { return (size_t)KW * (pairs ? 2 : 1) + CW + 32; }
    static __device__ __forceinline__ int phys(int p) { return p + (p >> 5); }

    // exclusive scan of the counters in (d, t) order; thread t owns flat [t NB, (t+1) NB)
    static __device__ __forceinline__ void scan(uint32_t* c, uint32_t* wsum)
    {
        const int t = threadIdx.x, lane = t & 31, w = t >> 5;
        const int e0 = t * NB;
        uint32_t s = 0;
#pragma unroll
        for (int i = 0; i < NB; ++i) s += c[phys(e0 + i)];
        uint32_t inc = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        uint32_t ws = lane < BLOCK / 32 ? wsum[lane] : 0u, wi = ws;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        uint32_t run = __shfl_sync(0xffffffffu, wi - ws, w) + inc - s;
#pragma unroll
        for (int i = 0; i < NB; ++i) {
            const uint32_t v = c[phys(e0 + i)];
            c[phys(e0 + i)] = run;
            run += v;
        }
    }

    template <bool PAIRS, bool LAST, int M>
    static __device__ __forceinline__ void pass(uint32_t (&x)[M], uint32_t (&y)[M], uint32_t* kb, uint32_t* vb, uint32_t* cnt,
                                                uint32_t* wsum, int sh, int items)
    {
        const int t = threadIdx.x;
        uint32_t* ct = cnt + t + (t >> 5);                       // phys(d*BLOCK + t) = ct + d*(BLOCK + BLOCK/32)
        constexpr int DS = BLOCK + BLOCK / 32;
#pragma unroll
        for (int d = 0; d < NB; ++d) ct[d * DS] = 0u;
        uint32_t rk[NRK];
#pragma unroll
        for (int q = 0; q < NRK; ++q) rk[q] = 0u;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            if (k < items) {
                const uint32_t d = (x[k] >> sh) & (NB - 1);
                const uint32_t c = ct[d * DS];
                ct[d * DS] = c + 1;
                rk[k >> 1] |= c << ((k & 1) * 16);
            }
        }
        __syncthreads();
        scan(cnt, wsum);
        __syncthreads();
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            if (k < items) {
                const uint32_t d = (x[k] >> sh) & (NB - 1);
                const int pos = (int)(ct[d * DS] + ((rk[k >> 1] >> ((k & 1) * 16)) & 0xFFFFu));
                kb[phys(pos)] = x[k];
                if (PAIRS) vb[phys(pos)] = y[k];
            }
        }
        __syncthreads();
        if (!LAST) {
            const int p0 = phys(t * ITEMS);
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) {
                if (k < items) {
                    x[k] = kb[p0 + k + (k >> 5)];
                    if (PAIRS) y[k] = vb[p0 + k + (k >> 5)];
                }
            }
        }
    }

    // x/y: thread t holds positions t*ITEMS + k (sentinels 0xFFFFFFFF at >= valid).  On
    // return kb[phys(p)] (vb[phys(p)]) hold the sorted tile, p < valid.
    template <bool PAIRS, int M>
    static __device__ __forceinline__ void sort(uint32_t (&x)[M], uint32_t (&y)[M], uint32_t* kb, uint32_t* vb, uint32_t* cnt,
                                                uint32_t* wsum, int valid)
    {
        const int rem = valid - (int)threadIdx.x * ITEMS;
        const int items = rem <= 0 ? 0 : min(ITEMS, rem);
#pragma unroll
        for (int ps = 0; ps < PASSES - 1; ++ps) pass<PAIRS, false>(x, y, kb, vb, cnt, wsum, ps * BITS, items);
        pass<PAIRS, true>(x, y, kb, vb, cnt, wsum, (PASSES - 1) * BITS, items);
    }
};

}  // namespace gbs
