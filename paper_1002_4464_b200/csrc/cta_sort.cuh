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
// trailing zero bits: ITEMS = 2^Ctz * odd
template <int X> struct Ctz { static constexpr int value = (X & 1) ? 0 : 1 + Ctz<X / 2>::value; };
template <> struct Ctz<0> { static constexpr int value = 0; };

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

// Sorts x[0..N) of a register array of M >= N entries (a larger array lets one set of
// registers serve several tile sizes).
template <typename T, int N, int M, size_t... Cs>
__device__ __forceinline__ void apply_net(T (&x)[M], std::index_sequence<Cs...>)
{
    constexpr BatcherNet<N> net{};
    (cas(x[net.a[Cs]], x[net.b[Cs]]), ...);
}

template <typename T, int N, int M>
__device__ __forceinline__ void reg_sort(T (&x)[M])
{
    static_assert(N <= M, "register array too small");
    if constexpr (N > 1) apply_net<T, N, M>(x, std::make_index_sequence<BatcherNet<N>::C>{});
}

#ifndef GBS_SHFL_LEVELS
#define GBS_SHFL_LEVELS 4   // first merge levels on warp shuffles, 4-byte keys (0 = all through smem; 4 vs 3: C2 -0.4 %, C3 -0.3 %)
#endif
#ifndef GBS_SHFL_LEVELS_WIDE
#define GBS_SHFL_LEVELS_WIDE 1   // the same for 8-byte items (u64 composites, pairs): 1 measured +0.9% at C4, 2 slower
#endif

// Shared-memory merge levels keep the B run of every pair stored descending (a bitonic
// pair): a merge pointer that runs past the end of its run then walks down the other run
// from its far end, so no end-of-run checks are needed (see merge_thread).

template <typename T, int BLOCK, int ITEMS, int CHAINS_ = 0, int SHFL_ = -1>
struct CtaSort {
    static constexpr int TILE = BLOCK * ITEMS;
    // A tile that is not a power of two (BLOCK not a power of two, e.g. 544 x 32) has a
    // short last run at some levels; with B runs stored descending the merge handles it by
    // clipping the pair's run lengths (la, lb), nothing else changes.
    static constexpr bool POW2_TILE = (TILE & (TILE - 1)) == 0;
    static constexpr int LOG_ITEMS = Ctz<ITEMS>::value;   // log2(ITEMS) for a power of two
    static constexpr int WARP_SPAN = 32 * ITEMS;                  // items owned by one warp
    // Shared-memory layout: one pad slot every 2^PAD items.  PAD = ctz(ITEMS) (log2 for a
    // power of two) makes a thread's stride ITEMS + ITEMS/2^PAD odd, so the blocked
    // stores are conflict-free.
    static constexpr int PAD = LOG_ITEMS;
    static constexpr int SMEM_ELEMS = TILE + (TILE >> PAD) + 2;
    // independent merge chains per thread (ILP); overridable by the instantiation
    static constexpr int CHAINS = CHAINS_ > 0 ? CHAINS_ : ((ITEMS * sizeof(T) <= 256) ? 2 : 1);
    static constexpr T TMAX = ~T(0);
    // merge levels done with warp shuffles (power-of-two ITEMS only)
    // (SHFL_ >= 0: the instantiation's own count)
    static constexpr int SHFL_LEVELS =
        ((ITEMS & (ITEMS - 1)) == 0 && ITEMS >= 2)
            ? (SHFL_ >= 0 ? SHFL_ : (sizeof(T) == 4 ? GBS_SHFL_LEVELS : GBS_SHFL_LEVELS_WIDE))
            : 0;

    static __device__ __forceinline__ int phys(int p) { return p + (p >> PAD); }

    // Position of register slot k of the calling thread in the load order: each warp
    // owns a contiguous span of 32*ITEMS positions, read 32 consecutive at a time
    // (coalesced).  Valid positions then form a prefix of every warp span, which is
    // what the skip logic below relies on.
    static __device__ __forceinline__ int load_pos(int k)
    {
        return (threadIdx.x >> 5) * WARP_SPAN + k * 32 + (threadIdx.x & 31);
    }

    // Merge-path split of output diagonal `diag` of the pair (A = [a0, a0+w),
    // B = [a0+w, a0+2w), B stored descending), knowing the split lies in [lo, hi]: the
    // number of outputs taken from A (ties: A first -> stable).  B[diag-1-mid] sits at
    // a0 + 2w - 1 - (diag - 1 - mid) = bt + mid.
    static __device__ __forceinline__ int split_in(const T* sm, int a0, int w, int diag, int lo, int hi)
    {
        const int bt = a0 + 2 * w - diag;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sm[phys(a0 + mid)] <= sm[phys(bt + mid)]) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    }

    // REV layout with an explicit B top (first B item): B[j] at top - j
    static __device__ __forceinline__ int split_top(const T* sm, int a0, int top, int diag, int lo, int hi)
    {
        const int bt = top - diag + 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sm[phys(a0 + mid)] <= sm[phys(bt + mid)]) lo = mid + 1;
            else hi = mid;
        }
        return lo;
    }

    // Store the thread's ITEMS outputs [start, start+ITEMS), which belong to runs of
    // length w: ascending, or mirrored inside the run when the run is the B of the next
    // level's pair (odd run index).  The branch is warp-uniform once w >= 32 ITEMS.
    // lg = log2(w / ITEMS): the run of thread t is t >> lg (start = t ITEMS).
    template <int M>
    static __device__ __forceinline__ void store_run(const T (&x)[M], T* sm, int start, int w, int lg)
    {
        const int q = (int)threadIdx.x >> lg;                 // run index
        if (q & 1) {
            const int r0 = (q << lg) * ITEMS;                 // run start
            const int lr = POW2_TILE ? w : min(w, TILE - r0); // run length (the tile's last run may be short)
            const int e = 2 * r0 + lr - ITEMS - start;        // mirrored block start
            // e and start are multiples of ITEMS, hence of the pad group 2^PAD, so
            // phys(e + k) = phys(e) + k + (k >> PAD): one address, constant offsets
            const int pe = phys(e);
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) sm[pe + k + (k >> PAD)] = x[ITEMS - 1 - k];
        } else {
            const int ps = phys(start);
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) sm[ps + k + (k >> PAD)] = x[k];
        }
    }

    // The thread's ITEMS outputs [start, start+ITEMS) of the merge of the pair of
    // sorted runs (A = [base, base+w), B = [base+w, base+2w)) containing `start`,
    // produced by CHAINS independent merge-path chains of ITEMS/CHAINS outputs each,
    // interleaved for ILP (each step of a chain waits on one shared-memory load).
    // Ties take A first, so the merge is stable.
    //
    // B is stored descending (B[j] at base + 2w - 1 - j).  Per chain only the A position
    // ai is kept; the B head sits at ai + E - k after k outputs.  A pointer that passes
    // the end of its run reads the other run from its far end (its largest remaining
    // item), so every output is still the smallest remaining item and no end-of-run check
    // is needed: the two pointers consume the remaining items from both ends and never
    // cross within the thread's outputs.  The only items that can then be taken "from the
    // wrong side" are equal to the true output: keys (values only) are unaffected, and
    // 8-byte items (u64 composites, pairs as key<<32|position) are distinct.
    template <int M>
    static __device__ __forceinline__ void merge_thread(T (&x)[M], const T* sm, int start, int w)
    {
        static_assert(M >= ITEMS, "register array too small");
        constexpr int H = ITEMS / CHAINS;
        // w = ITEMS * 2^k; ITEMS itself need not be a power of two (the pair index is
        // taken on the thread index start / ITEMS)
        const int base = ((start / ITEMS) & ~(2 * (w / ITEMS) - 1)) * ITEMS;
        // run lengths of the pair (a short last run only in a non-power-of-two tile: then
        // B is empty or A is full); B's first item sits at `top` (B descending)
        const int la = POW2_TILE ? w : min(w, TILE - base);
        const int lb = POW2_TILE ? w : max(0, min(w, TILE - base - w));
        const int top = base + la + lb - 1;
        int ai[CHAINS], cb[CHAINS];
        T a[CHAINS], b[CHAINS];
        // chain c's split lies in [split(c-1), split(c-1) + H]: H more outputs take at most
        // H more items of A, so only the first chain searches the whole diagonal
        int sp = 0;
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) {
            const int diag = start - base + c * H;
            if (POW2_TILE)
                sp = c == 0 ? split_in(sm, base, w, diag, max(0, diag - w), min(diag, w))
                            : split_in(sm, base, w, diag, max(sp, diag - w), min(sp + H, min(diag, w)));
            else
                sp = split_top(sm, base, top, diag, c == 0 ? max(0, diag - lb) : max(sp, diag - lb),
                               c == 0 ? min(diag, la) : min(sp + H, min(diag, la)));
            ai[c] = base + sp;
            cb[c] = top - base - diag;                    // E: B head = ai + E - k
            a[c] = sm[phys(ai[c])];
            b[c] = sm[phys(ai[c] + cb[c])];
        }
#pragma unroll
        for (int k = 0; k < H; ++k) {
#pragma unroll
            for (int c = 0; c < CHAINS; ++c) {
                const bool t = a[c] <= b[c];
                x[c * H + k] = t ? a[c] : b[c];
                const int bnext = ai[c] + cb[c] - (k + 1);
                ai[c] += t ? 1 : 0;
                const int nidx = t ? ai[c] : bnext;
                const T v = sm[phys(nidx)];
                a[c] = t ? v : a[c];
                b[c] = t ? b[c] : v;
            }
        }
    }

    // The first SHFL_LEVELS merge levels (runs of ITEMS -> ITEMS << SHFL_LEVELS, i.e.
    // blocks of 2, 4, ... lanes) in registers with warp shuffles instead of shared
    // memory: a bitonic merge of two ascending runs whose first half-cleaner pairs each
    // item of the lower block with the mirror item of the upper one (folding in the
    // reversal of the upper run), after which both halves are bitonic and the remaining
    // half-cleaners (across lanes, then inside each lane) are all ascending.  On return
    // lane l of each block holds positions [l ITEMS, (l+1) ITEMS) of the block's sorted
    // run.  No shared-memory traffic and no merge-path search for these levels.
    template <int M>
    static __device__ __forceinline__ void warp_bitonic(T (&x)[M])
    {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int j = 0; j < SHFL_LEVELS; ++j) {
            const bool lower = !(lane & (1 << j));
            const int mirror = (2 << j) - 1;
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) {
                const T a = lower ? x[k] : x[ITEMS - 1 - k];
                const T r = __shfl_xor_sync(0xffffffffu, a, mirror);
                const T v = lower ? (r < a ? r : a) : (r < a ? a : r);
                if (lower) x[k] = v;
                else x[ITEMS - 1 - k] = v;
            }
#pragma unroll
            for (int q = j - 1; q >= 0; --q) {
                const bool lo = !(lane & (1 << q));
#pragma unroll
                for (int k = 0; k < ITEMS; ++k) {
                    const T r = __shfl_xor_sync(0xffffffffu, x[k], 1 << q);
                    x[k] = lo ? (r < x[k] ? r : x[k]) : (r < x[k] ? x[k] : r);
                }
            }
#pragma unroll
            for (int d = ITEMS / 2; d >= 1; d /= 2)
#pragma unroll
                for (int k = 0; k < ITEMS; ++k)
                    if ((k & d) == 0) cas(x[k], x[k + d]);
        }
    }

    // The thread's ITEMS outputs [start, start+ITEMS) of the merge of two sorted runs of
    // arbitrary lengths that fill the tile: run 1 = [0, len1), run 2 = [len1, TILE)
    // (ties: run 1 first).  The final, cross-CTA level of a CTA-pair sort.
    template <int M>
    static __device__ __forceinline__ void merge_two(T (&x)[M], const T* sm, int start, int len1)
    {
        static_assert(M >= ITEMS, "register array too small");
        const int len2 = TILE - len1;
        int lo = max(0, start - len2), hi = min(start, len1);
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sm[phys(mid)] <= sm[phys(len1 + start - 1 - mid)]) lo = mid + 1;
            else hi = mid;
        }
        int ai = lo, bi = len1 + start - lo;
        T a = ai < len1 ? sm[phys(ai)] : TMAX;
        T b = bi < TILE ? sm[phys(bi)] : TMAX;
        // warp-uniform fast path: no lane can exhaust a run within its ITEMS outputs
        if (__all_sync(__activemask(), ai + ITEMS <= len1 && bi + ITEMS <= TILE)) {
            const int cb = len1 + start + 1;             // bi after k steps = cb + k - ai
#pragma unroll
            for (int k = 0; k < ITEMS; ++k) {
                const bool t = a <= b;
                x[k] = t ? a : b;
                ai += t ? 1 : 0;
                const int nidx = t ? ai : cb + k - ai;
                const T v = sm[phys(nidx)];
                a = t ? v : a;
                b = t ? b : v;
            }
            return;
        }
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const bool t = a <= b;
            x[k] = t ? a : b;
            ai += t ? 1 : 0;
            bi += t ? 0 : 1;
            const int nidx = t ? ai : bi;
            const bool ok = nidx < (t ? len1 : TILE);
            T v = sm[phys(ok ? nidx : 0)];
            v = ok ? v : TMAX;
            a = t ? v : a;
            b = t ? b : v;
        }
    }

    // Tile whose runs of length R (power of two >= ITEMS) are already sorted: load it
    // into shared memory (phys layout, TMAX beyond valid) and run only the merge levels
    // w = R, 2R, ... .  Used for Step 4, whose input is m sorted runs of s samples
    // (each sublist's samples come out of its sorted sublist).  Block-synchronised.
    template <int M, typename Src>
    static __device__ __forceinline__ void sort_presorted(T (&x)[M], Src src, T* sm, int valid, int R)
    {
        static_assert(POW2_TILE, "presorted runs: power-of-two tiles only");
        const int t = threadIdx.x;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const int p = t + k * BLOCK;
            x[k] = p < valid ? src[p] : TMAX;
        }
        // odd runs of R stored mirrored: the B of each first-level pair
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) {
            const int p = t + k * BLOCK;
            const int r0 = p & ~(R - 1);
            sm[phys((p & R) && R < TILE ? 2 * r0 + R - 1 - p : p)] = x[k];
        }
        __syncthreads();
        const int start = t * ITEMS;
        const int wspan0 = (t >> 5) * WARP_SPAN;
        int lg = __ffs(R / ITEMS) - 1;                   // log2(w / ITEMS)
#pragma unroll 1
        for (int w = R; w < TILE; w *= 2, ++lg) {
            const bool intra = 2 * w <= WARP_SPAN;
            const bool active = intra ? (wspan0 < valid) : (start < valid);
            if (active) merge_thread(x, sm, start, w);
            if (intra) __syncwarp(); else __syncthreads();
            // every position is rewritten (the layout of the sentinel tail changes with
            // the run parity); idle threads' outputs are all sentinels
            if (!active) {
#pragma unroll
                for (int k = 0; k < ITEMS; ++k) x[k] = TMAX;
            }
            store_run(x, sm, start, 2 * w, lg + 1);
            // the NEXT level's readers decide the barrier: a cross-warp level reads
            // other warps' stores
            if (4 * w <= WARP_SPAN) __syncwarp(); else __syncthreads();
        }
    }

    // Load x[0..ITEMS) with the positions load_pos(k) of src[0, valid) (coalesced:
    // 32 consecutive per warp instruction); TMAX beyond valid.
    template <int M, typename Src>
    static __device__ __forceinline__ void load(T (&x)[M], Src src, int valid)
    {
        const int p0 = load_pos(0), rem = valid - p0;     // load_pos(k) = p0 + 32k
#pragma unroll
        for (int k = 0; k < ITEMS; ++k) x[k] = 32 * k < rem ? (T)src[p0 + 32 * k] : TMAX;
    }

    // Sort: x[] holds the items of positions load_pos(k) (sentinels at >= valid).
    // On return sm[phys(p)] holds the sorted tile for p < valid (block-synchronised).
    template <int M>
    static __device__ __forceinline__ void sort(T (&x)[M], T* sm, int valid)
    {
        const int t = threadIdx.x;
        const int wspan0 = (t >> 5) * WARP_SPAN;
        if (wspan0 < valid) {
            reg_sort<T, ITEMS, M>(x);
            if constexpr (SHFL_LEVELS > 0) warp_bitonic(x);
        }
        const int start = t * ITEMS;
        int lg = SHFL_LEVELS;                            // log2(w / ITEMS)
#pragma unroll 1
        for (int w = ITEMS << SHFL_LEVELS; w < TILE; w *= 2, ++lg) {
            const bool intra = 2 * w <= WARP_SPAN;
            store_run(x, sm, start, w, lg);
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
