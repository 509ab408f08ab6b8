// gbs_api.cu -- planner, launch sequence and C-ABI of libgbs.so (include/gbs.h).
//
// The plan is static: it depends on (n, item kind, config) only, never on the data
// (the paper's guaranteed bucket sizes, make every grid size known up
// front), so a sort is a fixed, host-sync-free sequence of launches on one stream
// (CUDA-graph capturable).  See DESIGN.md section 5 for the plan rule.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <type_traits>
#include <vector>
#include <vector>

#include "../../include/gbs.h"
#include "gbs_internal.h"
#include "gbs_kernels.cuh"

namespace gbs {

// ----------------------------------------------------------------- errors
static thread_local char g_err[512] = "";

static gbs_status_t fail(gbs_status_t st, const char* fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return st;
}

#define GBS_CUDA(call)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(GBS_ERROR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),   \
                        __FILE__, __LINE__);                                               \
    } while (0)

// GBS_DEBUG_SYNC=1 in the environment: synchronise after every launch so a device fault
// is attributed to its launch site (debugging only; never set in benchmarks).
static bool debug_sync()
{
    static const bool on = getenv("GBS_DEBUG_SYNC") != nullptr;
    return on;
}

#define GBS_LAUNCHED()                                                                     \
    do {                                                                                   \
        cudaError_t e_ = cudaGetLastError();                                               \
        if (e_ == cudaSuccess && debug_sync()) e_ = cudaDeviceSynchronize();               \
        if (e_ != cudaSuccess)                                                             \
            return fail(GBS_ERROR_CUDA, "kernel launch: %s (%s:%d, node kind %d B %u)",     \
                        cudaGetErrorString(e_), __FILE__, __LINE__, KIND, nd.B);           \
    } while (0)

// ----------------------------------------------------------------- step profiling
// Per-step CUDA events on the call's stream for the top level (gbs_profile_begin/end).
static thread_local bool g_prof = false;
struct ProfCall {
    int level;                       // 0 = top level, k = k-th nested Step 9 level
    std::array<cudaEvent_t, 8> ev;
};
static thread_local std::deque<ProfCall> g_prof_calls;   // deque: stable element addresses

struct ProfMarks {
    cudaEvent_t* ev = nullptr;
    cudaStream_t st = nullptr;
    int next = 0;
    void mark()
    {
        if (ev) cudaEventRecord(ev[next++], st);
    }
};

// ----------------------------------------------------------------- plan
constexpr uint32_t TILE_KEYS = 1u << 15;   // u32 keys per CTA tile
constexpr uint32_t TILE_PAIRS = 1u << 14;  // pairs per CTA tile (u64 on chip + values)
constexpr uint32_t TILE_U64 = 1u << 14;    // u64 composites per CTA tile
constexpr uint32_t SMALL_TILE = 2048;      // small CTA configuration
#ifndef GBS_SPLIT_STEP9
#define GBS_SPLIT_STEP9 1
#endif
#ifndef GBS_FUSE_89
#define GBS_FUSE_89 1     // fused Step 8+9 for CTA-bucket levels
#endif
#ifndef GBS_PAIR_BUCKETS
#define GBS_PAIR_BUCKETS 1  // keys: Step 9 on CTA pairs when one-tile buckets would nest
#endif
#ifndef GBS_FUSE_PAIRS
#define GBS_FUSE_PAIRS 1  // ... for pairs as well (C4: 81.6 -> 80.8 ms)
#endif
#ifndef GBS_FUSE_MIN_D
#define GBS_FUSE_MIN_D 32 // ... whose average run d = L/s is at least this many items
#endif
constexpr bool GBS_SPLIT_STEP9_ON = GBS_SPLIT_STEP9;
constexpr uint64_t SMALL_U64_TOTAL = 1u << 18;   // u64 levels up to this many samples use 2K tiles
#ifndef GBS_PAIR_BELOW_D
#define GBS_PAIR_BELOW_D 16                       // CTA-pair sublists when the one-tile d is below (0 = off)
#endif
#ifndef GBS_SMALL_N_KEYS
#define GBS_SMALL_N_KEYS (1u << 17)   // keys problems up to this size use 2K sublists and buckets (0 = off)
#endif
constexpr uint32_t D_MIN = 8;              // single level needs d >= 8
constexpr uint32_t D_NEST = 32;            // d of a level with a nested Step 9
constexpr uint32_t MAX_S = 4096;           // shared-memory limit of Steps 6 and 8
#ifndef GBS_IDX_BLOCK
#define GBS_IDX_BLOCK 512
#endif
constexpr int IDX_BLOCK = GBS_IDX_BLOCK;   // Steps 6 and 8 CTA size

static constexpr uint32_t tile_of_c(int kind) { return kind == KIND_KEYS ? TILE_KEYS : (kind == KIND_PAIRS ? TILE_PAIRS : TILE_U64); }
static uint32_t tile_of(int kind) { return tile_of_c(kind); }
static size_t key_bytes(int kind) { return kind == KIND_U64 ? 8 : 4; }

static uint64_t hi_bound(uint64_t cap, uint32_t L, uint32_t s)
{
    const uint64_t m = (cap + L - 1) / L, d = L / s;
    return m * L / s + (m - 1) * (d - 1);
}

struct Node {
    int kind = 0;
    uint32_t B = 1;
    uint64_t N = 0;
    bool leaf = false, small = false;
    uint32_t L = 0, s = 0, m = 0, d = 0;
    uint64_t Np = 0, hi = 0;
    uint32_t pad_base = 0;
    bool local_small = false, bucket_small = false;
    bool local_pair = false;   // Step 2 on CTA pairs (L = 2 tiles, keys)
    bool bucket_pair = false;  // Step 9 on CTA pairs (buckets up to 2 tiles, keys)
    int step4 = -1, step9 = -1;
    size_t o_samples = 0, o_splitters = 0, o_a = 0, o_l = 0, o_state = 0;
    size_t o_child_off = 0, o_child_len = 0, o_reloc = SIZE_MAX, o_reloc_v = SIZE_MAX;
    size_t o_child_scnt = 0;   // the nested level's samples to sort per problem (k_child_desc)
    size_t o_tiers = 0;   // Step 9 size-tier lists (3 x B*s) + counters (4)
    size_t o_pex = 0;     // fused Step 8+9: run starts P_i,j-1 (B*m*s)
    bool fuse89 = false;  // Step 9 gathers straight from the sorted sublists (no Step 8 pass)
    bool s4_tree = false; // Step 4 as a merge tree (R22) instead of a u64 level
    int s4_levels = 0;    // its global merge levels (between the tile merge and the selection)
    int level = 0;        // 0 top, k nested Step 9 level k, -1 a Step 4 sample level (profiling)
    size_t o_s4tmp = 0;   // its ping-pong buffer (m*s u64)
};

// big / small CTA configurations per kind
// (overridable with -D for tuning experiments)
#ifndef GBS_KEYS_BLOCK
#define GBS_KEYS_BLOCK 1024
#define GBS_KEYS_ITEMS 32
#endif
#ifndef GBS_WIDE_BLOCK
#define GBS_WIDE_BLOCK 1024
#define GBS_WIDE_ITEMS 16
#endif
#define GBS_BIG_KEYS GBS_KEYS_BLOCK, GBS_KEYS_ITEMS
#define GBS_BIG_WIDE GBS_WIDE_BLOCK, GBS_WIDE_ITEMS
// Step 9 of pairs (packed 4-byte tile items): the full tile, the mid tier and the tier of
// buckets up to its capacity (tier 0)
#ifndef GBS_PAIRS_BIG_BLOCK
#define GBS_PAIRS_BIG_BLOCK 1024
#define GBS_PAIRS_BIG_ITEMS 16
#endif
#ifndef GBS_PAIRS_MID_BLOCK
#define GBS_PAIRS_MID_BLOCK 1024
#define GBS_PAIRS_MID_ITEMS 10
#endif
#ifndef GBS_PAIRS_T0_BLOCK
#define GBS_PAIRS_T0_BLOCK 512
#define GBS_PAIRS_T0_ITEMS 16
#endif
// the full-tile CTA of Step 9 per kind
#define BIGB(K) ((K) == KIND_KEYS ? GBS_KEYS_BLOCK : ((K) == KIND_PAIRS ? GBS_PAIRS_BIG_BLOCK : GBS_WIDE_BLOCK))
#define BIGI(K) ((K) == KIND_KEYS ? GBS_KEYS_ITEMS : ((K) == KIND_PAIRS ? GBS_PAIRS_BIG_ITEMS : GBS_WIDE_ITEMS))
#ifndef GBS_PAIRS_LOCAL_BLOCK
#define GBS_PAIRS_LOCAL_BLOCK 512   // Step 2 of pairs: 512 x 32 (C4 80.9 -> 78.8 ms vs 1024 x 16)
#define GBS_PAIRS_LOCAL_ITEMS 32
#endif
#define GBS_PAIRS_LOCAL GBS_PAIRS_LOCAL_BLOCK, GBS_PAIRS_LOCAL_ITEMS
#ifndef GBS_SMALL
#define GBS_SMALL 256, 8
#endif

// Step 9 in size tiers (<= half a tile on 512-thread CTAs, then a 1024-thread mid tier,
// then the full tile) when the buckets use the big configuration and may exceed half a
// tile.
#ifndef GBS_MID_STEP9
#define GBS_MID_STEP9 1
#endif
// Step 9 mid tier: 5/8 of the full tile; keys on 512 threads x 40 (64 registers, 2 CTAs
// per SM), 8-byte items on 1024 x 10 (20 u64 per thread would spill)
// Step 9 mid tier (buckets just above half a tile), keys: at the top level 544 x 32
// (17408 keys: a non-power-of-two tile whose short last run the bitonic-pair merge clips;
// power-of-two items keep the shuffle levels), in nested levels 512 x 40 (wider bucket
// spread).  Buckets above the mid tier go to the full-tile tier.
#ifndef GBS_MID_TOP_BLOCK
#define GBS_MID_TOP_BLOCK 544
#define GBS_MID_TOP_ITEMS 32
#endif
#ifndef GBS_MID_KEYS_ITEMS_NESTED
#define GBS_MID_KEYS_ITEMS_NESTED 40
#endif
#ifndef GBS_U64_MID_BLOCK
#define GBS_U64_MID_BLOCK 512   // u64 sample levels' mid tier: 512 x 20 (C4 Step 4 -0.06 ms per level vs 1024 x 10)
#define GBS_U64_MID_ITEMS 20
#endif
#define MID_BLOCK_OF(KIND) \
    ((KIND) == KIND_KEYS ? GBS_MID_TOP_BLOCK : ((KIND) == KIND_PAIRS ? GBS_PAIRS_MID_BLOCK : GBS_U64_MID_BLOCK))
#define MID_ITEMS_OF(KIND) \
    ((KIND) == KIND_KEYS ? GBS_MID_TOP_ITEMS : ((KIND) == KIND_PAIRS ? GBS_PAIRS_MID_ITEMS : GBS_U64_MID_ITEMS))
static uint32_t mid_cap(int kind, uint32_t B)
{
    if (kind == KIND_PAIRS) return (uint32_t)GBS_PAIRS_MID_BLOCK * GBS_PAIRS_MID_ITEMS;
    if (kind != KIND_KEYS) return (uint32_t)GBS_U64_MID_BLOCK * GBS_U64_MID_ITEMS;
    return B == 1 ? (uint32_t)GBS_MID_TOP_BLOCK * GBS_MID_TOP_ITEMS : 512u * GBS_MID_KEYS_ITEMS_NESTED;
}
// The mid tiers of a node: keys at the top level have two, (C/2, 544 x 32] and
// (544 x 32, 512 x 48] (few-bucket problems spread wider); everything else one.
// cuts[0..2] are the tiers' upper bounds (an unused tier repeats the previous cut).
#ifndef GBS_MID2_TOP_ITEMS
#define GBS_MID2_TOP_ITEMS 48
#endif
static void tier_cuts(int kind, const Node& nd, uint32_t tile, uint32_t cuts[3])
{
    cuts[0] = kind == KIND_PAIRS ? (uint32_t)GBS_PAIRS_T0_BLOCK * GBS_PAIRS_T0_ITEMS : tile / 2;
    cuts[1] = GBS_MID_STEP9 ? mid_cap(kind, nd.B) : tile;
    cuts[2] = cuts[1];
    if (GBS_MID_STEP9 && kind == KIND_KEYS && nd.B == 1 && GBS_MID2_TOP_ITEMS > 0)
        cuts[2] = std::max(cuts[1], 512u * GBS_MID2_TOP_ITEMS);
}
static bool split_step9(int kind, const Node& nd)
{
    return !nd.bucket_small && nd.step9 < 0 && nd.hi > tile_of(kind) / 2;
}
// Step 9 launches of a CTA-bucket node: one, or the size tiers <= tile/2, mid, > mid
static int step9_launches(int kind, const Node& nd)
{
    if (!(GBS_SPLIT_STEP9_ON && split_step9(kind, nd))) return 1;
    // + the classification kernel (k_bucket_tiers)
    if (!GBS_MID_STEP9) return 3;
    uint32_t cuts[3];
    tier_cuts(kind, nd, tile_of(kind), cuts);
    return 3 + (nd.hi > cuts[1] && cuts[2] > cuts[1] ? 1 : 0) + (nd.hi > cuts[2] ? 1 : 0);
}

struct Plan {
    std::vector<Node> nodes;
    size_t ws = 0;
    int launches = 0;
    size_t alloc(size_t bytes)
    {
        const size_t o = ws;
        ws += (bytes + 255) / 256 * 256;
        return o;
    }
};

#ifndef GBS_S4_TREE
#define GBS_S4_TREE 1     // Step 4 of one problem with <= GBS_S4_TREE_MAX samples as a merge tree (R22)
#endif
#ifndef GBS_S4_TREE_MAX
#define GBS_S4_TREE_MAX (1u << 23)   // 64 MB of composites: L2-resident (126 MB)
#endif
#ifndef GBS_S4_TILE_BLOCK
#define GBS_S4_TILE_BLOCK 1024        // tile merge CTA: x 16 u64 per thread
#endif
constexpr uint32_t S4_TILE = GBS_S4_TILE_BLOCK * 16;

static bool pow2(uint64_t x) { return x && !(x & (x - 1)); }
static int reloc_launches(int kind);   // Step 8: 1, or 2 when both relocation forms are launched

// Returns node index, or -1 with g_err set.
static int build_node(Plan& P, int kind, uint32_t B, uint64_t N, uint32_t pad_base, const gbs_config_t* cfg,
                      bool own_reloc, int level = 0)
{
    const uint32_t tile = tile_of(kind);
    Node nd;
    nd.kind = kind;
    nd.B = B;
    nd.N = N;
    nd.pad_base = pad_base;
    nd.level = level;
    const bool use_cfg = cfg && cfg->L;
    if (!use_cfg && N <= tile) {
        nd.leaf = true;
        nd.small = N <= SMALL_TILE;
        P.launches += 1;
        P.nodes.push_back(nd);
        return (int)P.nodes.size() - 1;
    }
    uint32_t L, s = 0;
    if (use_cfg) {
        L = cfg->L;
        s = cfg->s;
    } else {
        // A small u64 level (few hundred thousand samples at most) would run as a handful
        // of big-tile CTAs, i.e. at the latency of one CTA sort; with 2K tiles it spreads
        // over many SMs.  Only when a single level with d >= D_MIN exists at that tile.
        if (kind == KIND_U64 && (uint64_t)B * N <= SMALL_U64_TOTAL) {
            for (uint32_t c = 2; c <= SMALL_TILE / D_MIN; c *= 2)
                if (hi_bound(N, SMALL_TILE, c) <= SMALL_TILE) { s = c; break; }
        }
        // A small keys problem (a few big-tile sublists) is latency-bound the same way:
        // 2K sublists and 2K buckets spread Steps 2 and 9 over many SMs (2^16: 0.119 ->
        // 0.047 ms).  Up to 2^17 keys, where the samples still sort in one CTA; above,
        // the larger Step 4 costs more than the spread saves (measured at 2^20, 2^21).
        if (kind == KIND_KEYS && B == 1 && N <= GBS_SMALL_N_KEYS) {
            for (uint32_t c = 2; c <= SMALL_TILE / D_MIN && !s; c *= 2)
                if (hi_bound(N, SMALL_TILE, c) <= SMALL_TILE) s = c;
        }
        // (8K tiles for mid-size u64 levels measured slower at C2 and C3)
        if (s) {
            L = SMALL_TILE;
        } else {
            L = tile;
            for (uint32_t c = 2; c <= L / D_MIN; c *= 2)
                if (hi_bound(N, L, c) <= tile) { s = c; break; }
            // keys whose one-tile plan needs d < GBS_PAIR_BELOW_D (samples > n/16): sublists
            // of two tiles sorted by CTA pairs (NEXT-2) when that gives a one-level plan
            // -- half the samples (Step 4) and twice the run length (Step 8) at equal bound
            if (kind == KIND_KEYS && GBS_PAIR_BELOW_D > 0 && s && L / s < GBS_PAIR_BELOW_D) {
                for (uint32_t c = 2; c <= 2 * tile / D_MIN; c *= 2)
                    if (hi_bound(N, 2 * tile, c) <= tile) { L = 2 * tile; s = c; break; }
            }
            // keys with no one-level plan at one-tile buckets: buckets of two tiles sorted
            // by CTA pairs (NEXT-2, R20) when that gives one level (2^27: 2^16-key sublists,
            // s = 4096, bound 63,473) -- one fewer CTA-sort pass than a nested Step 9
            if (kind == KIND_KEYS && B == 1 && !s && GBS_PAIR_BUCKETS) {
                for (uint32_t Lc = 2 * tile; Lc >= tile && !s; Lc /= 2)
                    for (uint32_t c = 2; c <= Lc / D_MIN && c <= MAX_S; c *= 2)
                        if (hi_bound(N, Lc, c) <= 2 * tile) { L = Lc; s = c; break; }
                if (s) nd.bucket_pair = true;
            }
            if (!s) s = L / D_NEST;
        }
    }
    nd.L = L;
    nd.s = s;
    nd.m = (uint32_t)((N + L - 1) / L);
    nd.d = L / s;
    nd.Np = (uint64_t)nd.m * L;
    nd.hi = hi_bound(N, L, s);
    if (nd.Np >= (1ull << 32) - (1ull << 20)) { snprintf(g_err, sizeof g_err, "problem too large for 32-bit tags"); return -1; }
    if (kind == KIND_U64 && (uint64_t)pad_base + nd.Np >= (1ull << 32)) { snprintf(g_err, sizeof g_err, "sentinel tag overflow"); return -1; }
    nd.local_small = L <= SMALL_TILE;
    nd.local_pair = kind == KIND_KEYS && L == 2 * tile;
    const uint64_t ms = (uint64_t)B * nd.m * s;
    nd.o_samples = P.alloc(ms * 8);
    nd.o_splitters = P.alloc((uint64_t)B * s * 8);
    nd.o_a = P.alloc(ms * 4);
    nd.o_l = P.alloc(ms * 4);
    nd.o_state = P.alloc((uint64_t)B * ((s + 31) / 32) * 8 + 8);   // + the longest-run word (Step 7)
    nd.o_pex = P.alloc(ms * 4);   // run starts P_i,j-1 (Step 6 -> grouped Step 8 / fused Step 8+9)
    if (own_reloc) {
        nd.o_reloc = P.alloc((uint64_t)B * N * key_bytes(kind));
        if (kind == KIND_PAIRS) nd.o_reloc_v = P.alloc((uint64_t)B * N * 4);
    }
    P.launches += 3;  // local sort (+samples), sample index (+splitters), scan
    const int idx = (int)P.nodes.size();
    P.nodes.push_back(nd);
    const uint32_t child_pad = kind == KIND_U64 ? pad_base + (uint32_t)(nd.Np - N) : (uint32_t)nd.Np;
    if (GBS_S4_TREE && B == 1 && ms > S4_TILE && ms <= GBS_S4_TREE_MAX) {
        // Step 4 as a merge tree (R22): tile merge, global pair levels until two runs are
        // left, then the selection of the s splitters
        Node& me = P.nodes[idx];
        me.s4_tree = true;
        me.o_s4tmp = P.alloc(ms * 8);
        for (uint64_t R = S4_TILE; 2 * R < ms; R *= 2) ++me.s4_levels;
        P.launches += 2 + me.s4_levels;
    } else {
        const int c4 = build_node(P, KIND_U64, B, (uint64_t)nd.m * s, child_pad, nullptr, true, -1);
        if (c4 < 0) return -1;
        P.nodes[idx].step4 = c4;
    }
    if (nd.bucket_pair) {
        // relocate + tiers (k_bucket_tiers, <= C/2, <= C, CTA pairs)
        P.launches += reloc_launches(kind) + 4;
        P.nodes[idx].o_tiers = P.alloc(((uint64_t)B * s * 4 + 4) * 4);
    } else if (nd.hi <= tile) {
        P.nodes[idx].bucket_small = nd.hi <= SMALL_TILE;
        // buckets that may exceed half a tile: size tiers (see exec_kind)
        P.launches += step9_launches(kind, P.nodes[idx]);
        if (GBS_SPLIT_STEP9_ON && split_step9(kind, P.nodes[idx]))
            P.nodes[idx].o_tiers = P.alloc(((uint64_t)B * s * 4 + 4) * 4);
        // fused Step 8+9 when the bucket's m run descriptors fit the staging area
        // (a production call; stop_after_step runs keep the explicit Step 8)
        // (keys only for now: the 16-item u64 / pair gather variants spill registers)
        // and the runs are long enough (d = L/s items on average) for the gathered reads
        // not to over-fetch: at d = 16 (64-byte runs) the scattered reads cost what the
        // relocation pass costs (measured); at d >= 32 and on small inputs the fused path wins
        if (GBS_FUSE_89 && (kind == KIND_KEYS || (kind == KIND_PAIRS && GBS_FUSE_PAIRS)) &&
            P.nodes[idx].m <= gather_max_m(kind) &&
            P.nodes[idx].d >= GBS_FUSE_MIN_D) {
            P.nodes[idx].fuse89 = true;
        } else {
            P.launches += reloc_launches(kind);
        }
    } else {
        P.nodes[idx].o_child_off = P.alloc((uint64_t)B * s * 8);
        P.nodes[idx].o_child_len = P.alloc((uint64_t)B * s * 4);
        P.nodes[idx].o_child_scnt = P.alloc((uint64_t)B * s * 4);
        P.launches += reloc_launches(kind) + 1;  // relocate + child descriptors
        const uint64_t nb = (uint64_t)B * s;
        if (nb >= (1ull << 31)) { snprintf(g_err, sizeof g_err, "too many nested problems"); return -1; }
        const int c9 = build_node(P, kind, (uint32_t)nb, nd.hi, child_pad, nullptr, false, level >= 0 ? level + 1 : -1);
        if (c9 < 0) return -1;
        P.nodes[idx].step9 = c9;
    }
    return idx;
}

static gbs_status_t make_plan(size_t n, int kind, const gbs_config_t* cfg, Plan& P)
{
    if (n > (1ull << 31)) return fail(GBS_ERROR_UNSUPPORTED, "n = %zu > 2^31", n);
    if (cfg && (cfg->L || cfg->s)) {
        const uint32_t L = cfg->L, s = cfg->s;
        // keys may use sublists of two tiles (CTA-pair local sort); Step 9 stays one tile
        const uint32_t maxL = kind == KIND_KEYS ? 2 * tile_of(kind) : tile_of(kind);
        if (!pow2(L) || !pow2(s) || s > L || L > maxL || s > MAX_S || (L > tile_of(kind) && s < 2))
            return fail(GBS_ERROR_INVALID_VALUE, "bad config L=%u s=%u (powers of two, s<=L<=%u, s<=%u)", L, s,
                        maxL, MAX_S);
    }
    P = Plan();
    if (n <= 1) return GBS_SUCCESS;
    const gbs_config_t* c = (cfg && cfg->L) ? cfg : nullptr;
    if (build_node(P, kind, 1, n, 0, c, true) < 0) return fail(GBS_ERROR_UNSUPPORTED, "%s", g_err);
    return GBS_SUCCESS;
}

// ----------------------------------------------------------------- launches
static uint32_t num_sms();
constexpr int S4_MERGE_BLOCK = 256, S4_MERGE_ITEMS = 16;
#ifndef GBS_IDX_TMA
#define GBS_IDX_TMA 1
#endif

#ifndef GBS_PDL
#define GBS_PDL 1   // programmatic dependent launch between the kernels of a sort
#endif
// <<<grid, block, smem, st>>> with the programmatic-stream-serialization attribute: the
// kernel may launch while its predecessor on the stream drains (each kernel waits on
// griddepcontrol.wait before touching global memory; pdl_entry in gbs_kernels.cuh).
template <typename... KArgs, typename... Args>
static void launch_k(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                     Args&&... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = GBS_PDL;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename K>
static void set_smem(K kernel, size_t bytes)
{
    if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// One-time setup per device and kernel: the dynamic shared-memory opt-in is a function
// attribute of the current device, so a process that sorts on several GPUs configures
// each of them (and caches the occupancy the setup returns per device).
constexpr int MAX_DEVICES = 64;
static int cur_device()
{
    int d = 0;
    cudaGetDevice(&d);
    return (d >= 0 ? d : 0) % MAX_DEVICES;
}
struct DevOnce {
    std::once_flag f[MAX_DEVICES];
    int val[MAX_DEVICES] = {};
    template <typename F>
    int run(F&& fn)
    {
        const int d = cur_device();
        std::call_once(f[d], [&] { val[d] = fn(); });
        return val[d];
    }
};
template <typename K>
static int occupancy(K kernel, int block, size_t smem)
{
    int occ = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, block, smem) != cudaSuccess || occ < 1) occ = 1;
    return occ;
}

template <int KIND, int BLOCK, int ITEMS>
static void launch_local_t(const LevelDev& lv0, cudaStream_t st)
{
    const size_t sm = Seg<KIND, BLOCK, ITEMS>::smem_bytes();
    static DevOnce once;
    const int occ = once.run([&] {
        set_smem(k_local_sort<KIND, BLOCK, ITEMS>, sm);
        return occupancy(k_local_sort<KIND, BLOCK, ITEMS>, BLOCK, sm);
    });
    // persistent: one CTA per resident slot, each walks tiles blockIdx.x + k*gridDim.x
    const unsigned grid = std::min<unsigned>(lv0.B * lv0.m, num_sms() * (unsigned)occ);
    launch_k(k_local_sort<KIND, BLOCK, ITEMS>, grid, BLOCK, sm, st, lv0);
}

template <int KIND, int BLOCK, int ITEMS, int MODE>
static void launch_seg_t(const LevelDev& lv, unsigned count, cudaStream_t st)
{
    // the fused Step 8+9 stages its run table (m + 1 uint2) behind the tile
    const size_t sm = MODE == MODE_GATHER
                          ? gather_smem_offset<KIND, BLOCK, ITEMS>() + ((size_t)gather_max_m(KIND) + 1) * 8
                          : Seg<KIND, BLOCK, ITEMS>::smem_bytes();
    static DevOnce once;
    once.run([&] {
        set_smem(k_segment_sort<KIND, BLOCK, ITEMS, MODE>, sm);
        return 1;
    });
    // one CTA per segment (for a size tier: per list slot, the unused tail exits at once)
    launch_k(k_segment_sort<KIND, BLOCK, ITEMS, MODE>, count, BLOCK, sm, st, lv);
}


#ifndef GBS_RARE_PERSIST
#define GBS_RARE_PERSIST 1   // Step 9's full-tile tier on persistent CTAs (k_segment_sort_rare)
#endif
template <int KIND, int BLOCK, int ITEMS, int MODE = MODE_BUCKET>
static void launch_rare_t(const LevelDev& lv, unsigned count, cudaStream_t st)
{
    const size_t sm = MODE == MODE_GATHER
                          ? gather_smem_offset<KIND, BLOCK, ITEMS>() + ((size_t)gather_max_m(KIND) + 1) * 8
                          : Seg<KIND, BLOCK, ITEMS>::smem_bytes();
    static DevOnce once;
    const int occ = once.run([&] {
        set_smem(k_segment_sort_rare<KIND, BLOCK, ITEMS, MODE>, sm);
        return occupancy(k_segment_sort_rare<KIND, BLOCK, ITEMS, MODE>, BLOCK, sm);
    });
    launch_k(k_segment_sort_rare<KIND, BLOCK, ITEMS, MODE>, std::min<unsigned>(count, num_sms() * (unsigned)occ), BLOCK,
             sm, st, lv);
}

// Step 2 on CTA pairs: persistent clusters of two (one CTA per SM)
static void launch_local_pair(const LevelDev& lv, cudaStream_t st)
{
    constexpr int BLOCK = GBS_KEYS_BLOCK, ITEMS = GBS_KEYS_ITEMS;
    const size_t sm = Seg<KIND_KEYS, BLOCK, ITEMS>::smem_bytes();
    static DevOnce once;
    once.run([&] {
        set_smem(k_local_sort_pair<BLOCK, ITEMS>, sm);
        return 1;
    });
    const unsigned pairs = std::min<unsigned>(lv.B * lv.m, num_sms() / 2);
    launch_k(k_local_sort_pair<BLOCK, ITEMS>, 2 * pairs, BLOCK, sm, st, lv);
}

// Step 9 on CTA pairs: one cluster of two per bucket slot, persistent (one CTA per SM)
static void launch_seg_pair(const LevelDev& lv, unsigned count, cudaStream_t st)
{
    constexpr int BLOCK = GBS_KEYS_BLOCK, ITEMS = GBS_KEYS_ITEMS;
    const size_t sm = Seg<KIND_KEYS, BLOCK, ITEMS>::smem_bytes();
    static DevOnce once;
    once.run([&] {
        set_smem(k_segment_sort_pair<BLOCK, ITEMS>, sm);
        return 1;
    });
    const unsigned pairs = std::min<unsigned>(count, num_sms() / 2);
    launch_k(k_segment_sort_pair<BLOCK, ITEMS>, 2 * pairs, BLOCK, sm, st, lv);
}

template <int KIND>
static void launch_local(const LevelDev& lv, bool small, cudaStream_t st)
{
    if (small) launch_local_t<KIND, GBS_SMALL>(lv, st);
    else if constexpr (KIND == KIND_KEYS) launch_local_t<KIND, GBS_BIG_KEYS>(lv, st);
    else if constexpr (KIND == KIND_PAIRS) launch_local_t<KIND, GBS_PAIRS_LOCAL>(lv, st);
    else launch_local_t<KIND, GBS_BIG_WIDE>(lv, st);
}

template <int KIND, int MODE>
static void launch_seg(const LevelDev& lv, bool small, unsigned grid, cudaStream_t st)
{
    if (small) launch_seg_t<KIND, GBS_SMALL, MODE>(lv, grid, st);
    else if constexpr (KIND == KIND_KEYS) launch_seg_t<KIND, GBS_BIG_KEYS, MODE>(lv, grid, st);
    else launch_seg_t<KIND, BIGB(KIND), BIGI(KIND), MODE>(lv, grid, st);
}

template <int KIND>
static void launch_index(const LevelDev& lv, cudaStream_t st)
{
    const size_t kb = key_bytes(KIND);
    // streaming TMA form (any item alignment: misaligned chunk starts are copied from the
    // 16-byte boundary below)
    const bool tma = GBS_IDX_TMA && (kb == 4 || kb == 8) && lv.s <= 8 * IDX_BLOCK;
    if (tma) {
        const size_t sm = 2 * ((size_t)IDX_CHUNK_BYTES + 16) + (size_t)lv.s * 12;
        static DevOnce once;
        const int occ = once.run([&] {
            set_smem(k_sample_index_tma<KIND, IDX_BLOCK, 8>, 220 * 1024);
            // occupancy at the largest table this kernel sees (s <= 4096)
            return occupancy(k_sample_index_tma<KIND, IDX_BLOCK, 8>, IDX_BLOCK, 2 * ((size_t)IDX_CHUNK_BYTES + 16) + 4096 * 12);
        });
        const unsigned grid = std::min<unsigned>(lv.B * lv.m, num_sms() * (unsigned)occ);
        launch_k(k_sample_index_tma<KIND, IDX_BLOCK, 8>, grid, IDX_BLOCK, sm, st, lv);
        return;
    }
    const size_t chunk = std::min<size_t>((size_t)lv.L * key_bytes(KIND), IDX_CHUNK_BYTES);
    const size_t sm = (size_t)lv.s * 8 + (size_t)(lv.s + (lv.s & 1)) * 4 + chunk;
    static DevOnce once;
    once.run([&] {
        set_smem(k_sample_index<KIND, IDX_BLOCK>, 227 * 1024);
        return 1;
    });
    launch_k(k_sample_index<KIND, IDX_BLOCK>, lv.B * lv.m, IDX_BLOCK, sm, st, lv);
}

// Step 8 grouped by destination: sublists per group, per item kind (0 = one CTA per
// sublist, k_relocate).  Measured: keys 8 (C2 Step 8 0.105 -> 0.085 ms, C3 0.258 ->
// 0.159); pairs and the u64 sample levels measured slower grouped (C4; m = 128 at C2).
#ifndef GBS_RELOC_GROUP_KEYS
#define GBS_RELOC_GROUP_KEYS 8
#endif
#ifndef GBS_RELOC_GROUP_PAIRS
#define GBS_RELOC_GROUP_PAIRS 0
#endif
#ifndef GBS_RELOC_GROUP_U64
#define GBS_RELOC_GROUP_U64 0
#endif
static int reloc_launches(int kind)
{
    const int g = kind == KIND_KEYS ? GBS_RELOC_GROUP_KEYS : (kind == KIND_PAIRS ? GBS_RELOC_GROUP_PAIRS : GBS_RELOC_GROUP_U64);
    return g > 0 ? 2 : 1;
}
template <int KIND>
static void launch_relocate(const LevelDev& lv, cudaStream_t st)
{
    constexpr int GROUP = KIND == KIND_KEYS ? GBS_RELOC_GROUP_KEYS
                                            : (KIND == KIND_PAIRS ? GBS_RELOC_GROUP_PAIRS : GBS_RELOC_GROUP_U64);
    if constexpr (GROUP > 0) {
        if (lv.pex && lv.maxrun) {
            // Both forms are launched; each reads Step 7's longest run and one exits at
            // once: grouped by destination when runs are short (spread inputs), one CTA
            // per sublist when some run is long (sorted / clustered inputs), where the
            // grouped form would leave whole buckets to single warps (R21).
            constexpr int G = GROUP, BLOCK = 256, JB = 64;
            const unsigned grid = lv.B * ((lv.m + G - 1) / G) * ((lv.s + JB - 1) / JB);
            launch_k(k_relocate_grouped<KIND, BLOCK, G, JB>, grid, BLOCK, 0, st, lv);
        }
    }
    constexpr int MAXPER = (int)(tile_of_c(KIND) / IDX_BLOCK);
    const size_t per = std::max<size_t>(1, lv.L / IDX_BLOCK);
    const size_t sm = (size_t)2 * lv.s * 4 + (lv.L + 2 * (lv.L / per) + 4) * 2;
    static DevOnce once;
    once.run([&] {
        set_smem(k_relocate<KIND, IDX_BLOCK, MAXPER>, 220 * 1024);
        return 1;
    });
    LevelDev lr = lv;   // the per-sublist form defers to the grouped one only if that was launched
    if (!(GROUP > 0 && lv.pex)) lr.maxrun = nullptr;
    launch_k(k_relocate<KIND, IDX_BLOCK, MAXPER>, lv.B * lv.m, IDX_BLOCK, sm, st, lr);
}

static uint32_t num_sms()
{
    static DevOnce once;
    return (uint32_t)once.run([] {
        int n = 0, dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        return n;
    });
}

// A second stream per device for work that runs beside the call's stream inside one
// step (fork/join through events, so the call stays ordered on the caller's stream;
// capturable into a CUDA graph).  Shared by concurrent calls: that only serialises the
// side work, the dependencies stay per call.
// Side streams per calling thread and device (like the scratch events): calls from
// different threads never share one, so a call being captured into a graph (the caller's
// capture, or the library's own for latency-bound sizes) cannot pull another thread's
// work into it.
static cudaStream_t side_stream(int k = 0)   // k: 0 = Step 9 tiers, 1 = H2D, 2 = D2H, 3 = more Step 9 tiers
{
    static thread_local cudaStream_t ss[MAX_DEVICES][4] = {};
    const int dev = cur_device();
    if (k < 0 || k > 3) return nullptr;
    if (!ss[dev][k] && cudaStreamCreateWithFlags(&ss[dev][k], cudaStreamNonBlocking) != cudaSuccess) ss[dev][k] = nullptr;
    return ss[dev][k];
}

// Events for fork/join inside one call, created once per thread and device and reused:
// cudaStreamWaitEvent waits for the record that precedes it, so a later re-record of the
// same event (next chunk, next call) does not affect an earlier wait.
static cudaEvent_t scratch_event(int k)
{
    static thread_local cudaEvent_t ev[MAX_DEVICES][8] = {};
    const int d = cur_device();
    if (!ev[d][k] && cudaEventCreateWithFlags(&ev[d][k], cudaEventDisableTiming) != cudaSuccess) ev[d][k] = nullptr;
    return ev[d][k];
}

// Host-buffer calls (gbs_sort_keys_host): the H2D copy is split into chunks of sublists
// and Step 2 sorts each chunk as it lands; Step 9 runs in groups of buckets and each
// group's final output range is copied back while the next groups sort.
struct HostPipe {
    uint32_t* h;              // pinned host keys (in and out)
    uint32_t* hv;             // pinned host values (pairs) or nullptr
    size_t n;
    cudaStream_t cin, cout;   // copy streams
};
#ifndef GBS_HOST_PIPE
#define GBS_HOST_PIPE 1
#endif
constexpr uint32_t HP_CHUNK_TILES = 64;   // sublists per H2D chunk (8 MB of keys)
constexpr uint32_t HP_GROUPS = 16;        // Step 9 bucket groups (D2H chunks)
#ifndef GBS_HP_NEST_GROUPS
#define GBS_HP_NEST_GROUPS 32  // groups of a nested Step 9's problems (D2H chunks): C4 e2e 8 -> 32: 337 -> 326 ms
#endif
constexpr uint32_t HP_NEST_GROUPS = GBS_HP_NEST_GROUPS;

struct Bufs {
    void *in, *reloc, *out;
    uint32_t *in_v, *reloc_v, *out_v;
    // out-of-place sorts (keys): where Step 2 writes the sorted sublists (in stays
    // read-only); null = in place (in)
    void* srt = nullptr;
    // typed keys: transform at the first level's loads / the last level's stores
    int xf_in = 0, xf_out = 0;
    // nested level: per problem, the samples of its non-empty sublists (Step 4 sorts these)
    const uint32_t* scnt = nullptr;
};

// A window of a node's problems: [b0, b0 + bn) (bn = 0: all B).  Bufs / Probs passed to
// exec describe all B problems; exec_kind offsets them and the node's own per-problem
// workspace arrays by b0, and a nested child's window is [b0 s, (b0 + bn) s).  Used by
// the host-pipelined call to finish a nested level in groups of problems, so that the
// D2H copy of each group's final output overlaps the next groups' sorts.
struct Win {
    uint32_t b0 = 0, bn = 0;
};

template <int KIND>
static gbs_status_t exec_kind(const Plan& P, int ni, char* ws, const Bufs& bf, Probs pr, cudaStream_t st, int stop,
                              const HostPipe* hp, Win win);

static gbs_status_t exec(const Plan& P, int ni, char* ws, const Bufs& bf, Probs pr, cudaStream_t st, int stop,
                         const HostPipe* hp = nullptr, Win win = Win())
{
    switch (P.nodes[ni].kind) {
        case KIND_KEYS: return exec_kind<KIND_KEYS>(P, ni, ws, bf, pr, st, stop, hp, win);
        case KIND_PAIRS: return exec_kind<KIND_PAIRS>(P, ni, ws, bf, pr, st, stop, hp, win);
        default: return exec_kind<KIND_U64>(P, ni, ws, bf, pr, st, stop, hp, win);
    }
}

// Step 4 as a merge tree (R22): the m runs of s samples -> runs of TILE_U64 on chip, pair
// levels to two runs, then the s splitters by selection (full: the last level merges
// everything, for stage parity of the sorted samples).  The last level reads the tmp
// buffer and writes the samples array, so the tile merge starts on whichever buffer makes
// the G pair levels end in tmp.
static gbs_status_t launch_s4_tree(const Node& nd, const LevelDev& lv, char* ws, cudaStream_t st, bool full)
{
    constexpr int KIND = KIND_U64;   // (GBS_LAUNCHED reports the node kind)
    constexpr int TB = GBS_S4_TILE_BLOCK, TI = 16, TILE = TB * TI;
    const uint32_t N = nd.m * nd.s;
    u64* S = lv.samples;
    u64* T = reinterpret_cast<u64*>(ws + nd.o_s4tmp);
    u64* cur = (nd.s4_levels % 2 == 0) ? T : S;
    u64* oth = cur == T ? S : T;
    const size_t sm = sizeof(u64) * CtaSort<unsigned long long, TB, TI>::SMEM_ELEMS;
    static DevOnce once;
    once.run([&] {
        set_smem(k_s4_tile<TB, TI>, sm);
        return 1;
    });
    launch_k(k_s4_tile<TB, TI>, (N + TILE - 1) / TILE, TB, sm, st, (const u64*)S, cur, N, nd.s);
    GBS_LAUNCHED();
    constexpr uint32_t TO = S4_MERGE_BLOCK * S4_MERGE_ITEMS;
    const unsigned mgrid = (N + TO - 1) / TO;
    uint32_t R = TILE;
    for (int g = 0; g < nd.s4_levels; ++g, R *= 2) {
        launch_k(k_s4_merge<S4_MERGE_BLOCK, S4_MERGE_ITEMS>, mgrid, S4_MERGE_BLOCK, 0, st, (const u64*)cur, oth, N, R);
        GBS_LAUNCHED();
        std::swap(cur, oth);
    }
    if (cur != T) return fail(GBS_ERROR_CUDA, "internal: merge tree parity");
    if (full) launch_k(k_s4_merge<S4_MERGE_BLOCK, S4_MERGE_ITEMS>, mgrid, S4_MERGE_BLOCK, 0, st, (const u64*)T, S, N, R);
    else launch_k(k_s4_select, (nd.s * 32 + 255) / 256, 256, 0, st, (const u64*)T, S, N, R, nd.m, nd.s);
    GBS_LAUNCHED();
    return GBS_SUCCESS;
}

// Step 9 over CTA buckets: one launch, or the size tiers (MODE_BUCKET reads the
// relocated buckets, MODE_GATHER gathers them from the sorted sublists)
template <int KIND, int MODE>
static gbs_status_t launch_step9(const LevelDev& lv, const Node& nd, char* ws, cudaStream_t st)
{
    {
        constexpr uint32_t TILE = tile_of_c(KIND);
        constexpr int ITEMS = KIND == KIND_KEYS ? GBS_KEYS_ITEMS : GBS_WIDE_ITEMS;
        if (GBS_SPLIT_STEP9_ON && split_step9(KIND, nd)) {
            // Size tiers: buckets of at most half a tile on 512-thread CTAs (2 per SM:
            // one's load/store phases overlap the other's sort); those a little over half
            // a tile (common: the average bucket n/s is about half the tight bound) on a
            // 5/8-tile configuration (keys: 512 threads, still 2 CTAs per SM); the rare
            // larger ones on the full tile.  Each tier launches over its list (built by
            // k_bucket_tiers).
            const uint32_t count = lv.B * nd.s;
            uint32_t* lists = reinterpret_cast<uint32_t*>(ws + nd.o_tiers);
            uint32_t* lens = lists + 4 * (uint64_t)count;
            uint32_t cuts[3];
            tier_cuts(KIND, nd, TILE, cuts);
            GBS_CUDA(cudaMemsetAsync(lens, 0, 16, st));
            launch_k(k_bucket_tiers, (count + 255) / 256, 256, 0, st, lv, lists, lens, cuts[0], cuts[1], cuts[2]);
            GBS_LAUNCHED();
            LevelDev tl[4];
            for (int q = 0; q < 4; ++q) {
                tl[q] = lv;
                tl[q].tier_list = lists + q * (uint64_t)count;
                tl[q].tier_len = lens + q;
            }
            // The tiers run concurrently: the larger tiers (few CTAs, each a full-tile
            // sort) on the side stream, so they are not a serial tail after tier 0.
            // (tier 1 on one side stream; tiers 2 and 3 -- usually empty -- on another)
            cudaStream_t ss = side_stream(), ss2 = side_stream(3);
            cudaEvent_t fork = scratch_event(0), join = scratch_event(1), join2 = scratch_event(2);
            if (ss && ss2 && fork && join && join2) {
                GBS_CUDA(cudaEventRecord(fork, st));
                GBS_CUDA(cudaStreamWaitEvent(ss, fork, 0));
                GBS_CUDA(cudaStreamWaitEvent(ss2, fork, 0));
            } else {
                ss = ss2 = nullptr;
            }
            cudaStream_t s12 = ss ? ss : st, s23 = ss2 ? ss2 : st;
            if (GBS_MID_STEP9) {
                if (nd.hi > cuts[2]) {   // the full tile
                    if constexpr (GBS_RARE_PERSIST) {
                        if constexpr (KIND == KIND_KEYS) launch_rare_t<KIND, GBS_BIG_KEYS, MODE>(tl[3], count, s23);
                        else launch_rare_t<KIND, BIGB(KIND), BIGI(KIND), MODE>(tl[3], count, s23);
                    } else {
                        if constexpr (KIND == KIND_KEYS) launch_seg_t<KIND, GBS_BIG_KEYS, MODE>(tl[3], count, s23);
                        else launch_seg_t<KIND, BIGB(KIND), BIGI(KIND), MODE>(tl[3], count, s23);
                    }
                    GBS_LAUNCHED();
                }
                bool mid_done = false;
                if constexpr (KIND == KIND_KEYS) {
                    if (nd.B != 1) {   // nested: a sparse tier (see below)
                        if (GBS_RARE_PERSIST) launch_rare_t<KIND, 512, GBS_MID_KEYS_ITEMS_NESTED, MODE>(tl[1], count, s12);
                        else launch_seg_t<KIND, 512, GBS_MID_KEYS_ITEMS_NESTED, MODE>(tl[1], count, s12);
                        mid_done = true;
                    } else if (nd.hi > cuts[1] && cuts[2] > cuts[1]) {
                        // the second mid tier on persistent CTAs (usually few buckets)
                        if constexpr (MODE == MODE_BUCKET) launch_rare_t<KIND, 512, GBS_MID2_TOP_ITEMS>(tl[2], count, s23);
                        else launch_seg_t<KIND, 512, GBS_MID2_TOP_ITEMS, MODE>(tl[2], count, s23);
                        GBS_LAUNCHED();
                    }
                }
                if (!mid_done) {
                    // nested levels: buckets average a quarter of the bound, so the mid tier
                    // is sparse -> persistent CTAs over its list
                    if (nd.B != 1 && GBS_RARE_PERSIST)
                        launch_rare_t<KIND, MID_BLOCK_OF(KIND), MID_ITEMS_OF(KIND), MODE>(tl[1], count, s12);
                    else
                        launch_seg_t<KIND, MID_BLOCK_OF(KIND), MID_ITEMS_OF(KIND), MODE>(tl[1], count, s12);
                }
                GBS_LAUNCHED();
            } else {   // no mid tier: (C/2, C] on the full tile
                if constexpr (KIND == KIND_KEYS) launch_seg_t<KIND, GBS_BIG_KEYS, MODE>(tl[1], count, s12);
                else launch_seg_t<KIND, BIGB(KIND), BIGI(KIND), MODE>(tl[1], count, s12);
                GBS_LAUNCHED();
            }
            // (pairs on 256 x 32 instead: C4 78.8 -> 81.7 ms)
            if constexpr (KIND == KIND_PAIRS)
                launch_seg_t<KIND, GBS_PAIRS_T0_BLOCK, GBS_PAIRS_T0_ITEMS, MODE>(tl[0], count, st);
            else
                launch_seg_t<KIND, 512, ITEMS, MODE>(tl[0], count, st);
            GBS_LAUNCHED();
            if (ss) {
                GBS_CUDA(cudaEventRecord(join, ss));
                GBS_CUDA(cudaEventRecord(join2, ss2));
                GBS_CUDA(cudaStreamWaitEvent(st, join, 0));
                GBS_CUDA(cudaStreamWaitEvent(st, join2, 0));
            }
        } else {
            launch_seg<KIND, MODE>(lv, nd.bucket_small, lv.B * nd.s, st);
        }
        GBS_LAUNCHED();
    }
    return GBS_SUCCESS;
}

// Step 9 of a level with two-tile buckets (keys): size tiers so a bucket takes the
// smallest unit that holds it -- <= C/2 on 512-thread CTAs (2 per SM), <= C on one full
// CTA, larger on a CTA pair (k_segment_sort_pair) -- all three concurrently (fork/join).
// (One CTA pair per bucket measured 25.2 Gkeys/s at 2^27 against 26.8 for the nested
// plan: the average bucket, n/s = C, half-fills a pair.)
static gbs_status_t launch_step9_pair(const LevelDev& lv, const Node& nd, char* ws, cudaStream_t st)
{
    constexpr int KIND = KIND_KEYS;
    const uint32_t count = lv.B * nd.s;
    uint32_t* lists = reinterpret_cast<uint32_t*>(ws + nd.o_tiers);
    uint32_t* lens = lists + 4 * (uint64_t)count;
    GBS_CUDA(cudaMemsetAsync(lens, 0, 16, st));
    launch_k(k_bucket_tiers, (count + 255) / 256, 256, 0, st, lv, lists, lens, TILE_KEYS / 2, TILE_KEYS, TILE_KEYS);
    GBS_LAUNCHED();
    LevelDev tl[4];
    for (int q = 0; q < 4; ++q) {
        tl[q] = lv;
        tl[q].tier_list = lists + q * (uint64_t)count;
        tl[q].tier_len = lens + q;
    }
    cudaStream_t ss = side_stream(), ss2 = side_stream(3);
    cudaEvent_t fork = scratch_event(0), join = scratch_event(1), join2 = scratch_event(2);
    if (ss && ss2 && fork && join && join2) {
        GBS_CUDA(cudaEventRecord(fork, st));
        GBS_CUDA(cudaStreamWaitEvent(ss, fork, 0));
        GBS_CUDA(cudaStreamWaitEvent(ss2, fork, 0));
    } else {
        ss = ss2 = nullptr;
    }
    launch_seg_pair(tl[3], count, ss2 ? ss2 : st);
    GBS_LAUNCHED();
    launch_seg_t<KIND, GBS_BIG_KEYS, MODE_BUCKET>(tl[1], count, ss ? ss : st);
    GBS_LAUNCHED();
    launch_seg_t<KIND, 512, GBS_KEYS_ITEMS, MODE_BUCKET>(tl[0], count, st);
    GBS_LAUNCHED();
    if (ss) {
        GBS_CUDA(cudaEventRecord(join, ss));
        GBS_CUDA(cudaEventRecord(join2, ss2));
        GBS_CUDA(cudaStreamWaitEvent(st, join, 0));
        GBS_CUDA(cudaStreamWaitEvent(st, join2, 0));
    }
    return GBS_SUCCESS;
}

template <int KIND>
static gbs_status_t exec_kind(const Plan& P, int ni, char* ws, const Bufs& bf_all, Probs pr, cudaStream_t st,
                              int stop, const HostPipe* hp, Win win)
{
    const Node& nd = P.nodes[ni];
    // the window: problems [b0, b0 + B) of the node (everything indexed by problem is
    // offset by b0 below; kernels index problems relative to it)
    const uint32_t b0 = win.b0, B = win.bn ? win.bn : nd.B;
    Bufs bf = bf_all;
    if (b0) {
        if (pr.off) pr.off += b0;
        if (pr.len) pr.len += b0;
        if (!pr.off) {   // contiguous problems: the data pointers move
            const size_t o = (size_t)b0 * pr.stride;
            auto mv = [o](void* p, size_t eb) { return p ? (void*)((char*)p + o * eb) : p; };
            const size_t kb = key_bytes(KIND);
            bf.in = mv(bf.in, kb);
            bf.reloc = mv(bf.reloc, kb);
            bf.out = mv(bf.out, kb);
            bf.srt = mv(bf.srt, kb);
            bf.in_v = (uint32_t*)mv(bf.in_v, 4);
            bf.reloc_v = (uint32_t*)mv(bf.reloc_v, 4);
            bf.out_v = (uint32_t*)mv(bf.out_v, 4);
        }
        if (bf.scnt) bf.scnt += b0;
    }
    LevelDev lv;
    memset(&lv, 0, sizeof lv);
    lv.pr = pr;
    lv.B = B;
    lv.N = (uint32_t)nd.N;
    lv.pad_base = nd.pad_base;
    lv.in = bf.in;
    lv.reloc = bf.reloc;
    lv.out = bf.out;
    lv.in_v = bf.in_v;
    lv.reloc_v = bf.reloc_v;
    lv.out_v = bf.out_v;
    lv.pf_stride = num_sms();
    lv.presorted = pr.presorted;
    lv.xf_in = bf.xf_in;
    lv.xf_out = (nd.leaf || nd.step9 < 0) ? bf.xf_out : 0;
    lv.seg_min = 0;
    lv.seg_max = 0xFFFFFFFFu;
    if (nd.leaf) {
        launch_seg<KIND, MODE_LEAF>(lv, nd.small, B, st);
        GBS_LAUNCHED();
        return GBS_SUCCESS;
    }
    lv.L = nd.L;
    lv.s = nd.s;
    lv.d = nd.d;
    lv.m = nd.m;
    const uint64_t ms = (uint64_t)nd.m * nd.s, nblk = (nd.s + 31) / 32;
    lv.samples = reinterpret_cast<u64*>(ws + nd.o_samples) + b0 * ms;
    lv.splitters = reinterpret_cast<u64*>(ws + nd.o_splitters) + (uint64_t)b0 * nd.s;
    lv.a = reinterpret_cast<uint32_t*>(ws + nd.o_a) + b0 * ms;
    lv.l = reinterpret_cast<uint32_t*>(ws + nd.o_l) + b0 * ms;
    lv.state = reinterpret_cast<unsigned long long*>(ws + nd.o_state) + b0 * nblk;
    // the longest-run word (Step 7 -> Step 8) follows the look-back words of all B problems
    uint32_t* maxrun = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned long long*>(ws + nd.o_state) + nd.B * nblk);
    // fused Step 8+9: Step 2 must not sort in place when the output is the input (the
    // bucket CTAs would overwrite runs other CTAs still gather), so it writes the sorted
    // sublists to the reloc buffer, which Step 8 no longer needs
    const bool fuse = nd.fuse89 && stop == 0 && !hp;
    const HostPipe* hp9 = (hp && stop == 0) ? hp : nullptr;   // D2H under a nested Step 9 (top level)
    lv.srt = bf.srt ? bf.srt : lv.in;
    lv.srt_v = lv.in_v;
    lv.pex = reinterpret_cast<uint32_t*>(ws + nd.o_pex) + b0 * ms;
    if (fuse && lv.srt == lv.out) {
        lv.srt = lv.reloc;
        lv.srt_v = lv.reloc_v;
    }
    ProfMarks pm;
    if (g_prof && nd.level >= 0 && nd.level < GBS_MAX_LEVELS && stop == 0) {
        ProfCall pc;
        pc.level = nd.level;
        for (auto& e : pc.ev) cudaEventCreate(&e);
        g_prof_calls.push_back(pc);
        pm.ev = g_prof_calls.back().ev.data();
        pm.st = st;
    }
    // zero Step 7's look-back words and its longest-run word before the level's first
    // kernel, where the memset delays nothing (between Steps 6 and 7 it would)
    if (B == nd.B) {   // the look-back words and the longest-run word are contiguous
        GBS_CUDA(cudaMemsetAsync(lv.state, 0, (size_t)B * nblk * 8 + 8, st));
    } else {
        GBS_CUDA(cudaMemsetAsync(lv.state, 0, (size_t)B * nblk * 8, st));
        GBS_CUDA(cudaMemsetAsync(maxrun, 0, 8, st));
    }
    pm.mark();

    // Steps 2-3: local sort + local samples (one CTA per sublist)
    if (hp) {
        // chunk c of sublists is copied in on hp->cin, then sorted on st
        cudaEvent_t ev = scratch_event(3);
        if (!ev) return fail(GBS_ERROR_CUDA, "cannot create an event");
        GBS_CUDA(cudaEventRecord(ev, st));                  // d_keys free (earlier work on st)
        GBS_CUDA(cudaStreamWaitEvent(hp->cin, ev, 0));
        uint32_t* dk = reinterpret_cast<uint32_t*>(lv.in);
        for (uint32_t t0 = 0; t0 < nd.m; t0 += HP_CHUNK_TILES) {
            const uint32_t t1 = std::min(nd.m, t0 + HP_CHUNK_TILES);
            const size_t e0 = (size_t)t0 * nd.L, e1 = std::min(hp->n, (size_t)t1 * nd.L);
            GBS_CUDA(cudaMemcpyAsync(dk + e0, hp->h + e0, (e1 - e0) * 4, cudaMemcpyHostToDevice, hp->cin));
            if (hp->hv)
                GBS_CUDA(cudaMemcpyAsync(lv.in_v + e0, hp->hv + e0, (e1 - e0) * 4, cudaMemcpyHostToDevice, hp->cin));
            GBS_CUDA(cudaEventRecord(ev, hp->cin));
            GBS_CUDA(cudaStreamWaitEvent(st, ev, 0));
            LevelDev lc = lv;
            lc.tile_lo = t0;
            lc.tile_hi = t1;
            if (nd.local_pair) launch_local_pair(lc, st);
            else launch_local<KIND>(lc, nd.local_small, st);
            GBS_LAUNCHED();
        }
    } else {
        if (nd.local_pair) launch_local_pair(lv, st);
        else launch_local<KIND>(lv, nd.local_small, st);
        GBS_LAUNCHED();
    }
    if (stop == 2 || stop == 3) return GBS_SUCCESS;
    pm.mark();

    // Step 4: sort the B*m*s samples = a U64 level on B problems of m*s composites, or
    // (one problem, L2-resident samples) a merge tree of the m presorted runs of s
    if (nd.s4_tree) {
        gbs_status_t r = launch_s4_tree(nd, lv, ws, st, stop == 4 || stop == 5);
        if (r) return r;
    } else {
        const Node& c = P.nodes[nd.step4];
        // (all B problems' arrays; the child applies this window to them)
        u64* smp_all = reinterpret_cast<u64*>(ws + nd.o_samples);
        Bufs b4{smp_all, c.leaf ? (void*)smp_all : (void*)(ws + c.o_reloc), smp_all, nullptr, nullptr, nullptr};
        // each sublist's s samples are sorted and contiguous: runs of length s
        // (a nested level sorts only the samples of each problem's non-empty sublists: the
        // rest are virtual sentinels already in their sorted places, k_child_desc)
        Probs p4{nullptr, bf_all.scnt, (uint64_t)nd.m * nd.s, nd.m * nd.s, nd.s};
        gbs_status_t r = exec(P, nd.step4, ws, b4, p4, st, 0, nullptr, Win{b0, B});
        if (r) return r;
    }
    if (stop == 4) return GBS_SUCCESS;
    pm.mark();

    // Step 5 (global samples) is fused into Step 6's prologue; the stand-alone kernel
    // runs only when a caller stops right after Step 5 (stage parity).
    if (stop == 5) {
        const uint64_t tot = (uint64_t)B * nd.s;
        launch_k(k_global_samples, (unsigned)((tot + 255) / 256), 256, 0, st, lv);
        GBS_LAUNCHED();
        return GBS_SUCCESS;
    }
    pm.mark();

    // Steps 5-6: sample indexing -> a
    launch_index<KIND>(lv, st);
    GBS_LAUNCHED();
    if (debug_sync()) {   // invariants of Steps 4 and 6 (debugging only)
        unsigned* dflag = nullptr;
        GBS_CUDA(cudaMallocManaged(&dflag, 8 * sizeof(unsigned)));
        memset(dflag, 0, 8 * sizeof(unsigned));
        launch_k(k_check_level, 1024, 256, 0, st, lv, dflag, (int)(nd.s4_tree && !(stop == 4 || stop == 5)));
        GBS_CUDA(cudaStreamSynchronize(st));
        unsigned fl[8];
        memcpy(fl, dflag, sizeof fl);
        cudaFree(dflag);
        if (fl[0])
            return fail(GBS_ERROR_CUDA, "invariant check failed (flag %u: 1 = samples unsorted, 2 = a rows) at node "
                        "%d kind %d B %u N %llu L %u s %u m %u; first bad row b %u i %u sum %u v %u len %u "
                        "g_last %08x:%08x", fl[0], ni, KIND, nd.B, (unsigned long long)nd.N, nd.L, nd.s, nd.m,
                        fl[1], fl[2], fl[3], fl[4], fl[5], fl[6], fl[7]);
    }
    if (stop == 6) return GBS_SUCCESS;
    pm.mark();

    // Step 7: column-major exclusive scan -> l
    lv.maxrun = maxrun;
    launch_k(k_scan, B * (unsigned)nblk, SCAN_BLOCK, 0, st, lv);
    GBS_LAUNCHED();
    if (stop == 7) return GBS_SUCCESS;
    pm.mark();

    // Step 8: relocation in -> reloc (fused into Step 9 on the production path)
    if (!fuse) {
        launch_relocate<KIND>(lv, st);
        GBS_LAUNCHED();
    }
    if (stop == 8) return GBS_SUCCESS;
    pm.mark();

    // Step 9: bucket sort reloc -> out (one CTA per bucket) or a nested level
    if (hp && nd.step9 < 0) {
        // groups of buckets; after buckets [0, j1) are sorted, the output prefix
        // [0, j1 m d - V) is final: exactly j1 m samples are <= g_{j1-1}, and a sublist
        // with c samples <= g has >= c d items <= g, so >= j1 m d items (V of them
        // possibly virtual, V = m L - n) fall in buckets < j1 (Alg. 1 Steps 3-5)
        const uint64_t V = (uint64_t)nd.m * nd.L - hp->n;
        const uint32_t G = std::max(1u, nd.s / HP_GROUPS);
        uint64_t done = 0;
        cudaEvent_t ev = scratch_event(4);
        if (!ev) return fail(GBS_ERROR_CUDA, "cannot create an event");
        for (uint32_t j0 = 0; j0 < nd.s; j0 += G) {
            const uint32_t j1 = std::min(nd.s, j0 + G);
            LevelDev lg = lv;
            lg.seg_lo = j0;
            lg.seg_hi = j1;
            if (nd.bucket_pair) {
                if constexpr (KIND == KIND_KEYS) launch_seg_pair(lg, j1 - j0, st);
            } else {
                launch_seg<KIND, MODE_BUCKET>(lg, nd.bucket_small, j1 - j0, st);
            }
            GBS_LAUNCHED();
            const uint64_t lo_cnt = (uint64_t)j1 * nd.m * nd.d;
            const uint64_t upto = j1 == nd.s ? hp->n : std::min<uint64_t>(hp->n, lo_cnt > V ? lo_cnt - V : 0);
            if (upto > done) {
                GBS_CUDA(cudaEventRecord(ev, st));
                GBS_CUDA(cudaStreamWaitEvent(hp->cout, ev, 0));
                GBS_CUDA(cudaMemcpyAsync(hp->h + done, reinterpret_cast<uint32_t*>(lv.out) + done, (upto - done) * 4,
                                         cudaMemcpyDeviceToHost, hp->cout));
                if (hp->hv)
                    GBS_CUDA(cudaMemcpyAsync(hp->hv + done, lv.out_v + done, (upto - done) * 4, cudaMemcpyDeviceToHost,
                                             hp->cout));
                done = upto;
            }
        }
        GBS_CUDA(cudaEventRecord(ev, hp->cout));
        GBS_CUDA(cudaStreamWaitEvent(st, ev, 0));          // the call completes on st
    } else if (nd.bucket_pair) {
        if constexpr (KIND == KIND_KEYS) {
            gbs_status_t r9 = launch_step9_pair(lv, nd, ws, st);
            if (r9) return r9;
        }
    } else if (nd.step9 < 0) {
        gbs_status_t r9;
        if constexpr (KIND == KIND_KEYS || (KIND == KIND_PAIRS && GBS_FUSE_PAIRS))
            r9 = fuse ? launch_step9<KIND, MODE_GATHER>(lv, nd, ws, st) : launch_step9<KIND, MODE_BUCKET>(lv, nd, ws, st);
        else
            r9 = launch_step9<KIND, MODE_BUCKET>(lv, nd, ws, st);
        if (r9) return r9;
    } else {
        // the nested problems of this window: [b0 s, (b0 + B) s)
        u64* coff = reinterpret_cast<u64*>(ws + nd.o_child_off);
        uint32_t* clen = reinterpret_cast<uint32_t*>(ws + nd.o_child_len);
        lv.child_off = coff + (uint64_t)b0 * nd.s;
        lv.child_len = clen + (uint64_t)b0 * nd.s;
        const uint64_t tot = (uint64_t)B * nd.s;
        const Node& ch = P.nodes[nd.step9];
        uint32_t* scnt = (!ch.leaf && ch.step4 >= 0) ? reinterpret_cast<uint32_t*>(ws + nd.o_child_scnt) : nullptr;
        launch_k(k_child_desc, (unsigned)((tot + 255) / 256), 256, 0, st, lv, scnt ? scnt + (uint64_t)b0 * nd.s : nullptr,
                 ch.L, ch.s);
        GBS_LAUNCHED();
        // the nested level sorts its problems in place in the reloc buffer and uses the
        // sublists' buffer (dead after Step 8) as its own relocation target
        Bufs b9{bf.reloc, bf.srt ? bf.srt : bf.in, bf.out, bf.reloc_v, bf.in_v, bf.out_v};
        b9.xf_out = bf.xf_out;   // the keys entered the sort at this level's Step 2
        b9.scnt = scnt;
        Probs p9{coff, clen, 0, 0};
        gbs_status_t r = GBS_SUCCESS;
        if (hp9) {
            // host-pipelined call: the nested level in groups of this level's buckets; once
            // buckets [0, j1) are sorted, the output prefix [0, j1 m d - V) is final (R18),
            // and its D2H copy overlaps the next groups
            const uint64_t V = (uint64_t)nd.m * nd.L - hp9->n;
            const uint32_t G = std::max(1u, nd.s / HP_NEST_GROUPS);
            uint64_t done = 0;
            cudaEvent_t ev = scratch_event(4);
            if (!ev) return fail(GBS_ERROR_CUDA, "cannot create an event");
            for (uint32_t j0 = 0; j0 < nd.s; j0 += G) {
                const uint32_t j1 = std::min(nd.s, j0 + G);
                r = exec(P, nd.step9, ws, b9, p9, st, 0, nullptr, Win{j0, j1 - j0});
                if (r) return r;
                const uint64_t lo_cnt = (uint64_t)j1 * nd.m * nd.d;
                const uint64_t upto = j1 == nd.s ? hp9->n : std::min<uint64_t>(hp9->n, lo_cnt > V ? lo_cnt - V : 0);
                if (upto > done) {
                    GBS_CUDA(cudaEventRecord(ev, st));
                    GBS_CUDA(cudaStreamWaitEvent(hp9->cout, ev, 0));
                    GBS_CUDA(cudaMemcpyAsync(hp9->h + done, reinterpret_cast<uint32_t*>(bf.out) + done,
                                             (upto - done) * 4, cudaMemcpyDeviceToHost, hp9->cout));
                    if (hp9->hv)
                        GBS_CUDA(cudaMemcpyAsync(hp9->hv + done, bf.out_v + done, (upto - done) * 4,
                                                 cudaMemcpyDeviceToHost, hp9->cout));
                    done = upto;
                }
            }
            GBS_CUDA(cudaEventRecord(ev, hp9->cout));
            GBS_CUDA(cudaStreamWaitEvent(st, ev, 0));      // the call completes on st
        } else {
            r = exec(P, nd.step9, ws, b9, p9, st, 0, nullptr, Win{b0 * nd.s, B * nd.s});
        }
        if (r) return r;
    }
    pm.mark();
    return GBS_SUCCESS;
}

static gbs_status_t check_device()
{
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(GBS_ERROR_CUDA, "no CUDA device");
    static DevOnce once;   // 1 = sm_100, 0 = other, -1 = query failed
    const int ok = once.run([dev] {
        int major = 0;
        if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return -1;
        return major == 10 ? 1 : 0;
    });
    if (ok < 0) return fail(GBS_ERROR_CUDA, "cannot query device");
    return ok ? GBS_SUCCESS : fail(GBS_ERROR_UNSUPPORTED, "device is not sm_100 (Blackwell B200)");
}

// Latency-bound sizes: a sort of at most GBS_GRAPH_MAX_N items is a short chain of small
// kernels whose cost is mostly the host's launch path.  Its launch sequence is fixed by
// (n, kind, buffers, workspace) (static plan, no host sync), so the first call with a
// given key captures it into a CUDA graph (on a per-thread capture stream) and every call
// replays that graph on the caller's stream: one launch instead of a dozen.  Calls on a
// stream that is itself being captured, profiled calls and debug runs enqueue directly.
#ifndef GBS_GRAPH_MAX_N
#define GBS_GRAPH_MAX_N (1u << 20)
#endif
constexpr size_t GRAPH_CACHE = 32;   // instantiated graphs kept (least recently used evicted)
struct GraphKey {
    uintptr_t k, v, ws;
    size_t n, ws_bytes;
    int xf, dev;
    bool operator==(const GraphKey& o) const
    {
        return k == o.k && v == o.v && ws == o.ws && n == o.n && ws_bytes == o.ws_bytes && xf == o.xf && dev == o.dev;
    }
};
struct GraphEnt {
    GraphKey key;
    cudaGraphExec_t exec;
    uint64_t used;
};
static std::mutex g_graph_mu;
static std::vector<GraphEnt> g_graphs;
static uint64_t g_graph_tick = 0;

static cudaGraphExec_t graph_find(const GraphKey& key)
{
    std::lock_guard<std::mutex> g(g_graph_mu);
    for (auto& e : g_graphs)
        if (e.key == key) {
            e.used = ++g_graph_tick;
            return e.exec;
        }
    return nullptr;
}
static void graph_put(const GraphKey& key, cudaGraphExec_t exec)
{
    std::lock_guard<std::mutex> g(g_graph_mu);
    if (g_graphs.size() >= GRAPH_CACHE) {
        auto lru = std::min_element(g_graphs.begin(), g_graphs.end(),
                                    [](const GraphEnt& a, const GraphEnt& b) { return a.used < b.used; });
        cudaGraphExecDestroy(lru->exec);   // (a launch in flight keeps its resources)
        g_graphs.erase(lru);
    }
    g_graphs.push_back(GraphEnt{key, exec, ++g_graph_tick});
}
static cudaStream_t capture_stream()
{
    static thread_local cudaStream_t cs[MAX_DEVICES] = {};
    const int d = cur_device();
    if (!cs[d] && cudaStreamCreateWithFlags(&cs[d], cudaStreamNonBlocking) != cudaSuccess) cs[d] = nullptr;
    return cs[d];
}

static gbs_status_t run_sort(uint32_t* keys, uint32_t* vals, size_t n, const gbs_config_t* cfg, int stop,
                             void* ws, size_t ws_bytes, cudaStream_t st, int xf = 0)
{
    const int kind = vals ? KIND_PAIRS : KIND_KEYS;
    Plan P;
    gbs_status_t r = make_plan(n, kind, cfg, P);
    if (r) return r;
    if (n <= 1) return GBS_SUCCESS;
    if (!keys) return fail(GBS_ERROR_INVALID_VALUE, "d_keys is NULL");
    if (((uintptr_t)keys & 3) || (vals && ((uintptr_t)vals & 3)))
        return fail(GBS_ERROR_INVALID_VALUE, "keys/values must be 4-byte aligned");
    if (vals) {
        const uintptr_t k0 = (uintptr_t)keys, k1 = k0 + n * 4, v0 = (uintptr_t)vals, v1 = v0 + n * 4;
        if (k0 < v1 && v0 < k1) return fail(GBS_ERROR_INVALID_VALUE, "keys and values overlap");
    }
    if (ws_bytes < P.ws) return fail(GBS_ERROR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu bytes", ws_bytes, P.ws);
    if (P.ws && (!ws || ((uintptr_t)ws & 255))) return fail(GBS_ERROR_INVALID_VALUE, "workspace NULL or not 256-byte aligned");
    if (stop && (stop < 2 || stop > 8)) return fail(GBS_ERROR_INVALID_VALUE, "stop_after_step must be 0 or 2..8");
    r = check_device();
    if (r) return r;
    char* w = reinterpret_cast<char*>(ws);
    const Node& top = P.nodes[0];
    Bufs bf{keys, top.leaf ? (void*)keys : (void*)(w + top.o_reloc), keys, vals,
            (top.leaf || !vals) ? vals : reinterpret_cast<uint32_t*>(w + top.o_reloc_v), vals};
    bf.xf_in = bf.xf_out = xf;
    Probs pr{nullptr, nullptr, 0, (uint32_t)n};
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (n <= GBS_GRAPH_MAX_N && !cfg && !stop && !g_prof && !debug_sync() &&
        cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone) {
        const GraphKey key{(uintptr_t)keys, (uintptr_t)vals, (uintptr_t)ws, n, ws_bytes, xf, cur_device()};
        cudaGraphExec_t ge = graph_find(key);
        if (ge) {
            GBS_CUDA(cudaGraphLaunch(ge, st));
            return GBS_SUCCESS;
        }
        // first call with this key: run it directly (this also does every one-time setup:
        // kernel attributes, side streams, events), then record the same sequence into a
        // graph for the next calls (capturing executes nothing)
        const gbs_status_t rd = exec(P, 0, w, bf, pr, st, 0);
        if (rd) return rd;
        cudaStream_t cs = capture_stream();
        if (cs && cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
            const gbs_status_t rc = exec(P, 0, w, bf, pr, cs, 0);
            cudaGraph_t g = nullptr;
            const cudaError_t ec = cudaStreamEndCapture(cs, &g);
            if (!rc && ec == cudaSuccess && g && cudaGraphInstantiate(&ge, g, 0) == cudaSuccess) graph_put(key, ge);
            if (g) cudaGraphDestroy(g);
        }
        cudaGetLastError();   // a failed capture only means no graph: the sort itself is done
        return GBS_SUCCESS;
    }
    return exec(P, 0, w, bf, pr, st, stop);
}

gbs_status_t fail_msg(gbs_status_t st, const char* msg) { return fail(st, "%s", msg); }

gbs_status_t sort_u64_ws(size_t n, size_t* bytes)
{
    Plan P;
    gbs_status_t r = make_plan(n, KIND_U64, nullptr, P);
    if (r) return r;
    *bytes = P.ws;
    return GBS_SUCCESS;
}

gbs_status_t sort_u64_inplace(unsigned long long* d, size_t n, void* ws, size_t ws_bytes, cudaStream_t st)
{
    // single-tile only: a multi-level u64 sort would need a sentinel tag base above
    // every caller tag (R8), which only the recursive Step 4 knows.
    if (n > TILE_U64) return fail(GBS_ERROR_UNSUPPORTED, "sort_u64_inplace: n > %u", TILE_U64);
    Plan P;
    gbs_status_t r = make_plan(n, KIND_U64, nullptr, P);
    if (r) return r;
    if (n <= 1) return GBS_SUCCESS;
    if (ws_bytes < P.ws) return fail(GBS_ERROR_WORKSPACE_TOO_SMALL, "u64 workspace too small");
    char* w = reinterpret_cast<char*>(ws);
    const Node& top = P.nodes[0];
    Bufs bf{d, top.leaf ? (void*)d : (void*)(w + top.o_reloc), d, nullptr, nullptr, nullptr};
    Probs pr{nullptr, nullptr, 0, (uint32_t)n};
    return exec(P, 0, w, bf, pr, st, 0);
}

// Out-of-place keys sort (the multi-GPU entry's local sort, E1): in[0, n) is only read;
// Step 2 writes the sorted sublists to a workspace buffer of n keys behind the plan's
// workspace, and the result lands in out (no extra pass).
gbs_status_t sort_keys_oop_ws(size_t n, size_t* bytes)
{
    Plan P;
    gbs_status_t r = make_plan(n, KIND_KEYS, nullptr, P);
    if (r) return r;
    *bytes = P.ws + (n * 4 + 255) / 256 * 256;
    return GBS_SUCCESS;
}

gbs_status_t sort_keys_oop(const uint32_t* in, uint32_t* out, size_t n, void* ws, size_t ws_bytes, cudaStream_t st)
{
    Plan P;
    gbs_status_t r = make_plan(n, KIND_KEYS, nullptr, P);
    if (r) return r;
    if (n == 0) return GBS_SUCCESS;
    if (!in || !out || ((uintptr_t)in & 3) || ((uintptr_t)out & 3)) return fail(GBS_ERROR_INVALID_VALUE, "oop sort: bad buffers");
    if (n == 1) {
        GBS_CUDA(cudaMemcpyAsync(out, in, 4, cudaMemcpyDeviceToDevice, st));
        return GBS_SUCCESS;
    }
    const size_t need = P.ws + (n * 4 + 255) / 256 * 256;
    if (ws_bytes < need) return fail(GBS_ERROR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu bytes", ws_bytes, need);
    if (!ws || ((uintptr_t)ws & 255)) return fail(GBS_ERROR_INVALID_VALUE, "workspace NULL or not 256-byte aligned");
    r = check_device();
    if (r) return r;
    char* w = reinterpret_cast<char*>(ws);
    const Node& top = P.nodes[0];
    Bufs bf{const_cast<uint32_t*>(in), top.leaf ? (void*)out : (void*)(w + top.o_reloc), out, nullptr, nullptr, nullptr};
    bf.srt = w + P.ws;
    Probs pr{nullptr, nullptr, 0, (uint32_t)n};
    return exec(P, 0, w, bf, pr, st, 0);
}

bool profiling() { return g_prof; }

}  // namespace gbs

using namespace gbs;

extern "C" {

const char* gbs_last_error(void) { return g_err; }

gbs_status_t gbs_profile_begin(void)
{
    g_prof = true;
    return GBS_SUCCESS;
}

gbs_status_t gbs_profile_end(gbs_step_times_t* out)
{
    g_prof = false;
    if (out) memset(out, 0, sizeof *out);
    gbs_status_t rc = GBS_SUCCESS;
    for (auto& pc : g_prof_calls) {
        if (cudaEventSynchronize(pc.ev[7]) != cudaSuccess) rc = fail(GBS_ERROR_CUDA, "profile event sync failed");
        static const int step_of[7] = {2, 4, 5, 6, 7, 8, 9};
        for (int k = 0; k < 7 && out && !rc; ++k) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, pc.ev[k], pc.ev[k + 1]);
            out->ms_level[pc.level][step_of[k]] += ms;
            if (pc.level == 0) out->ms[step_of[k]] += ms;
        }
        if (out && !rc) {
            if (pc.level == 0) out->calls += 1;
            if (pc.level + 1 > out->levels) out->levels = pc.level + 1;
        }
        for (auto e : pc.ev) cudaEventDestroy(e);
    }
    g_prof_calls.clear();
    return rc;
}

const char* gbs_status_string(gbs_status_t s)
{
    switch (s) {
        case GBS_SUCCESS: return "success";
        case GBS_ERROR_INVALID_VALUE: return "invalid value";
        case GBS_ERROR_WORKSPACE_TOO_SMALL: return "workspace too small";
        case GBS_ERROR_UNSUPPORTED: return "unsupported";
        case GBS_ERROR_CUDA: return "CUDA error";
        case GBS_ERROR_NCCL: return "NCCL error";
    }
    return "unknown status";
}

gbs_status_t gbs_workspace_size_ex(size_t n, int pairs, const gbs_config_t* cfg, size_t* bytes)
{
    if (!bytes) return fail(GBS_ERROR_INVALID_VALUE, "bytes is NULL");
    Plan P;
    gbs_status_t r = make_plan(n, pairs ? KIND_PAIRS : KIND_KEYS, cfg, P);
    if (r) return r;
    *bytes = P.ws;
    return GBS_SUCCESS;
}

gbs_status_t gbs_sort_keys_workspace_size(size_t n, size_t* bytes) { return gbs_workspace_size_ex(n, 0, nullptr, bytes); }
gbs_status_t gbs_sort_pairs_workspace_size(size_t n, size_t* bytes) { return gbs_workspace_size_ex(n, 1, nullptr, bytes); }

gbs_status_t gbs_plan(size_t n, int pairs, const gbs_config_t* cfg, gbs_plan_t* out)
{
    if (!out) return fail(GBS_ERROR_INVALID_VALUE, "out is NULL");
    Plan P;
    gbs_status_t r = make_plan(n, pairs ? KIND_PAIRS : KIND_KEYS, cfg, P);
    if (r) return r;
    memset(out, 0, sizeof *out);
    out->ws_bytes = P.ws;
    out->kernels_per_sort = P.launches;
    int ni = P.nodes.empty() ? -1 : 0;
    while (ni >= 0 && !P.nodes[ni].leaf && out->levels < GBS_MAX_LEVELS) {
        const Node& nd = P.nodes[ni];
        const int k = out->levels++;
        out->L[k] = nd.L;
        out->s[k] = nd.s;
        out->m[k] = nd.m;
        out->cap[k] = nd.N;
        out->bucket_bound[k] = nd.hi;
        ni = nd.step9;
    }
    return GBS_SUCCESS;
}

gbs_status_t gbs_debug_layout(size_t n, int pairs, const gbs_config_t* cfg, gbs_layout_t* out)
{
    if (!out) return fail(GBS_ERROR_INVALID_VALUE, "out is NULL");
    Plan P;
    gbs_status_t r = make_plan(n, pairs ? KIND_PAIRS : KIND_KEYS, cfg, P);
    if (r) return r;
    memset(out, 0xff, sizeof *out);
    if (P.nodes.empty() || P.nodes[0].leaf) return GBS_SUCCESS;
    const Node& t = P.nodes[0];
    out->samples = t.o_samples;
    out->splitters = t.o_splitters;
    out->a = t.o_a;
    out->l = t.o_l;
    out->relocated = t.o_reloc;
    out->relocated_vals = t.o_reloc_v;
    return GBS_SUCCESS;
}

gbs_status_t gbs_sort_keys(uint32_t* d_keys, size_t n, void* d_ws, size_t ws_bytes, gbs_stream_t stream)
{
    return run_sort(d_keys, nullptr, n, nullptr, 0, d_ws, ws_bytes, (cudaStream_t)stream);
}

gbs_status_t gbs_sort_pairs(uint32_t* d_keys, uint32_t* d_vals, size_t n, void* d_ws, size_t ws_bytes,
                            gbs_stream_t stream)
{
    if (n > 1 && !d_vals) return fail(GBS_ERROR_INVALID_VALUE, "d_vals is NULL");
    return run_sort(d_keys, d_vals, n, nullptr, 0, d_ws, ws_bytes, (cudaStream_t)stream);
}

// 64-bit keys: LSD over the two 32-bit halves of the key's order-preserving image, each
// pass a stable GBS of (half, index) pairs; then one gather of the original keys (and
// values) by the final index permutation.  Workspace: the pairs sort's + lo/hi halves,
// indices, a copy of the keys (and values).
struct K64Layout {
    size_t pairs_ws, half, idx, kcopy, vcopy, total;
};
static gbs_status_t k64_layout(size_t n, bool pairs, K64Layout* L)
{
    Plan P;
    gbs_status_t r = make_plan(n, KIND_PAIRS, nullptr, P);
    if (r) return r;
    size_t o = 0;
    auto al = [](size_t x) { return (x + 255) / 256 * 256; };
    L->pairs_ws = o; o += al(P.ws);
    L->half = o;     o += al(n * 4);
    L->idx = o;      o += al(n * 4);
    L->kcopy = o;    o += al(n * 8);
    L->vcopy = o;    o += pairs ? al(n * 4) : 0;
    L->total = o;
    return GBS_SUCCESS;
}

static gbs_status_t run_sort64(void* keys, uint32_t* vals, size_t n, int type, void* ws, size_t ws_bytes, cudaStream_t st)
{
    if (type < GBS_KEY64_U64 || type > GBS_KEY64_F64) return fail(GBS_ERROR_INVALID_VALUE, "key_type %d", type);
    K64Layout L;
    gbs_status_t r = k64_layout(n, vals != nullptr, &L);
    if (r) return r;
    if (n <= 1) return GBS_SUCCESS;
    if (!keys || ((uintptr_t)keys & 7)) return fail(GBS_ERROR_INVALID_VALUE, "d_keys NULL or not 8-byte aligned");
    if (vals) {
        if ((uintptr_t)vals & 3) return fail(GBS_ERROR_INVALID_VALUE, "d_vals not 4-byte aligned");
        const uintptr_t k0 = (uintptr_t)keys, k1 = k0 + n * 8, v0 = (uintptr_t)vals, v1 = v0 + n * 4;
        if (k0 < v1 && v0 < k1) return fail(GBS_ERROR_INVALID_VALUE, "keys and values overlap");
    }
    if (ws_bytes < L.total) return fail(GBS_ERROR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu bytes", ws_bytes, L.total);
    if (!ws || ((uintptr_t)ws & 255)) return fail(GBS_ERROR_INVALID_VALUE, "workspace NULL or not 256-byte aligned");
    r = check_device();
    if (r) return r;
    char* w = reinterpret_cast<char*>(ws);
    auto* k = reinterpret_cast<unsigned long long*>(keys);
    uint32_t* half = reinterpret_cast<uint32_t*>(w + L.half);
    uint32_t* idx = reinterpret_cast<uint32_t*>(w + L.idx);
    auto* kc = reinterpret_cast<unsigned long long*>(w + L.kcopy);
    uint32_t* vc = vals ? reinterpret_cast<uint32_t*>(w + L.vcopy) : nullptr;
    const unsigned grid = num_sms() * 8;
    launch_k(k_k64_lo, grid, 256, 0, st, (const unsigned long long*)k, (uint64_t)n, type, half, idx);
    GBS_CUDA(cudaGetLastError());
    r = run_sort(half, idx, n, nullptr, 0, w + L.pairs_ws, L.half - L.pairs_ws, st);    // pass 1: by the low half
    if (r) return r;
    launch_k(k_k64_hi, grid, 256, 0, st, (const unsigned long long*)k, (uint64_t)n, type, (const uint32_t*)idx, half);
    GBS_CUDA(cudaGetLastError());
    r = run_sort(half, idx, n, nullptr, 0, w + L.pairs_ws, L.half - L.pairs_ws, st);    // pass 2: by the high half
    if (r) return r;
    GBS_CUDA(cudaMemcpyAsync(kc, k, n * 8, cudaMemcpyDeviceToDevice, st));
    if (vals) GBS_CUDA(cudaMemcpyAsync(vc, vals, n * 4, cudaMemcpyDeviceToDevice, st));
    launch_k(k_k64_gather, grid, 256, 0, st, (const unsigned long long*)kc, (const uint32_t*)idx, (uint64_t)n, k,
             (const uint32_t*)vc, vals);
    GBS_CUDA(cudaGetLastError());
    return GBS_SUCCESS;
}

// Typed keys: validate everything run_sort would (so nothing is enqueued on a bad call),
// then sort the keys' u32 images: the transform is applied where keys enter the sort
// (Step 2's load) and inverted where they leave it (the last level's Step 9 store).
static gbs_status_t run_sort_typed(void* keys, uint32_t* vals, size_t n, int type, void* ws, size_t ws_bytes,
                                   cudaStream_t st)
{
    if (type < GBS_KEY_U32 || type > GBS_KEY_F32) return fail(GBS_ERROR_INVALID_VALUE, "key_type %d", type);
    uint32_t* k = reinterpret_cast<uint32_t*>(keys);
    if (type == GBS_KEY_U32 || n <= 1) return run_sort(k, vals, n, nullptr, 0, ws, ws_bytes, st);
    Plan P;
    gbs_status_t r = make_plan(n, vals ? KIND_PAIRS : KIND_KEYS, nullptr, P);
    if (r) return r;
    if (!k) return fail(GBS_ERROR_INVALID_VALUE, "d_keys is NULL");
    if (((uintptr_t)k & 3) || (vals && ((uintptr_t)vals & 3)))
        return fail(GBS_ERROR_INVALID_VALUE, "keys/values must be 4-byte aligned");
    if (vals) {
        const uintptr_t k0 = (uintptr_t)k, k1 = k0 + n * 4, v0 = (uintptr_t)vals, v1 = v0 + n * 4;
        if (k0 < v1 && v0 < k1) return fail(GBS_ERROR_INVALID_VALUE, "keys and values overlap");
    }
    if (ws_bytes < P.ws) return fail(GBS_ERROR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu bytes", ws_bytes, P.ws);
    if (P.ws && (!ws || ((uintptr_t)ws & 255))) return fail(GBS_ERROR_INVALID_VALUE, "workspace NULL or not 256-byte aligned");
    r = check_device();
    if (r) return r;
    // the transform runs inside the sort: at Step 2's load and the last Step 9's store
    return run_sort(k, vals, n, nullptr, 0, ws, ws_bytes, st, type);
}

gbs_status_t gbs_sort_keys_typed(void* d_keys, size_t n, int key_type, void* d_ws, size_t ws_bytes,
                                 gbs_stream_t stream)
{
    return run_sort_typed(d_keys, nullptr, n, key_type, d_ws, ws_bytes, (cudaStream_t)stream);
}

gbs_status_t gbs_sort_pairs_typed(void* d_keys, uint32_t* d_vals, size_t n, int key_type, void* d_ws,
                                  size_t ws_bytes, gbs_stream_t stream)
{
    if (n > 1 && !d_vals) return fail(GBS_ERROR_INVALID_VALUE, "d_vals is NULL");
    return run_sort_typed(d_keys, d_vals, n, key_type, d_ws, ws_bytes, (cudaStream_t)stream);
}

gbs_status_t gbs_sort64_workspace_size(size_t n, int pairs, size_t* bytes)
{
    if (!bytes) return fail(GBS_ERROR_INVALID_VALUE, "bytes is NULL");
    K64Layout L;
    gbs_status_t r = k64_layout(n, pairs != 0, &L);
    if (r) return r;
    *bytes = L.total;
    return GBS_SUCCESS;
}

gbs_status_t gbs_sort_keys64(void* d_keys, size_t n, int key_type, void* d_ws, size_t ws_bytes, gbs_stream_t stream)
{
    return run_sort64(d_keys, nullptr, n, key_type, d_ws, ws_bytes, (cudaStream_t)stream);
}

gbs_status_t gbs_sort_pairs64(void* d_keys, uint32_t* d_vals, size_t n, int key_type, void* d_ws, size_t ws_bytes,
                              gbs_stream_t stream)
{
    if (n > 1 && !d_vals) return fail(GBS_ERROR_INVALID_VALUE, "d_vals is NULL");
    return run_sort64(d_keys, d_vals, n, key_type, d_ws, ws_bytes, (cudaStream_t)stream);
}

gbs_status_t gbs_sort_ex(uint32_t* d_keys, uint32_t* d_vals, size_t n, const gbs_config_t* cfg, int stop_after_step,
                         void* d_ws, size_t ws_bytes, gbs_stream_t stream)
{
    return run_sort(d_keys, d_vals, n, cfg, stop_after_step, d_ws, ws_bytes, (cudaStream_t)stream);
}

// End to end from pinned host buffers (keys, or keys + values).  Above HP_CHUNK_TILES
// sublists the H2D copy is chunked so Step 2 sorts each chunk as it lands; with CTA
// buckets (one level) the D2H copy of each bucket group's final output prefix (R18)
// overlaps the remaining Step 9 groups; with a nested Step 9 the nested level runs in
// groups of problems and each group's final output prefix is copied back under the next.
static gbs_status_t run_sort_host(uint32_t* h_keys, uint32_t* h_vals, size_t n, uint32_t* d_keys, uint32_t* d_vals,
                                  void* d_ws, size_t ws_bytes, cudaStream_t st)
{
    const bool pairs = h_vals != nullptr;
    if (n > 1 && (!h_keys || !d_keys || (pairs && !d_vals))) return fail(GBS_ERROR_INVALID_VALUE, "NULL buffer");
    if (n == 0) return GBS_SUCCESS;
    const int kind = pairs ? KIND_PAIRS : KIND_KEYS;
    Plan P;
    gbs_status_t r = make_plan(n, kind, nullptr, P);
    if (r) return r;
    if (ws_bytes < P.ws) return fail(GBS_ERROR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu bytes", ws_bytes, P.ws);
    const size_t bytes = n * 4;
    if (GBS_HOST_PIPE && !P.nodes.empty() && !P.nodes[0].leaf && P.nodes[0].B == 1 &&
        n >= (size_t)HP_CHUNK_TILES * P.nodes[0].L) {
        const Node& top = P.nodes[0];
        cudaStream_t cin = side_stream(1), cout = side_stream(2);
        if (cin && cout) {
            r = check_device();
            if (r) return r;
            if (!d_ws || ((uintptr_t)d_ws & 255)) return fail(GBS_ERROR_INVALID_VALUE, "workspace NULL or not 256-byte aligned");
            if (((uintptr_t)d_keys & 3) || (pairs && ((uintptr_t)d_vals & 3)))
                return fail(GBS_ERROR_INVALID_VALUE, "keys/values must be 4-byte aligned");
            if (pairs) {
                const uintptr_t k0 = (uintptr_t)d_keys, k1 = k0 + bytes, v0 = (uintptr_t)d_vals, v1 = v0 + bytes;
                if (k0 < v1 && v0 < k1) return fail(GBS_ERROR_INVALID_VALUE, "keys and values overlap");
            }
            char* w = reinterpret_cast<char*>(d_ws);
            Bufs bf{d_keys, (void*)(w + top.o_reloc), d_keys, d_vals,
                    pairs ? reinterpret_cast<uint32_t*>(w + top.o_reloc_v) : nullptr, d_vals};
            Probs pr{nullptr, nullptr, 0, (uint32_t)n};
            HostPipe hp{h_keys, h_vals, n, cin, cout};
            // (a nested Step 9 copies each group of finished problems back itself)
            r = exec(P, 0, w, bf, pr, st, 0, &hp);
            if (r) return r;
            return GBS_SUCCESS;
        }
    }
    GBS_CUDA(cudaMemcpyAsync(d_keys, h_keys, bytes, cudaMemcpyHostToDevice, st));
    if (pairs) GBS_CUDA(cudaMemcpyAsync(d_vals, h_vals, bytes, cudaMemcpyHostToDevice, st));
    r = run_sort(d_keys, d_vals, n, nullptr, 0, d_ws, ws_bytes, st);
    if (r) return r;
    GBS_CUDA(cudaMemcpyAsync(h_keys, d_keys, bytes, cudaMemcpyDeviceToHost, st));
    if (pairs) GBS_CUDA(cudaMemcpyAsync(h_vals, d_vals, bytes, cudaMemcpyDeviceToHost, st));
    return GBS_SUCCESS;
}

gbs_status_t gbs_sort_keys_host(uint32_t* h_keys, size_t n, uint32_t* d_keys, void* d_ws, size_t ws_bytes,
                                gbs_stream_t stream)
{
    return run_sort_host(h_keys, nullptr, n, d_keys, nullptr, d_ws, ws_bytes, (cudaStream_t)stream);
}

gbs_status_t gbs_sort_pairs_host(uint32_t* h_keys, uint32_t* h_vals, size_t n, uint32_t* d_keys, uint32_t* d_vals,
                                 void* d_ws, size_t ws_bytes, gbs_stream_t stream)
{
    if (n > 1 && !h_vals) return fail(GBS_ERROR_INVALID_VALUE, "h_vals is NULL");
    return run_sort_host(h_keys, n > 1 ? h_vals : nullptr, n, d_keys, d_vals, d_ws, ws_bytes, (cudaStream_t)stream);
}

}  // extern "C"
