// gbs_dist.cu -- multi-GPU GPU Bucket Sort.
//
// The paper is single-GPU.  Across the GPUs of one box Alg. 1 is applied once more as an
// outer level with one sublist per rank (parallel sorting by regular sampling, the scheme
// of [Schaeffer] behind the paper's bucket bound):
//   E1 local GBS of the shard, out of place (the whole single-GPU path = outer Step 2)
//   E2 s_r regular samples per rank, composites (key, global position)     (Step 3)
//   E3 every rank receives every rank's samples                            (Step 4 input)
//   E4 every rank sorts the p*s_r samples identically (no broadcast)       (Step 4)
//   E5 splitters G_k = sorted[(k+1) s_r - 1]                               (Step 5)
//   E6 "fine cuts": for EVERY sorted sample q, F[r][q] = #items of rank r's sorted shard
//      that are <= sample q (bisection; the splitters' cuts are F[r][(k+1) s_r - 1]) (Step 6)
//   E7 every rank receives the p x (p s_r) matrix F                        (Step 7)
//   E8 relocation as the exchange: rank r's run for rank k, W_r[F[r][q_{k-1}], F[r][q_k]),
//      goes to rank k's receive buffer at sum_{r'<r} (F[r'][q_k] - F[r'][q_{k-1}]) (Step 8)
//   E9 the p runs a rank received are merged in ONE pass: the sorted samples inside its
//      bucket cut every run into s_r chunks (run r's share of chunk q is
//      [F[r][q-1], F[r][q]) relative to its run), each chunk is a k-way merge of <= p
//      pieces by one CTA                                                   (Step 9)
//
// Transport.  The product path is NVLink peer memory: every rank owns a
// window (signal pad, sample slots, the F matrix, the receive buffer) mapped into every
// peer with CUDA IPC (handles exchanged over NCCL once per window size).  E3, E7 and E8 are
// stores from our own kernels straight into the peers' windows, separated by device-side
// barriers (flag stores / acquire loads at system scope): no host synchronisation and no
// host-side counts until the call returns *n_out.  Where peer mapping is unavailable the
// same phases run with NCCL collectives instead (allgather of samples and of F, grouped
// send/recv, one stream sync for the counts).  The single-GPU emulation runs the P2P
// kernels of all p ranks on one GPU with the peers' windows as regions of one buffer.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "gbs_internal.h"

namespace {

constexpr uint32_t S_R_MAX = 1024;   // regular samples per rank (E2)
constexpr int MAX_RANKS = 16;        // p * s_r composites sort in one CTA tile (E4)
constexpr int MERGE_MAX_P = 16;

// s_r: the largest power of two <= S_R_MAX that divides n_local, so the regular sample
// positions (k+1) n_l / s_r - 1 are exactly equidistant (d = n_l / s_r).
uint32_t s_r_of(size_t n_local)
{
    uint32_t s = 1;
    while (s < S_R_MAX && n_local % (2ull * s) == 0) s *= 2;
    return s;
}

// receive bound n_l + (p-1)(n_l/s_r - 1) (the tight bound with m = p)
size_t out_cap(size_t n_local, int p)
{
    const size_t d = n_local / s_r_of(n_local);
    return n_local + (size_t)(p - 1) * (d - 1);
}

size_t al(size_t x) { return (x + 255) / 256 * 256; }

#define NCCL_OK(call)                                                                     \
    do {                                                                                  \
        ncclResult_t r_ = (call);                                                         \
        if (r_ != ncclSuccess) {                                                          \
            char b_[256];                                                                 \
            snprintf(b_, sizeof b_, "%s: %s", #call, ncclGetErrorString(r_));             \
            return gbs::fail_msg(GBS_ERROR_NCCL, b_);                                     \
        }                                                                                 \
    } while (0)

#define CUDA_OK(call)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            char b_[256];                                                                 \
            snprintf(b_, sizeof b_, "%s: %s", #call, cudaGetErrorString(e_));             \
            return gbs::fail_msg(GBS_ERROR_CUDA, b_);                                     \
        }                                                                                 \
    } while (0)

// ------------------------------------------------------------------ layouts
// The window: identical offsets on every rank (every rank passes the same n_local).
struct WinLayout {
    size_t flags;      // MAX_RANKS u64 barrier flags (flags[src] written by src) + status
    size_t gathered;   // p * s_r u64: rank r's samples at [r s_r, (r+1) s_r) (E3), sorted in place (E4)
    size_t fcut;       // p x (p s_r) u64: row r = F[r][.] (E7)
    size_t recv;       // out_cap u32: the received runs in source order (E8)
    size_t total;
};
WinLayout win_layout(size_t n_local, int p)
{
    const uint32_t s_r = s_r_of(n_local);
    WinLayout L;
    size_t o = 0;
    L.flags = o;    o += al((MAX_RANKS + 2) * 8);
    L.gathered = o; o += al((size_t)p * s_r * 8);
    L.fcut = o;     o += al((size_t)p * p * s_r * 8);
    L.recv = o;     o += al(out_cap(n_local, p) * 4);
    L.total = o;
    return L;
}

// The rank's local workspace.
struct DistLayout {
    size_t sort_ws, sort_ws_bytes;   // E1 (out of place)
    size_t shard;                    // n_l u32: the sorted shard W (E1 output, E8 source)
    size_t samples;                  // s_r u64 (NCCL path: E3 send buffer)
    size_t frow;                     // p s_r u64 (NCCL path: E7 send buffer)
    size_t u64ws, u64ws_bytes;       // E4 sample sort
    size_t words;                    // 4 u64: n_out, bytes sent to other ranks, status
    size_t total;
};
gbs_status_t dist_layout(size_t n_local, int p, DistLayout* L)
{
    size_t a = 0, u = 0;
    gbs_status_t r = gbs::sort_keys_oop_ws(n_local, &a);
    if (r) return r;
    const uint32_t s_r = s_r_of(n_local);
    r = gbs::sort_u64_ws((size_t)p * s_r, &u);
    if (r) return r;
    size_t o = 0;
    L->sort_ws = o;  o += al(a);
    L->sort_ws_bytes = al(a);
    L->shard = o;    o += al(n_local * 4);
    L->samples = o;  o += al((size_t)s_r * 8);
    L->frow = o;     o += al((size_t)p * s_r * 8);
    L->u64ws = o;    o += al(u);
    L->u64ws_bytes = u;
    L->words = o;    o += al(4 * 8);
    L->total = o;
    return GBS_SUCCESS;
}

// ------------------------------------------------------------------ kernels
typedef unsigned long long u64;

__device__ __forceinline__ u64 composite(uint32_t key, uint64_t gpos) { return ((u64)key << 32) | (u64)(uint32_t)gpos; }

// E2 (+E3 on the P2P path): regular sample k of this rank, composite (key, global
// position), stored into slot [rank s_r + k] of every destination window (dst[q] = base of
// window q's gathered array; one destination = the NCCL send buffer).
__global__ void k_dist_samples(const uint32_t* shard, size_t n_local, uint32_t s_r, int rank, u64* const* dst,
                               int ndst, size_t slot0)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= s_r) return;
    const size_t d = n_local / s_r;
    const size_t pos = (size_t)(k + 1) * d - 1;
    const u64 c = composite(shard[pos], (uint64_t)rank * n_local + pos);
    for (int q = 0; q < ndst; ++q) dst[q][slot0 + k] = c;
}

// E6 (+E7 on the P2P path): F[rank][q] = #{pos : (W[pos], gbase + pos) <= sorted[q]} for
// every sorted sample q, stored into row `rank` of every destination's F matrix.
__global__ void k_dist_finecuts(const uint32_t* shard, size_t n_local, uint64_t gbase, const u64* sorted, uint32_t nq,
                                u64* const* dst, int ndst, size_t row0)
{
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const u64 g = sorted[q];
    size_t lo = 0, hi = n_local;
    // keys above g's key are never <= g; a tie on the key is decided by the position
    while (lo < hi) {
        const size_t mid = (lo + hi) / 2;
        if (composite(shard[mid], gbase + mid) <= g) lo = mid + 1;
        else hi = mid;
    }
    for (int d = 0; d < ndst; ++d) dst[d][row0 + q] = lo;
}

// F[r][q] with F[r][-1] = 0
__device__ __forceinline__ u64 fcut(const u64* F, uint32_t nq, int r, long long q) { return q < 0 ? 0ull : F[(size_t)r * nq + q]; }

// E8 push: rank `rank` copies its run for every destination k into k's receive buffer
// (dst[k]), at the source-order offset derived from F (identical on every rank).
// blockIdx.y = destination, blockIdx.x strides over the run; 4-byte coalesced copies
// with 8 loads in flight per thread; every thread fences its peer stores (system scope)
// before the barrier that follows.
__global__ void __launch_bounds__(256) k_dist_push(const uint32_t* shard, const u64* F, uint32_t nq, uint32_t s_r, int p,
                                                   int rank, uint32_t* const* dst, u64* sent)
{
    const int k = blockIdx.y;
    const long long qlo = (long long)k * s_r - 1, qhi = (long long)(k + 1) * s_r - 1;
    const u64 a0 = fcut(F, nq, rank, qlo), a1 = fcut(F, nq, rank, qhi);
    u64 off = 0;
    for (int r = 0; r < rank; ++r) off += fcut(F, nq, r, qhi) - fcut(F, nq, r, qlo);
    const u64 cnt = a1 - a0;
    if (sent && k != rank && blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(sent, cnt * 4);
    const uint32_t* src = shard + a0;
    uint32_t* d = dst[k] + off;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    constexpr int U = 8;
    for (u64 i0 = (u64)blockIdx.x * blockDim.x + threadIdx.x; i0 < cnt; i0 += U * stride) {
        uint32_t v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const u64 i = i0 + u * stride;
            v[u] = i < cnt ? __ldg(src + i) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const u64 i = i0 + u * stride;
            if (i < cnt) d[i] = v[u];
        }
    }
    __threadfence_system();
}

// Device-side barrier over the ranks' windows: thread k signals rank k (flags[rank] in
// k's window := epoch, release at system scope) and waits until rank k has signalled us
// (acquire).  A bounded spin (~20 s) records a timeout in *status instead of hanging.
__global__ void k_p2p_barrier(u64* const* flags, int p, int rank, u64 epoch, unsigned* status)
{
    const int k = threadIdx.x;
    if (k >= p) return;
    __threadfence_system();
    u64* to = flags[k] + rank;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(to), "l"(epoch) : "memory");
    const u64* mine = flags[rank] + k;
    long long spins = 0;
    while (true) {
        u64 v;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(mine) : "memory");
        if (v >= epoch) break;
        __nanosleep(200);
        if (++spins > 100000000ll) {
            atomicOr(status, 1u);
            break;
        }
    }
}

// E9: k-way merge of the p runs received (recv, in source order) into out, one CTA per
// chunk between consecutive sorted samples of this rank's bucket.  Run r of chunk j is
// [F[r][q_j - 1], F[r][q_j]) - F[r][qlo] (relative to run r's start) with q_j = qlo + 1 + j.
// Inside a chunk the CTA streams: it loads a window of up to TW = CAP/p items of every
// piece (one batch of loads, all in flight), takes from each piece what is <= the smallest
// last-loaded item of the pieces that have more to load (ties broken by run index: the
// merge is stable by source rank), merges the taken pieces in shared memory (pairwise
// merge-path levels, piece table in shared memory) and writes them out coalesced.
constexpr int KM_BLOCK = 512, KM_ITEMS = 16, KM_CAP = KM_BLOCK * KM_ITEMS;   // 8192 items per window
// shared-memory layout with one pad slot per KM_ITEMS: a thread's KM_ITEMS consecutive
// outputs then sit at stride KM_ITEMS + 1 across the warp (conflict-free stores)
constexpr int KM_PAD_CAP = KM_CAP + KM_CAP / KM_ITEMS + 16;
__device__ __forceinline__ int km_pad(int i) { return i + (i >> 4); }

// merge-path split of diagonal `diag` of A = s[ao, ao+na) and B = s[bo, bo+nb) (padded)
__device__ __forceinline__ int merge_split_pad(const uint32_t* s, int ao, int na, int bo, int nb, int diag)
{
    int lo = max(0, diag - nb), hi = min(diag, na);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s[km_pad(ao + mid)] <= s[km_pad(bo + diag - 1 - mid)]) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(KM_BLOCK, 2) k_kway_merge(const uint32_t* recv, const u64* F, uint32_t nq, uint32_t s_r,
                                                         int p, int rank, uint32_t* out, u64* n_out)
{
    extern __shared__ __align__(16) uint32_t km_smem[];
    uint32_t* bufA = km_smem;
    uint32_t* bufB = km_smem + KM_PAD_CAP;
    __shared__ u64 s_base[MERGE_MAX_P], s_lo[MERGE_MAX_P], s_hi[MERGE_MAX_P];
    __shared__ int s_win[MERGE_MAX_P];
    // piece table per merge level: offset and length of every piece (level 0 = the windows)
    __shared__ int s_poff[5][MERGE_MAX_P + 1], s_plen[5][MERGE_MAX_P + 1];
    __shared__ u64 s_o;
    __shared__ int s_more;
    const int tw = KM_CAP / p;                                   // window per piece
    const long long qlo = (long long)rank * s_r - 1;
    const long long qj = qlo + 1 + blockIdx.x;
    if (threadIdx.x == 0) {
        u64 base = 0, o = 0;
        for (int r = 0; r < p; ++r) {
            const u64 f0 = fcut(F, nq, r, qlo), f1 = fcut(F, nq, r, (long long)(rank + 1) * s_r - 1);
            s_base[r] = base;                                    // run r's start in recv
            s_lo[r] = fcut(F, nq, r, qj - 1) - f0;
            s_hi[r] = fcut(F, nq, r, qj) - f0;
            o += s_lo[r];
            base += f1 - f0;
        }
        s_o = o;
        if (blockIdx.x == gridDim.x - 1 && n_out) *n_out = base;
    }
    __syncthreads();
    while (true) {
        if (threadIdx.x == 0) {
            int more = 0;
            for (int r = 0; r < p; ++r) {
                const int w = (int)min((u64)tw, s_hi[r] - s_lo[r]);
                s_win[r] = w;
                more |= w > 0;
            }
            s_more = more;
        }
        __syncthreads();
        if (!s_more) break;
        {   // the windows of all pieces in one batch of loads (piece r at bufA[r tw ...])
            uint32_t v[KM_ITEMS];
#pragma unroll
            for (int k = 0; k < KM_ITEMS; ++k) {
                const int i = threadIdx.x + k * KM_BLOCK;
                const int r = i / tw, j = i - r * tw;
                v[k] = (r < p && j < s_win[r]) ? __ldg(recv + s_base[r] + s_lo[r] + j) : 0u;
            }
#pragma unroll
            for (int k = 0; k < KM_ITEMS; ++k) {
                const int i = threadIdx.x + k * KM_BLOCK;
                const int r = i / tw, j = i - r * tw;
                if (r < p && j < s_win[r]) bufA[km_pad(i)] = v[k];
            }
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            // threshold: the smallest (key, run) among the last loaded items of pieces with more
            const int lane = threadIdx.x;
            uint32_t tk = 0xFFFFFFFFu;
            int tr = MERGE_MAX_P;                                 // MERGE_MAX_P = no threshold
            for (int r = 0; r < p; ++r) {
                if (s_lo[r] + s_win[r] < s_hi[r]) {
                    const uint32_t k = bufA[km_pad(r * tw + s_win[r] - 1)];
                    if (tr == MERGE_MAX_P || k < tk) { tk = k; tr = r; }
                }
            }
            // pieces: r < tr take keys <= tk, r > tr keys < tk, r == tr all (lane r)
            if (lane < p) {
                const int r = lane, w = s_win[r];
                int t = w;
                if (tr != MERGE_MAX_P && r != tr) {
                    int lo = 0, hi = w;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        const uint32_t am = bufA[km_pad(r * tw + mid)];
                        const bool take = r < tr ? am <= tk : am < tk;
                        if (take) lo = mid + 1;
                        else hi = mid;
                    }
                    t = lo;
                }
                s_plen[0][r] = t;
                s_poff[0][r] = r * tw;
            }
            __syncwarp();
            if (lane == 0) {   // the piece tables of the merge levels
                int np = p, lev = 0;
                while (np > 1) {
                    const int nn = (np + 1) / 2;
                    int o = 0;
                    for (int i = 0; i < nn; ++i) {
                        const int len = s_plen[lev][2 * i] + (2 * i + 1 < np ? s_plen[lev][2 * i + 1] : 0);
                        s_poff[lev + 1][i] = o;
                        s_plen[lev + 1][i] = len;
                        o += len;
                    }
                    s_poff[lev + 1][nn] = o;
                    np = nn;
                    ++lev;
                }
                int T = 0;
                for (int r = 0; r < p; ++r) T += s_plen[0][r];
                s_poff[0][MERGE_MAX_P] = T;
            }
        }
        __syncthreads();
        const int T = s_poff[0][MERGE_MAX_P];
        uint32_t* cur = bufA;
        uint32_t* nxt = bufB;
        int np = p, lev = 0;
        while (np > 1) {
            // merge pieces (2i, 2i+1) of level lev -> piece i of level lev+1
            const int nn = (np + 1) / 2;
            int q = threadIdx.x * KM_ITEMS, i = 0;
            const int q1 = min(T, q + KM_ITEMS);
            while (q < q1) {   // this thread's outputs may straddle two output pieces
                while (i + 1 < nn && s_poff[lev + 1][i + 1] <= q) ++i;
                const int ao = s_poff[lev][2 * i];
                const int nai = s_plen[lev][2 * i];
                const bool hasb = 2 * i + 1 < np;
                const int bo = hasb ? s_poff[lev][2 * i + 1] : ao + nai;
                const int nbi = hasb ? s_plen[lev][2 * i + 1] : 0;
                const int o0 = s_poff[lev + 1][i];
                const int qe = min(q1, o0 + s_plen[lev + 1][i]);
                int ia = merge_split_pad(cur, ao, nai, bo, nbi, q - o0);
                int ib = q - o0 - ia;
                uint32_t a = ia < nai ? cur[km_pad(ao + ia)] : 0u, b = ib < nbi ? cur[km_pad(bo + ib)] : 0u;
                for (; q < qe; ++q) {   // branch-free: one load per output
                    // ties: lower run first; an exhausted run is never taken (the load one
                    // past its end reads the buffer's next slot, within the slack)
                    const bool ta = ib >= nbi || (ia < nai && a <= b);
                    nxt[km_pad(q)] = ta ? a : b;
                    ia += ta ? 1 : 0;
                    ib += ta ? 0 : 1;
                    const uint32_t v = cur[km_pad(ta ? ao + ia : bo + ib)];
                    a = ta ? v : a;
                    b = ta ? b : v;
                }
            }
            __syncthreads();
            uint32_t* t = cur;
            cur = nxt;
            nxt = t;
            np = nn;
            ++lev;
        }
        // write out: the single piece of the last level (p = 1: the window itself)
        const u64 o0 = s_o;
        const int off = s_poff[lev][0];
        for (int i = threadIdx.x; i < T; i += KM_BLOCK) out[o0 + i] = cur[km_pad(off + i)];
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int r = 0; r < p; ++r) s_lo[r] += s_plen[0][r];
            s_o = o0 + T;
        }
        __syncthreads();
    }
}

}  // namespace

// ------------------------------------------------------------------ communicator
struct gbs_comm {
    ncclComm_t nc = nullptr;        // null: bootstrapped through a host allgather (P2P only)
    gbs_host_allgather_fn hag = nullptr;
    void* hag_ctx = nullptr;
    int nranks, rank, device;
    int mode;                       // 0 auto (P2P when every peer maps), 1 NCCL
    // window (P2P path): own allocation, every rank's base, device copies of the per-array
    // pointer tables; (re)created when a call needs more bytes
    char* win = nullptr;
    size_t win_bytes = 0;
    void* peer_base[MAX_RANKS] = {};
    bool p2p = false;
    u64 epoch = 0;
    void** d_tab = nullptr;         // [4][MAX_RANKS] device pointer tables
    char* scratch = nullptr;        // device scratch for handle exchange
    unsigned long long* h_cuts = nullptr;   // pinned host
    cudaEvent_t ev[8] = {};
};

namespace {

gbs_status_t close_window(gbs_comm* c)
{
    for (int k = 0; k < c->nranks; ++k)
        if (k != c->rank && c->peer_base[k]) cudaIpcCloseMemHandle(c->peer_base[k]);
    for (auto& b : c->peer_base) b = nullptr;
    if (c->win) cudaFree(c->win);
    c->win = nullptr;
    c->win_bytes = 0;
    c->p2p = false;
    return GBS_SUCCESS;
}

// Collective: (re)create the window of `bytes` on every rank and map the peers' windows.
gbs_status_t ensure_window(gbs_comm* c, size_t bytes, cudaStream_t st)
{
    if (c->win && c->win_bytes >= bytes) return GBS_SUCCESS;
    CUDA_OK(cudaStreamSynchronize(st));
    close_window(c);
    CUDA_OK(cudaMalloc(&c->win, bytes));
    CUDA_OK(cudaMemset(c->win, 0, bytes));
    c->win_bytes = bytes;
    c->epoch = 0;
    c->peer_base[c->rank] = c->win;
    int ok = 1;
    if (c->nranks > 1 && c->mode == 0) {
        cudaIpcMemHandle_t h;
        if (cudaIpcGetMemHandle(&h, c->win) != cudaSuccess) ok = 0;
        const size_t hb = sizeof(cudaIpcMemHandle_t);
        std::vector<char> all((size_t)c->nranks * hb);
        if (c->hag) {
            if (c->hag(&h, all.data(), hb, c->hag_ctx) != 0) return gbs::fail_msg(GBS_ERROR_NCCL, "host allgather failed");
        } else {
            CUDA_OK(cudaMemcpy(c->scratch + (size_t)c->rank * hb, &h, hb, cudaMemcpyHostToDevice));
            NCCL_OK(ncclAllGather(c->scratch + (size_t)c->rank * hb, c->scratch, hb, ncclChar, c->nc, st));
            CUDA_OK(cudaStreamSynchronize(st));
            CUDA_OK(cudaMemcpy(all.data(), c->scratch, all.size(), cudaMemcpyDeviceToHost));
        }
        for (int k = 0; k < c->nranks && ok; ++k) {
            if (k == c->rank) continue;
            cudaIpcMemHandle_t hk;
            memcpy(&hk, all.data() + (size_t)k * hb, hb);
            if (cudaIpcOpenMemHandle(&c->peer_base[k], hk, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                c->peer_base[k] = nullptr;
                ok = 0;
            }
        }
        cudaGetLastError();
        // every rank must agree on the path
        if (c->hag) {
            std::vector<int> oks(c->nranks);
            if (c->hag(&ok, oks.data(), sizeof ok, c->hag_ctx) != 0) return gbs::fail_msg(GBS_ERROR_NCCL, "host allgather failed");
            for (int v : oks) ok = std::min(ok, v);
        } else {
            int* d_ok = reinterpret_cast<int*>(c->scratch);
            CUDA_OK(cudaMemcpy(d_ok, &ok, sizeof ok, cudaMemcpyHostToDevice));
            NCCL_OK(ncclAllReduce(d_ok, d_ok, 1, ncclInt, ncclMin, c->nc, st));
            CUDA_OK(cudaStreamSynchronize(st));
            CUDA_OK(cudaMemcpy(&ok, d_ok, sizeof ok, cudaMemcpyDeviceToHost));
        }
    } else if (c->nranks > 1) {
        ok = 0;
    }
    c->p2p = ok != 0;
    if (c->nranks > 1 && !c->p2p && !c->nc)
        return gbs::fail_msg(GBS_ERROR_UNSUPPORTED, "peer windows could not be mapped and the communicator has no NCCL");
    return GBS_SUCCESS;
}

// One rank's context: local workspace, window (own + peers), stream.
struct RankCtx {
    const uint32_t* in;
    uint32_t* out;
    char* ws;
    size_t n_local;
    int p, rank;
    uint32_t s_r, nq;
    DistLayout L;
    WinLayout W;
    char* win;                      // own window
    uint32_t* shard;                // W (sorted shard)
    u64* words;
    cudaStream_t st;
};

gbs_status_t rank_ctx(RankCtx& c, const uint32_t* in, uint32_t* out, void* ws, char* win, size_t n_local, int p, int rank,
                      cudaStream_t st)
{
    c.in = in;
    c.out = out;
    c.ws = reinterpret_cast<char*>(ws);
    c.n_local = n_local;
    c.p = p;
    c.rank = rank;
    c.s_r = s_r_of(n_local);
    c.nq = (uint32_t)p * c.s_r;
    c.st = st;
    c.win = win;
    gbs_status_t r = dist_layout(n_local, p, &c.L);
    if (r) return r;
    c.W = win_layout(n_local, p);
    c.shard = reinterpret_cast<uint32_t*>(c.ws + c.L.shard);
    c.words = reinterpret_cast<u64*>(c.ws + c.L.words);
    return GBS_SUCCESS;
}

template <typename T>
T* at(char* base, size_t off) { return reinterpret_cast<T*>(base + off); }

// E1: local sort (out of place) d_in -> W; zero the result words
gbs_status_t phase_local(const RankCtx& c)
{
    CUDA_OK(cudaMemsetAsync(c.words, 0, 4 * 8, c.st));
    return gbs::sort_keys_oop(c.in, c.shard, c.n_local, c.ws + c.L.sort_ws, c.L.sort_ws_bytes, c.st);
}

// E2 (+E3): samples into the gathered arrays of `ndst` windows (device pointer table)
gbs_status_t phase_samples(const RankCtx& c, u64* const* d_dst, int ndst, size_t slot0)
{
    k_dist_samples<<<(c.s_r + 255) / 256, 256, 0, c.st>>>(c.shard, c.n_local, c.s_r, c.rank, d_dst, ndst, slot0);
    CUDA_OK(cudaGetLastError());
    return GBS_SUCCESS;
}

// E4 sort the gathered samples in the own window; E5-E6 (+E7) fine cuts to ndst windows
gbs_status_t phase_cuts(const RankCtx& c, u64* const* d_dst, int ndst, size_t row0)
{
    u64* g = at<u64>(c.win, c.W.gathered);
    gbs_status_t r = gbs::sort_u64_inplace(g, c.nq, c.ws + c.L.u64ws, c.L.u64ws_bytes, c.st);
    if (r) return r;
    k_dist_finecuts<<<(c.nq + 127) / 128, 128, 0, c.st>>>(c.shard, c.n_local, (uint64_t)c.rank * c.n_local, g, c.nq,
                                                          d_dst, ndst, row0);
    CUDA_OK(cudaGetLastError());
    return GBS_SUCCESS;
}

// E8 push to the p receive buffers (device pointer table)
gbs_status_t phase_push(const RankCtx& c, uint32_t* const* d_recv)
{
    const unsigned gx = std::max(1u, (unsigned)std::min<size_t>(256, c.n_local / ((size_t)c.p * 8 * 256) + 1));
    k_dist_push<<<dim3(gx, c.p), 256, 0, c.st>>>(c.shard, at<u64>(c.win, c.W.fcut), c.nq, c.s_r, c.p, c.rank, d_recv,
                                                c.words + 1);
    CUDA_OK(cudaGetLastError());
    return GBS_SUCCESS;
}

// E9 k-way merge recv -> out; n_out into words[0]
gbs_status_t phase_merge(const RankCtx& c)
{
    // 64 KB of dynamic shared memory (a per-device attribute: set on every call, cheap)
    cudaFuncSetAttribute(k_kway_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * KM_PAD_CAP * 4);
    k_kway_merge<<<c.s_r, KM_BLOCK, 2 * KM_PAD_CAP * 4, c.st>>>(at<uint32_t>(c.win, c.W.recv), at<u64>(c.win, c.W.fcut), c.nq,
                                                           c.s_r, c.p, c.rank, c.out, c.words);
    CUDA_OK(cudaGetLastError());
    return GBS_SUCCESS;
}

// ------------------------------------------------------------------ phase profiling
struct DistProf {
    bool on = false;
    float ms[6] = {};
    double sent = 0;
    int calls = 0, path = 0;
};
thread_local DistProf g_dprof;

}  // namespace

extern "C" {

gbs_status_t gbs_get_unique_id(uint8_t id[GBS_UNIQUE_ID_BYTES])
{
    static_assert(sizeof(ncclUniqueId) == GBS_UNIQUE_ID_BYTES, "ncclUniqueId size");
    if (!id) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "id is NULL");
    ncclUniqueId u;
    NCCL_OK(ncclGetUniqueId(&u));
    memcpy(id, &u, sizeof u);
    return GBS_SUCCESS;
}

gbs_status_t gbs_comm_init(gbs_comm_t* comm, const uint8_t id[GBS_UNIQUE_ID_BYTES], int nranks, int rank)
{
    if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks)
        return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_comm_init: bad arguments");
    if (nranks > MAX_RANKS) return gbs::fail_msg(GBS_ERROR_UNSUPPORTED, "gbs_comm_init: more than 16 ranks");
    ncclUniqueId u;
    memcpy(&u, id, sizeof u);
    gbs_comm* c = new (std::nothrow) gbs_comm();
    if (!c) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "out of host memory");
    c->nranks = nranks;
    c->rank = rank;
    c->mode = 0;
    cudaGetDevice(&c->device);
    if (cudaMallocHost(&c->h_cuts, (size_t)nranks * nranks * S_R_MAX * 8) != cudaSuccess ||
        cudaMalloc(&c->scratch, 64 * 1024) != cudaSuccess || cudaMalloc(&c->d_tab, 4 * MAX_RANKS * sizeof(void*)) != cudaSuccess) {
        if (c->h_cuts) cudaFreeHost(c->h_cuts);
        if (c->scratch) cudaFree(c->scratch);
        delete c;
        return gbs::fail_msg(GBS_ERROR_CUDA, "gbs_comm_init: allocation failed");
    }
    for (auto& e : c->ev) cudaEventCreate(&e);
    ncclResult_t r = ncclCommInitRank(&c->nc, nranks, u, rank);
    if (r != ncclSuccess) {
        cudaFreeHost(c->h_cuts);
        cudaFree(c->scratch);
        cudaFree(c->d_tab);
        delete c;
        return gbs::fail_msg(GBS_ERROR_NCCL, ncclGetErrorString(r));
    }
    *comm = c;
    return GBS_SUCCESS;
}

gbs_status_t gbs_comm_init_host(gbs_comm_t* comm, int nranks, int rank, gbs_host_allgather_fn allgather, void* ctx)
{
    if (!comm || !allgather || nranks < 1 || rank < 0 || rank >= nranks)
        return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_comm_init_host: bad arguments");
    if (nranks > MAX_RANKS) return gbs::fail_msg(GBS_ERROR_UNSUPPORTED, "gbs_comm_init_host: more than 16 ranks");
    gbs_comm* c = new (std::nothrow) gbs_comm();
    if (!c) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "out of host memory");
    c->nranks = nranks;
    c->rank = rank;
    c->mode = 0;
    c->hag = allgather;
    c->hag_ctx = ctx;
    cudaGetDevice(&c->device);
    if (cudaMallocHost(&c->h_cuts, 8) != cudaSuccess || cudaMalloc(&c->scratch, 64 * 1024) != cudaSuccess ||
        cudaMalloc(&c->d_tab, 4 * MAX_RANKS * sizeof(void*)) != cudaSuccess) {
        if (c->h_cuts) cudaFreeHost(c->h_cuts);
        if (c->scratch) cudaFree(c->scratch);
        delete c;
        return gbs::fail_msg(GBS_ERROR_CUDA, "gbs_comm_init_host: allocation failed");
    }
    for (auto& e : c->ev) cudaEventCreate(&e);
    *comm = c;
    return GBS_SUCCESS;
}

gbs_status_t gbs_comm_set_exchange(gbs_comm_t comm, int mode)
{
    if (!comm || mode < 0 || mode > 1) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_comm_set_exchange: bad arguments");
    if (mode == 1 && !comm->nc) return gbs::fail_msg(GBS_ERROR_UNSUPPORTED, "a host-bootstrapped communicator has no NCCL");
    if (comm->mode != mode) {
        cudaDeviceSynchronize();
        close_window(comm);
        comm->mode = mode;
    }
    return GBS_SUCCESS;
}

gbs_status_t gbs_comm_destroy(gbs_comm_t comm)
{
    if (!comm) return GBS_SUCCESS;
    cudaDeviceSynchronize();
    close_window(comm);
    ncclResult_t r = comm->nc ? ncclCommDestroy(comm->nc) : ncclSuccess;
    cudaFreeHost(comm->h_cuts);
    cudaFree(comm->scratch);
    cudaFree(comm->d_tab);
    for (auto e : comm->ev) cudaEventDestroy(e);
    delete comm;
    return r == ncclSuccess ? GBS_SUCCESS : gbs::fail_msg(GBS_ERROR_NCCL, ncclGetErrorString(r));
}

gbs_status_t gbs_sort_keys_dist_workspace_size(size_t n_local, int nranks, size_t* ws_bytes, size_t* out_capacity)
{
    if (!ws_bytes || !out_capacity || nranks < 1) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "bad arguments");
    if ((uint64_t)n_local * nranks > (1ull << 32)) return gbs::fail_msg(GBS_ERROR_UNSUPPORTED, "N > 2^32");
    if (nranks > MAX_RANKS) return gbs::fail_msg(GBS_ERROR_UNSUPPORTED, "more than 16 ranks");
    DistLayout L;
    gbs_status_t r = dist_layout(n_local, nranks, &L);
    if (r) return r;
    *ws_bytes = nranks == 1 ? L.sort_ws_bytes : L.total;
    *out_capacity = nranks == 1 ? n_local : out_cap(n_local, nranks);
    return GBS_SUCCESS;
}

gbs_status_t gbs_sort_keys_dist_emulated_workspace_size(size_t n_local, int p, size_t* bytes)
{
    size_t w = 0, cap = 0;
    if (!bytes || p < 1) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "bad arguments");
    gbs_status_t r = gbs_sort_keys_dist_workspace_size(n_local, p, &w, &cap);
    if (r) return r;
    DistLayout L;
    r = dist_layout(n_local, p, &L);
    if (r) return r;
    *bytes = (size_t)p * (al(L.total) + al(win_layout(n_local, p).total)) + al(4 * MAX_RANKS * sizeof(void*));
    return GBS_SUCCESS;
}

// Host-side exchange plan (E7-E8 counts from the splitters' cuts), kept for tests of the
// protocol: cuts p x p row-major, cuts[r*p + k] = #items of rank r's sorted shard <=
// splitter k (cuts[r*p + p-1] = n_local).
gbs_status_t gbs_exchange_plan(const uint64_t* cuts, int p, int rank, uint64_t* send_off, uint64_t* send_cnt,
                               uint64_t* recv_off, uint64_t* recv_cnt, uint64_t* n_out)
{
    if (!cuts || p < 1 || rank < 0 || rank >= p || !send_off || !send_cnt || !recv_off || !recv_cnt || !n_out)
        return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_exchange_plan: bad arguments");
    for (int r = 0; r < p; ++r) {
        for (int k = 1; k < p; ++k)
            if (cuts[(size_t)r * p + k] < cuts[(size_t)r * p + k - 1])
                return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_exchange_plan: cuts not monotone");
        if (cuts[(size_t)r * p + p - 1] != cuts[(size_t)rank * p + p - 1])
            return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_exchange_plan: ranks disagree on n_local");
    }
    for (int k = 0; k < p; ++k) {
        const uint64_t lo = k ? cuts[(size_t)rank * p + k - 1] : 0;
        send_off[k] = lo;
        send_cnt[k] = cuts[(size_t)rank * p + k] - lo;
    }
    uint64_t run = 0;
    for (int r = 0; r < p; ++r) {
        const uint64_t lo = rank ? cuts[(size_t)r * p + rank - 1] : 0;
        recv_cnt[r] = cuts[(size_t)r * p + rank] - lo;
        recv_off[r] = run;
        run += recv_cnt[r];
    }
    *n_out = run;
    return GBS_SUCCESS;
}

gbs_status_t gbs_sort_keys_dist(gbs_comm_t comm, const uint32_t* d_in, size_t n_local, uint32_t* d_out,
                                size_t out_capacity, size_t* n_out, void* d_ws, size_t ws_bytes, gbs_stream_t stream)
{
    if (!comm || !n_out || (n_local && (!d_in || !d_out)))
        return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_sort_keys_dist: NULL argument");
    const int p = comm->nranks, rank = comm->rank;
    size_t need = 0, cap = 0;
    gbs_status_t r = gbs_sort_keys_dist_workspace_size(n_local, p, &need, &cap);
    if (r) return r;
    if (out_capacity < cap) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "out_capacity below the receive bound");
    if (ws_bytes < need) return gbs::fail_msg(GBS_ERROR_WORKSPACE_TOO_SMALL, "dist workspace too small");
    if (p > 1 && n_local < 2ull * s_r_of(n_local)) return gbs::fail_msg(GBS_ERROR_UNSUPPORTED, "n_local too small");
    if (n_local == 0) { *n_out = 0; return GBS_SUCCESS; }
    cudaStream_t st = (cudaStream_t)stream;
    const bool prof = gbs::profiling();
    if (prof) cudaEventRecord(comm->ev[0], st);
    if (p == 1) {   // one rank: the local sort is the whole job (no exchange, no copy, no sync)
        r = gbs::sort_keys_oop(d_in, d_out, n_local, d_ws, ws_bytes, st);
        if (r) return r;
        *n_out = n_local;
        if (prof) {
            cudaEventRecord(comm->ev[1], st);
            cudaEventSynchronize(comm->ev[1]);
            float ms = 0;
            cudaEventElapsedTime(&ms, comm->ev[0], comm->ev[1]);
            g_dprof.ms[0] += ms;
            g_dprof.ms[5] += ms;
            g_dprof.calls += 1;
            g_dprof.path = 0;
        }
        return GBS_SUCCESS;
    }
    const WinLayout W = win_layout(n_local, p);
    r = ensure_window(comm, W.total, st);
    if (r) return r;
    RankCtx c;
    r = rank_ctx(c, d_in, d_out, d_ws, comm->win, n_local, p, rank, st);
    if (r) return r;
    r = phase_local(c);                                                                   // E1
    if (r) return r;
    if (prof) cudaEventRecord(comm->ev[1], st);
    unsigned* status = reinterpret_cast<unsigned*>(comm->win + W.flags + MAX_RANKS * 8);
    void** tab = comm->d_tab;
    if (comm->p2p) {
        // pointer tables: flags, gathered, fcut rows, recv of every rank's window
        void* h[4][MAX_RANKS] = {};
        for (int k = 0; k < p; ++k) {
            char* b = reinterpret_cast<char*>(comm->peer_base[k]);
            h[0][k] = b + W.flags;
            h[1][k] = b + W.gathered;
            h[2][k] = b + W.fcut;
            h[3][k] = b + W.recv;
        }
        CUDA_OK(cudaMemcpyAsync(tab, h, sizeof h, cudaMemcpyHostToDevice, st));
        u64* const* flags = reinterpret_cast<u64* const*>(tab);
        auto barrier = [&]() -> gbs_status_t {
            k_p2p_barrier<<<1, 32, 0, st>>>(flags, p, rank, ++comm->epoch, status);
            CUDA_OK(cudaGetLastError());
            return GBS_SUCCESS;
        };
        if ((r = phase_samples(c, reinterpret_cast<u64* const*>(tab + MAX_RANKS), p, (size_t)rank * c.s_r))) return r;  // E2-E3
        if ((r = barrier())) return r;
        if ((r = phase_cuts(c, reinterpret_cast<u64* const*>(tab + 2 * MAX_RANKS), p, (size_t)rank * c.nq))) return r;  // E4-E7
        if ((r = barrier())) return r;
        if (prof) cudaEventRecord(comm->ev[2], st);
        if ((r = phase_push(c, reinterpret_cast<uint32_t* const*>(tab + 3 * MAX_RANKS)))) return r;                  // E8
        if ((r = barrier())) return r;
    } else {
        // NCCL transport: allgather samples (E3) and fine cuts (E7), grouped send/recv (E8)
        u64* smp = at<u64>(c.ws, c.L.samples);
        u64* frow = at<u64>(c.ws, c.L.frow);
        void* h[2] = {smp, frow};
        CUDA_OK(cudaMemcpyAsync(tab, h, sizeof h, cudaMemcpyHostToDevice, st));
        if ((r = phase_samples(c, reinterpret_cast<u64* const*>(tab), 1, 0))) return r;
        NCCL_OK(ncclAllGather(smp, at<u64>(comm->win, W.gathered), c.s_r, ncclUint64, comm->nc, st));
        if ((r = phase_cuts(c, reinterpret_cast<u64* const*>(tab + 1), 1, 0))) return r;
        NCCL_OK(ncclAllGather(frow, at<u64>(comm->win, W.fcut), c.nq, ncclUint64, comm->nc, st));
        // host counts: the splitters' columns of F
        std::vector<u64> F((size_t)p * c.nq);
        CUDA_OK(cudaMemcpyAsync(F.data(), at<u64>(comm->win, W.fcut), F.size() * 8, cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaStreamSynchronize(st));
        auto fc = [&](int rr, long long q) -> u64 { return q < 0 ? 0ull : F[(size_t)rr * c.nq + q]; };
        if (prof) cudaEventRecord(comm->ev[2], st);
        uint32_t* recv = at<uint32_t>(comm->win, W.recv);
        u64 sent = 0;
        NCCL_OK(ncclGroupStart());
        for (int k = 0; k < p; ++k) {
            const long long qlo = (long long)k * c.s_r - 1, qhi = (long long)(k + 1) * c.s_r - 1;
            const u64 so = fc(rank, qlo), sc = fc(rank, qhi) - so;       // our run for k
            const long long rlo = (long long)rank * c.s_r - 1, rhi = (long long)(rank + 1) * c.s_r - 1;
            u64 ro = 0;
            for (int rr = 0; rr < k; ++rr) ro += fc(rr, rhi) - fc(rr, rlo);
            const u64 rc = fc(k, rhi) - fc(k, rlo);                    // k's run for us
            if (k == rank) {
                if (sc) CUDA_OK(cudaMemcpyAsync(recv + ro, c.shard + so, sc * 4, cudaMemcpyDeviceToDevice, st));
                continue;
            }
            sent += sc * 4;
            if (sc) NCCL_OK(ncclSend(c.shard + so, sc, ncclUint32, k, comm->nc, st));
            if (rc) NCCL_OK(ncclRecv(recv + ro, rc, ncclUint32, k, comm->nc, st));
        }
        NCCL_OK(ncclGroupEnd());
        CUDA_OK(cudaMemcpyAsync(c.words + 1, &sent, 8, cudaMemcpyHostToDevice, st));
    }
    if (prof) cudaEventRecord(comm->ev[3], st);
    r = phase_merge(c);                                                                   // E9
    if (r) return r;
    if (prof) cudaEventRecord(comm->ev[4], st);
    u64 words[2];
    unsigned stat = 0;
    CUDA_OK(cudaMemcpyAsync(words, c.words, 16, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaMemcpyAsync(&stat, status, 4, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));                                                  // the one sync (n_out)
    if (stat) return gbs::fail_msg(GBS_ERROR_NCCL, "peer barrier timed out (a rank did not join the exchange)");
    if (words[0] > out_capacity) return gbs::fail_msg(GBS_ERROR_CUDA, "receive count exceeds the proven bound");
    *n_out = words[0];
    if (prof) {
        float ms[4];
        for (int k = 0; k < 4; ++k) cudaEventElapsedTime(&ms[k], comm->ev[k], comm->ev[k + 1]);
        g_dprof.ms[0] += ms[0];              // E1
        g_dprof.ms[1] += ms[1];              // E2-E7 (samples, cuts, barriers / allgathers)
        g_dprof.ms[2] += ms[2];              // E8 (exchange + its barrier)
        g_dprof.ms[3] += ms[3];              // E9 merge
        float tot = 0;
        cudaEventElapsedTime(&tot, comm->ev[0], comm->ev[4]);
        g_dprof.ms[5] += tot;
        g_dprof.sent += (double)words[1];
        g_dprof.calls += 1;
        g_dprof.path = comm->p2p ? 1 : 2;
    }
    return GBS_SUCCESS;
}

gbs_status_t gbs_dist_profile_end(gbs_dist_times_t* out)
{
    if (!out) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "out is NULL");
    memset(out, 0, sizeof *out);
    for (int k = 0; k < 6; ++k) out->ms[k] = g_dprof.ms[k];
    out->exchange_bytes = g_dprof.sent;
    out->calls = g_dprof.calls;
    out->path = g_dprof.path;
    g_dprof = DistProf();
    gbs_step_times_t dummy;
    return gbs_profile_end(&dummy);
}

gbs_status_t gbs_sort_keys_dist_emulated(int p, const uint32_t* d_keys, size_t n_local, uint32_t* d_out,
                                         size_t out_capacity, size_t* n_out, void* d_ws, size_t ws_bytes,
                                         gbs_stream_t stream)
{
    if (p < 1 || p > MAX_RANKS || !n_out || (n_local && (!d_keys || !d_out)))
        return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_sort_keys_dist_emulated: bad arguments");
    size_t need = 0, cap = 0, total = 0;
    gbs_status_t r = gbs_sort_keys_dist_workspace_size(n_local, p, &need, &cap);
    if (r) return r;
    r = gbs_sort_keys_dist_emulated_workspace_size(n_local, p, &total);
    if (r) return r;
    if (out_capacity < cap) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "out_capacity below the receive bound");
    if (ws_bytes < total) return gbs::fail_msg(GBS_ERROR_WORKSPACE_TOO_SMALL, "emulated workspace too small");
    if (!d_ws || ((uintptr_t)d_ws & 255)) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "workspace not 256-byte aligned");
    if (p > 1 && n_local < 2ull * s_r_of(n_local)) return gbs::fail_msg(GBS_ERROR_UNSUPPORTED, "n_local too small");
    cudaStream_t st = (cudaStream_t)stream;
    if (n_local == 0) {
        for (int k = 0; k < p; ++k) n_out[k] = 0;
        return GBS_SUCCESS;
    }
    if (p == 1) {
        r = gbs::sort_keys_oop(d_keys, d_out, n_local, d_ws, ws_bytes, st);
        n_out[0] = n_local;
        return r;
    }
    // the p ranks' local workspaces and windows, strided by their aligned sizes
    DistLayout L;
    r = dist_layout(n_local, p, &L);
    if (r) return r;
    const WinLayout W = win_layout(n_local, p);
    char* base = reinterpret_cast<char*>(d_ws);
    const size_t lstride = al(L.total), wstride = al(W.total);
    char* wins = base + (size_t)p * lstride;
    void** tab = reinterpret_cast<void**>(wins + (size_t)p * wstride);
    CUDA_OK(cudaMemsetAsync(wins, 0, (size_t)p * wstride, st));
    std::vector<RankCtx> c(p);
    void* h[4][MAX_RANKS] = {};
    for (int k = 0; k < p; ++k) {
        r = rank_ctx(c[k], d_keys + (size_t)k * n_local, d_out + (size_t)k * out_capacity, base + (size_t)k * lstride,
                     wins + (size_t)k * wstride, n_local, p, k, st);
        if (r) return r;
        char* b = c[k].win;
        h[0][k] = b + W.flags;
        h[1][k] = b + W.gathered;
        h[2][k] = b + W.fcut;
        h[3][k] = b + W.recv;
    }
    CUDA_OK(cudaMemcpyAsync(tab, h, sizeof h, cudaMemcpyHostToDevice, st));
    // the phases of all ranks in turn; stream order stands in for the device barriers
    // (profiling: events between the phases, summed over the ranks)
    const bool prof = gbs::profiling();
    cudaEvent_t ev[5] = {};
    if (prof)
        for (auto& e : ev) CUDA_OK(cudaEventCreate(&e));
    if (prof) cudaEventRecord(ev[0], st);
    for (int k = 0; k < p; ++k)
        if ((r = phase_local(c[k]))) return r;                                             // E1
    if (prof) cudaEventRecord(ev[1], st);
    for (int k = 0; k < p; ++k)
        if ((r = phase_samples(c[k], reinterpret_cast<u64* const*>(tab + MAX_RANKS), p, (size_t)k * c[k].s_r))) return r;
    for (int k = 0; k < p; ++k)
        if ((r = phase_cuts(c[k], reinterpret_cast<u64* const*>(tab + 2 * MAX_RANKS), p, (size_t)k * c[k].nq))) return r;
    if (prof) cudaEventRecord(ev[2], st);
    for (int k = 0; k < p; ++k)
        if ((r = phase_push(c[k], reinterpret_cast<uint32_t* const*>(tab + 3 * MAX_RANKS)))) return r;   // E8
    if (prof) cudaEventRecord(ev[3], st);
    for (int k = 0; k < p; ++k)
        if ((r = phase_merge(c[k]))) return r;                                             // E9
    if (prof) cudaEventRecord(ev[4], st);
    std::vector<u64> words((size_t)p * 4);
    for (int k = 0; k < p; ++k) CUDA_OK(cudaMemcpyAsync(&words[(size_t)k * 4], c[k].words, 32, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    for (int k = 0; k < p; ++k) {
        if (words[(size_t)k * 4] > out_capacity) return gbs::fail_msg(GBS_ERROR_CUDA, "receive count exceeds the bound");
        n_out[k] = words[(size_t)k * 4];
    }
    if (prof) {
        float ms[4], tot = 0;
        for (int k = 0; k < 4; ++k) cudaEventElapsedTime(&ms[k], ev[k], ev[k + 1]);
        cudaEventElapsedTime(&tot, ev[0], ev[4]);
        for (int k = 0; k < 4; ++k) g_dprof.ms[k] += ms[k];
        g_dprof.ms[5] += tot;
        for (int k = 0; k < p; ++k) g_dprof.sent += (double)words[(size_t)k * 4 + 1];
        g_dprof.calls += 1;
        g_dprof.path = 3;
        for (auto e : ev) cudaEventDestroy(e);
    }
    return GBS_SUCCESS;
}

}  // extern "C"
