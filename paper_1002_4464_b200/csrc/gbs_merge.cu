// gbs_merge.cu -- merge of p sorted runs (E9 of the multi-GPU outer level).
//
// A rank receives one sorted run from every rank (E8); sorting what it received is a
// p-way merge.  Pairwise merge-path tree: ceil(log2 p) passes, each pass one partition
// launch (merge-path split of every output tile, all pairs at once) and one merge
// launch (a CTA per output tile: both input ranges staged in shared memory, a serial
// merge per thread, coalesced write-back).  Ties keep run order (stable).
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "gbs_internal.h"

namespace {

constexpr int MT_BLOCK = 256;
constexpr int MT_ITEMS = 16;
constexpr int MT_TILE = MT_BLOCK * MT_ITEMS;   // outputs per CTA
constexpr int MAX_RUNS = 64;

struct PairDesc {
    unsigned long long a_off, na, b_off, nb, c_off;   // element offsets into src / dst
    unsigned long long tile0;                          // first global tile index of the pair
};

__device__ __forceinline__ int find_pair(const PairDesc* d, int npairs, unsigned long long g)
{
    int k = 0;
    while (k + 1 < npairs && d[k + 1].tile0 <= g) ++k;
    return k;
}

// split[g + pair] = #A items among the first min(t * TILE, na + nb) outputs of pair's merge,
// for t = 0..ntiles(pair) (g = tile0 of the pair); one thread per split point.
__global__ void k_merge_partition(const uint32_t* src, const PairDesc* d, int npairs, unsigned long long total_tiles,
                                  unsigned long long* splits)
{
    const unsigned long long idx = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= total_tiles + npairs) return;
    // split points of pair k occupy [tile0_k + k, tile0_{k+1} + k + 1)
    int k = 0;
    while (k + 1 < npairs && d[k + 1].tile0 + k + 1 <= idx) ++k;
    const PairDesc p = d[k];
    const unsigned long long t = idx - p.tile0 - k;
    const unsigned long long q = min(t * MT_TILE, p.na + p.nb);
    const uint32_t* A = src + p.a_off;
    const uint32_t* B = src + p.b_off;
    unsigned long long lo = q > p.nb ? q - p.nb : 0, hi = min(q, p.na);
    while (lo < hi) {
        const unsigned long long mid = (lo + hi) / 2;
        if (A[mid] <= B[q - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    splits[idx] = lo;
}

__global__ void __launch_bounds__(MT_BLOCK) k_merge_tile(const uint32_t* src, uint32_t* dst, const PairDesc* d, int npairs,
                                                         const unsigned long long* splits)
{
    __shared__ uint32_t s[MT_TILE + MT_TILE / MT_ITEMS + 2];
    const unsigned long long g = blockIdx.x;
    const int k = find_pair(d, npairs, g);
    const PairDesc p = d[k];
    const unsigned long long t = g - p.tile0;
    const unsigned long long q0 = t * MT_TILE, q1 = min(q0 + MT_TILE, p.na + p.nb);
    const unsigned long long a0 = splits[g + k], a1 = splits[g + k + 1];
    const unsigned long long b0 = q0 - a0, b1 = q1 - a1;
    const int la = (int)(a1 - a0), lb = (int)(b1 - b0), tot = la + lb;
    const uint32_t* A = src + p.a_off + a0;
    const uint32_t* B = src + p.b_off + b0;
    for (int i = threadIdx.x; i < la; i += MT_BLOCK) s[i] = A[i];
    for (int i = threadIdx.x; i < lb; i += MT_BLOCK) s[la + i] = B[i];
    __syncthreads();
    uint32_t out[MT_ITEMS];
    const int dg = threadIdx.x * MT_ITEMS;
    if (dg < tot) {
        int lo = max(0, dg - lb), hi = min(dg, la);
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (s[mid] <= s[la + dg - 1 - mid]) lo = mid + 1; else hi = mid;
        }
        int i = lo, j = dg - lo;
#pragma unroll
        for (int r = 0; r < MT_ITEMS; ++r) {
            const bool takeA = i < la && (j >= lb || s[i] <= s[la + j]);
            out[r] = takeA ? s[i] : s[la + j];
            i += takeA ? 1 : 0;
            j += takeA ? 0 : 1;
        }
    }
    __syncthreads();
    if (dg < tot) {
#pragma unroll
        for (int r = 0; r < MT_ITEMS; ++r) {
            const int o = dg + r;
            s[o + o / MT_ITEMS] = out[r];   // padded: conflict-free blocked stores
        }
    }
    __syncthreads();
    uint32_t* C = dst + p.c_off + q0;
    for (int o = threadIdx.x; o < tot; o += MT_BLOCK) C[o] = s[o + o / MT_ITEMS];
}

size_t al(size_t x) { return (x + 255) / 256 * 256; }

struct MergeLayout {
    size_t tmp, desc, splits, total;
};

MergeLayout merge_layout(size_t n, int p)
{
    MergeLayout L;
    size_t o = 0;
    L.tmp = o;    o += al(n * 4);
    L.desc = o;   o += al(sizeof(PairDesc) * (MAX_RUNS / 2 + 1));
    L.splits = o; o += al(8 * (n / MT_TILE + 2 * MAX_RUNS + 2));
    L.total = o;
    (void)p;
    return L;
}

}  // namespace

extern "C" {

gbs_status_t gbs_merge_runs_workspace_size(size_t n, int p, size_t* bytes)
{
    if (!bytes || p < 1 || p > MAX_RUNS) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_merge_runs_workspace_size: bad arguments");
    *bytes = merge_layout(n, p).total;
    return GBS_SUCCESS;
}

gbs_status_t gbs_merge_runs(uint32_t* d_keys, const uint64_t* run_off, int p, void* d_ws, size_t ws_bytes,
                            gbs_stream_t stream)
{
    if (!run_off || p < 1 || p > MAX_RUNS) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_merge_runs: bad arguments");
    if (run_off[0] != 0) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_merge_runs: run_off[0] != 0");
    for (int r = 0; r < p; ++r)
        if (run_off[r + 1] < run_off[r]) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_merge_runs: offsets decrease");
    const size_t n = run_off[p];
    if (n == 0 || p == 1) return GBS_SUCCESS;
    if (!d_keys || !d_ws) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_merge_runs: NULL buffer");
    const MergeLayout L = merge_layout(n, p);
    if (ws_bytes < L.total) return gbs::fail_msg(GBS_ERROR_WORKSPACE_TOO_SMALL, "gbs_merge_runs: workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    char* w = reinterpret_cast<char*>(d_ws);
    uint32_t* bufs[2] = {d_keys, reinterpret_cast<uint32_t*>(w + L.tmp)};
    PairDesc* ddesc = reinterpret_cast<PairDesc*>(w + L.desc);
    unsigned long long* dsplit = reinterpret_cast<unsigned long long*>(w + L.splits);
    std::vector<uint64_t> off(run_off, run_off + p + 1);
    int cur = 0;
    static thread_local PairDesc hdesc[MAX_RUNS / 2 + 1];
    while (off.size() > 2) {
        const int runs = (int)off.size() - 1;
        std::vector<uint64_t> noff{0};
        int npairs = 0;
        unsigned long long tiles = 0;
        for (int r = 0; r < runs; r += 2) {
            if (r + 1 < runs) {
                PairDesc& d = hdesc[npairs++];
                d.a_off = off[r];
                d.na = off[r + 1] - off[r];
                d.b_off = off[r + 1];
                d.nb = off[r + 2] - off[r + 1];
                d.c_off = off[r];
                d.tile0 = tiles;
                tiles += (d.na + d.nb + MT_TILE - 1) / MT_TILE;
                noff.push_back(off[r + 2]);
            } else {   // odd run out: copied through
                const size_t len = off[r + 1] - off[r];
                if (len && cudaMemcpyAsync(bufs[cur ^ 1] + off[r], bufs[cur] + off[r], len * 4,
                                           cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                    return gbs::fail_msg(GBS_ERROR_CUDA, "gbs_merge_runs: copy failed");
                noff.push_back(off[r + 1]);
            }
        }
        if (cudaMemcpyAsync(ddesc, hdesc, sizeof(PairDesc) * npairs, cudaMemcpyHostToDevice, st) != cudaSuccess)
            return gbs::fail_msg(GBS_ERROR_CUDA, "gbs_merge_runs: descriptor copy failed");
        const unsigned long long nsplit = tiles + npairs;
        k_merge_partition<<<(unsigned)((nsplit + 255) / 256), 256, 0, st>>>(bufs[cur], ddesc, npairs, tiles, dsplit);
        if (tiles) k_merge_tile<<<(unsigned)tiles, MT_BLOCK, 0, st>>>(bufs[cur], bufs[cur ^ 1], ddesc, npairs, dsplit);
        if (cudaGetLastError() != cudaSuccess) return gbs::fail_msg(GBS_ERROR_CUDA, "gbs_merge_runs: launch failed");
        // the host descriptor array is reused next pass: the copy above must have consumed it
        if (cudaStreamSynchronize(st) != cudaSuccess) return gbs::fail_msg(GBS_ERROR_CUDA, "gbs_merge_runs: sync failed");
        cur ^= 1;
        off.swap(noff);
    }
    if (cur != 0 && cudaMemcpyAsync(d_keys, bufs[cur], n * 4, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return gbs::fail_msg(GBS_ERROR_CUDA, "gbs_merge_runs: final copy failed");
    return GBS_SUCCESS;
}

}  // extern "C"
