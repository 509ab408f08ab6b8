// gbs_dist.cu -- multi-GPU GPU Bucket Sort.
//
// The paper is single-GPU.  Across the GPUs of one box we apply Alg. 1 once more as
// an outer level with one sublist per rank (parallel sorting by regular sampling,
// the scheme [Schaeffer] behind the paper's bucket bound):
//   E1 local GBS of the shard (the whole single-GPU path = the outer Step 2)
//   E2 s_r regular samples per rank, composites (key, global position)  (Step 3)
//   E3 ncclAllGather of the samples                                       (Step 4 input)
//   E4 every rank sorts the p*s_r samples identically (no broadcast)      (Step 4)
//   E5 splitters G_k = sorted[(k+1) s_r - 1]                              (Step 5)
//   E6 cut points by bisection in the sorted shard                        (Step 6)
//   E7 allgather of the p x p cut matrix, one D2H + stream sync           (Step 7)
//   E8 grouped ncclSend/ncclRecv over NVLink: contiguous runs, no pack    (Step 8)
//   E9 p-way merge of the received runs (gbs_merge_runs, gbs_merge.cu)   (Step 9)
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "gbs_internal.h"

struct gbs_comm {
    ncclComm_t nc;
    int nranks, rank;
    unsigned long long* h_cuts;   // pinned p*p
};

namespace {

constexpr uint32_t S_R_MAX = 1024;   // regular samples per rank (E2)

// s_r: the largest power of two <= S_R_MAX that divides n_local, so the regular
// sample positions (k+1) n_l / s_r - 1 are exactly equidistant (d = n_l / s_r).
uint32_t s_r_of(size_t n_local)
{
    uint32_t s = 1;
    while (s < S_R_MAX && n_local % (2ull * s) == 0) s *= 2;
    return s;
}

size_t out_cap(size_t n_local, int p)
{
    const size_t d = n_local / s_r_of(n_local);
    return n_local + (size_t)(p - 1) * (d - 1);
}

size_t al(size_t x) { return (x + 255) / 256 * 256; }

__global__ void k_dist_samples(const uint32_t* keys, size_t n_local, uint32_t s_r, uint64_t gbase,
                               unsigned long long* out)
{
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= s_r) return;
    const size_t d = n_local / s_r;
    const size_t pos = (size_t)(k + 1) * d - 1;
    out[k] = ((unsigned long long)keys[pos] << 32) | (unsigned long long)(uint32_t)(gbase + pos);
}

// E5 + E6: cut_k = #{pos : (S[pos], gbase + pos) <= G_k}, G_k = sorted[(k+1) s_r - 1].
__global__ void k_dist_cuts(const uint32_t* keys, size_t n_local, uint64_t gbase, const unsigned long long* sorted,
                            uint32_t s_r, int p, unsigned long long* cuts)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= p) return;
    const unsigned long long g = sorted[(size_t)(k + 1) * s_r - 1];
    size_t lo = 0, hi = n_local;
    while (lo < hi) {
        const size_t mid = (lo + hi) / 2;
        const unsigned long long c = ((unsigned long long)keys[mid] << 32) | (unsigned long long)(uint32_t)(gbase + mid);
        if (c <= g) lo = mid + 1; else hi = mid;
    }
    cuts[k] = lo;
}

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

struct DistLayout {
    size_t sort_ws, samples, gathered, cuts, all_cuts, u64ws, u64ws_bytes, total;
};

gbs_status_t dist_layout(size_t n_local, int p, DistLayout* L)
{
    size_t a = 0, b = 0;
    gbs_status_t r = gbs_sort_keys_workspace_size(n_local, &a);
    if (r) return r;
    r = gbs_merge_runs_workspace_size(out_cap(n_local, p), p, &b);     // E9 (p-way merge)
    if (r) return r;
    const uint32_t s_r = s_r_of(n_local);
    L->sort_ws = 0;
    size_t o = al(a > b ? a : b);
    L->samples = o;  o += al((size_t)s_r * 8);
    L->gathered = o; o += al((size_t)p * s_r * 8);
    L->cuts = o;     o += al((size_t)p * 8);
    L->all_cuts = o; o += al((size_t)p * p * 8);
    size_t u = 0;
    r = gbs::sort_u64_ws((size_t)p * s_r, &u);
    if (r) return r;
    L->u64ws = o;    o += al(u);
    L->u64ws_bytes = u;
    L->total = o;
    return GBS_SUCCESS;
}

}  // namespace

extern "C" {

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
    ncclUniqueId u;
    memcpy(&u, id, sizeof u);
    gbs_comm* c = new (std::nothrow) gbs_comm();
    if (!c) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "out of host memory");
    c->nranks = nranks;
    c->rank = rank;
    if (cudaMallocHost(&c->h_cuts, (size_t)nranks * nranks * 8) != cudaSuccess) {
        delete c;
        return gbs::fail_msg(GBS_ERROR_CUDA, "cudaMallocHost failed");
    }
    ncclResult_t r = ncclCommInitRank(&c->nc, nranks, u, rank);
    if (r != ncclSuccess) {
        cudaFreeHost(c->h_cuts);
        delete c;
        return gbs::fail_msg(GBS_ERROR_NCCL, ncclGetErrorString(r));
    }
    *comm = c;
    return GBS_SUCCESS;
}

gbs_status_t gbs_comm_destroy(gbs_comm_t comm)
{
    if (!comm) return GBS_SUCCESS;
    ncclResult_t r = ncclCommDestroy(comm->nc);
    cudaFreeHost(comm->h_cuts);
    delete comm;
    return r == ncclSuccess ? GBS_SUCCESS : gbs::fail_msg(GBS_ERROR_NCCL, ncclGetErrorString(r));
}

gbs_status_t gbs_sort_keys_dist_workspace_size(size_t n_local, int nranks, size_t* ws_bytes, size_t* out_capacity)
{
    if (!ws_bytes || !out_capacity || nranks < 1) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "bad arguments");
    if ((uint64_t)n_local * nranks > (1ull << 32)) return gbs::fail_msg(GBS_ERROR_UNSUPPORTED, "N > 2^32");
    if ((size_t)nranks * s_r_of(n_local) > 16384) return gbs::fail_msg(GBS_ERROR_UNSUPPORTED, "too many ranks");
    DistLayout L;
    gbs_status_t r = dist_layout(n_local, nranks, &L);
    if (r) return r;
    *ws_bytes = L.total;
    *out_capacity = out_cap(n_local, nranks);
    return GBS_SUCCESS;
}

}  // extern "C"

namespace {

// One rank's view of E1-E9: the phases between the collectives, shared by the NCCL path
// and the single-GPU emulation (gbs_sort_keys_dist_emulated).
struct RankCtx {
    uint32_t* keys;
    uint32_t* out;
    char* ws;
    size_t n_local;
    int p, rank;
    uint32_t s_r;
    DistLayout L;
    unsigned long long *samples, *gathered, *cuts, *all_cuts;
    cudaStream_t st;
};

gbs_status_t rank_ctx(RankCtx& c, uint32_t* keys, uint32_t* out, void* ws, size_t n_local, int p, int rank,
                      cudaStream_t st)
{
    c.keys = keys;
    c.out = out;
    c.ws = reinterpret_cast<char*>(ws);
    c.n_local = n_local;
    c.p = p;
    c.rank = rank;
    c.s_r = s_r_of(n_local);
    c.st = st;
    gbs_status_t r = dist_layout(n_local, p, &c.L);
    if (r) return r;
    c.samples = reinterpret_cast<unsigned long long*>(c.ws + c.L.samples);
    c.gathered = reinterpret_cast<unsigned long long*>(c.ws + c.L.gathered);
    c.cuts = reinterpret_cast<unsigned long long*>(c.ws + c.L.cuts);
    c.all_cuts = reinterpret_cast<unsigned long long*>(c.ws + c.L.all_cuts);
    return GBS_SUCCESS;
}

// E1 local GBS of the shard, E2 regular samples (key, global position)
gbs_status_t phase_local(const RankCtx& c)
{
    gbs_status_t r = gbs_sort_keys(c.keys, c.n_local, c.ws, c.L.samples, c.st);
    if (r) return r;
    const uint64_t gbase = (uint64_t)c.rank * c.n_local;
    k_dist_samples<<<(c.s_r + 255) / 256, 256, 0, c.st>>>(c.keys, c.n_local, c.s_r, gbase, c.samples);
    CUDA_OK(cudaGetLastError());
    return GBS_SUCCESS;
}

// E4 sort the gathered p*s_r samples (identical on every rank), E5-E6 cut points
gbs_status_t phase_cuts(const RankCtx& c)
{
    gbs_status_t r = gbs::sort_u64_inplace(c.gathered, (size_t)c.p * c.s_r, c.ws + c.L.u64ws, c.L.u64ws_bytes, c.st);
    if (r) return r;
    const uint64_t gbase = (uint64_t)c.rank * c.n_local;
    k_dist_cuts<<<(c.p + 127) / 128, 128, 0, c.st>>>(c.keys, c.n_local, gbase, c.gathered, c.s_r, c.p, c.cuts);
    CUDA_OK(cudaGetLastError());
    return GBS_SUCCESS;
}

// E9: the p received runs (one per source rank, each sorted) -> one sorted run
gbs_status_t phase_merge(const RankCtx& c, const uint64_t* recv_off, uint64_t total)
{
    std::vector<uint64_t> roff(c.p + 1);
    for (int k = 0; k < c.p; ++k) roff[k] = recv_off[k];
    roff[c.p] = total;
    return gbs_merge_runs(c.out, roff.data(), c.p, c.ws, c.L.samples, c.st);
}

}  // namespace

extern "C" {

gbs_status_t gbs_sort_keys_dist(gbs_comm_t comm, uint32_t* d_keys, size_t n_local, uint32_t* d_out,
                                size_t out_capacity, size_t* n_out, void* d_ws, size_t ws_bytes, gbs_stream_t stream)
{
    if (!comm || !n_out || (n_local && (!d_keys || !d_out)))
        return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_sort_keys_dist: NULL argument");
    const int p = comm->nranks, rank = comm->rank;
    size_t need = 0, cap = 0;
    gbs_status_t r = gbs_sort_keys_dist_workspace_size(n_local, p, &need, &cap);
    if (r) return r;
    if (out_capacity < cap) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "out_capacity below the receive bound");
    if (ws_bytes < need) return gbs::fail_msg(GBS_ERROR_WORKSPACE_TOO_SMALL, "dist workspace too small");
    if (n_local == 0) { *n_out = 0; return GBS_SUCCESS; }
    cudaStream_t st = (cudaStream_t)stream;
    RankCtx c;
    r = rank_ctx(c, d_keys, d_out, d_ws, n_local, p, rank, st);
    if (r) return r;
    r = phase_local(c);                                                                   // E1-E2
    if (r) return r;
    NCCL_OK(ncclAllGather(c.samples, c.gathered, c.s_r, ncclUint64, comm->nc, st));      // E3
    r = phase_cuts(c);                                                                    // E4-E6
    if (r) return r;
    NCCL_OK(ncclAllGather(c.cuts, c.all_cuts, p, ncclUint64, comm->nc, st));             // E7
    CUDA_OK(cudaMemcpyAsync(comm->h_cuts, c.all_cuts, (size_t)p * p * 8, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    std::vector<uint64_t> so(p), sc(p), ro(p), rc(p);
    uint64_t total = 0;
    r = gbs_exchange_plan(reinterpret_cast<const uint64_t*>(comm->h_cuts), p, rank, so.data(), sc.data(), ro.data(),
                          rc.data(), &total);
    if (r) return r;
    if (total > out_capacity) return gbs::fail_msg(GBS_ERROR_CUDA, "receive count exceeds the proven bound");
    NCCL_OK(ncclGroupStart());                                                           // E8
    for (int k = 0; k < p; ++k) {
        if (k == rank) continue;
        if (sc[k]) NCCL_OK(ncclSend(d_keys + so[k], sc[k], ncclUint32, k, comm->nc, st));
        if (rc[k]) NCCL_OK(ncclRecv(d_out + ro[k], rc[k], ncclUint32, k, comm->nc, st));
    }
    NCCL_OK(ncclGroupEnd());
    if (sc[rank])
        CUDA_OK(cudaMemcpyAsync(d_out + ro[rank], d_keys + so[rank], sc[rank] * 4, cudaMemcpyDeviceToDevice, st));
    r = phase_merge(c, ro.data(), total);                                                // E9
    if (r) return r;
    *n_out = total;
    return GBS_SUCCESS;
}

gbs_status_t gbs_sort_keys_dist_emulated(int p, uint32_t* d_keys, size_t n_local, uint32_t* d_out,
                                         size_t out_capacity, size_t* n_out, void* d_ws, size_t ws_bytes,
                                         gbs_stream_t stream)
{
    if (p < 1 || !n_out || (n_local && (!d_keys || !d_out)))
        return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "gbs_sort_keys_dist_emulated: bad arguments");
    size_t need = 0, cap = 0;
    gbs_status_t r = gbs_sort_keys_dist_workspace_size(n_local, p, &need, &cap);
    if (r) return r;
    if (out_capacity < cap) return gbs::fail_msg(GBS_ERROR_INVALID_VALUE, "out_capacity below the receive bound");
    if (ws_bytes < need) return gbs::fail_msg(GBS_ERROR_WORKSPACE_TOO_SMALL, "dist workspace too small");
    if (n_local == 0) {
        for (int k = 0; k < p; ++k) n_out[k] = 0;
        return GBS_SUCCESS;
    }
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<RankCtx> c(p);
    for (int k = 0; k < p; ++k) {
        r = rank_ctx(c[k], d_keys + (size_t)k * n_local, d_out + (size_t)k * out_capacity,
                     reinterpret_cast<char*>(d_ws) + (size_t)k * ws_bytes, n_local, p, k, st);
        if (r) return r;
    }
    for (int k = 0; k < p; ++k)                                                           // E1-E2
        if ((r = phase_local(c[k]))) return r;
    for (int k = 0; k < p; ++k)                                                           // E3 (allgather)
        for (int q = 0; q < p; ++q)
            CUDA_OK(cudaMemcpyAsync(c[k].gathered + (size_t)q * c[q].s_r, c[q].samples, (size_t)c[q].s_r * 8,
                                    cudaMemcpyDeviceToDevice, st));
    for (int k = 0; k < p; ++k)                                                           // E4-E6
        if ((r = phase_cuts(c[k]))) return r;
    std::vector<unsigned long long> all((size_t)p * p);                                   // E7 (allgather)
    for (int q = 0; q < p; ++q)
        CUDA_OK(cudaMemcpyAsync(all.data() + (size_t)q * p, c[q].cuts, (size_t)p * 8, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    std::vector<std::vector<uint64_t>> so(p, std::vector<uint64_t>(p)), sc = so, ro = so, rc = so;
    std::vector<uint64_t> total(p);
    for (int k = 0; k < p; ++k) {
        r = gbs_exchange_plan(reinterpret_cast<const uint64_t*>(all.data()), p, k, so[k].data(), sc[k].data(),
                              ro[k].data(), rc[k].data(), &total[k]);
        if (r) return r;
        if (total[k] > out_capacity) return gbs::fail_msg(GBS_ERROR_CUDA, "receive count exceeds the proven bound");
    }
    for (int src = 0; src < p; ++src)                                                     // E8 (all-to-all)
        for (int dst = 0; dst < p; ++dst)
            if (sc[src][dst])
                CUDA_OK(cudaMemcpyAsync(c[dst].out + ro[dst][src], c[src].keys + so[src][dst], sc[src][dst] * 4,
                                        cudaMemcpyDeviceToDevice, st));
    for (int k = 0; k < p; ++k) {                                                         // E9
        if ((r = phase_merge(c[k], ro[k].data(), total[k]))) return r;
        n_out[k] = total[k];
    }
    return GBS_SUCCESS;
}

}  // extern "C"
