/*
 * gbs.h -- C-ABI of libgbs.so: GPU Bucket Sort, the deterministic sample sort of
 * Dehne & Zaboli, "Deterministic Sample Sort For GPUs" (arXiv 1002.4464),
 * Algorithm 1, as hand-written sm_100a kernels.
 *
 * Problem statement: "Input: an array A with n data items stored in
 * global memory.  Output: Array A sorted."  Items are 32-bit unsigned keys in
 * ascending unsigned order (the paper never fixes the item width; R1),
 * optionally with 32-bit values that move with their keys (stable by key, R7).
 *
 * Conventions (all entry points):
 *   - Device pointers are caller-owned CUDA global memory on the current device;
 *     the library allocates no device memory (except NCCL internals in
 *     gbs_comm_init).  Workspace is caller-provided, sized by the *_workspace_size
 *     queries, 256-byte aligned.
 *   - Every argument is validated BEFORE anything is enqueued; on a
 *     validation error nothing is enqueued.  n = 0 and n = 1 succeed with no work.
 *   - Work is enqueued on `stream` and completes asynchronously; device faults
 *     surface as GBS_ERROR_CUDA from this or a later call.  No call aborts or
 *     throws; gbs_last_error() holds a thread-local message for the last failure.
 *   - The result is bit-identical across runs and streams (deterministic: no
 *     atomics decide any output position).
 *   - Calls on distinct buffers/workspaces/streams may run concurrently.  Inside a call,
 *     Step 9's size tiers and the host-buffer copies run on side streams of the calling
 *     thread (forked from and joined back into `stream` with events), so a call may be
 *     captured into a CUDA graph; while that capture is open the same thread must not
 *     enqueue another call on the same device.
 *   - Latency-bound sizes (n <= 2^20, default plan): the first call with given (buffers,
 *     n, workspace) runs directly and records its launch sequence into a cached CUDA
 *     graph (32 kept, least recently used evicted); later calls with the same arguments
 *     replay it on `stream`.  Not used while `stream` is being captured, while profiling
 *     (gbs_profile_begin) or with GBS_DEBUG_SYNC.
 *   - Limits: n <= 2^31 items per call (32-bit tags, R10).
 */
#ifndef GBS_H_
#define GBS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* gbs_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    GBS_SUCCESS = 0,
    GBS_ERROR_INVALID_VALUE = 1,       /* NULL with n > 1, bad config, keys/vals overlap */
    GBS_ERROR_WORKSPACE_TOO_SMALL = 2, /* ws_bytes < the *_workspace_size query */
    GBS_ERROR_UNSUPPORTED = 3,         /* n > 2^31, device is not sm_100 */
    GBS_ERROR_CUDA = 4,                /* launch/runtime error (see gbs_last_error) */
    GBS_ERROR_NCCL = 5                 /* NCCL error in a multi-GPU call */
} gbs_status_t;

/* ------------------------------------------------------------ single GPU */

/* Bytes of device workspace gbs_sort_keys needs for n keys (depends on n only). */
gbs_status_t gbs_sort_keys_workspace_size(size_t n, size_t* bytes);

/* Sort d_keys[0..n) ascending (unsigned), IN PLACE (Alg. 1).
 * d_keys: device, 4-byte aligned.  d_ws: device workspace of >= the queried size. */
gbs_status_t gbs_sort_keys(uint32_t* d_keys, size_t n, void* d_ws, size_t ws_bytes,
                           gbs_stream_t stream);

gbs_status_t gbs_sort_pairs_workspace_size(size_t n, size_t* bytes);

/* Sort (d_keys[i], d_vals[i]) pairs by key, IN PLACE, stable: equal keys keep their
 * input order (equals std::stable_sort by key; R7).  Keys and values must not overlap. */
gbs_status_t gbs_sort_pairs(uint32_t* d_keys, uint32_t* d_vals, size_t n, void* d_ws,
                            size_t ws_bytes, gbs_stream_t stream);

/* Key types beyond unsigned 32-bit (the paper never fixes the item
 * type, R1).  Signed int32 and IEEE-754 binary32 keys are sorted as u32 keys under
 * an order-preserving bijection of their bits, applied where the keys enter the sort
 * (Step 2's load) and inverted where they leave it (the last Step 9's store), so no pass
 * is added:
 *   GBS_KEY_I32: flip the sign bit;
 *   GBS_KEY_F32: negative (sign set) -> flip every bit, otherwise flip the sign bit.
 * Float order is the IEEE-754 totalOrder of the bit patterns: -NaN < -inf < ... < -0 <
 * +0 < ... < +inf < +NaN (so -0 sorts before +0, NaNs go to the ends by sign).
 * GBS_KEY_U32 is gbs_sort_keys / gbs_sort_pairs.  Every argument is validated before the
 * first kernel; d_keys must be 4-byte aligned; workspace as gbs_sort_keys_workspace_size
 * (keys) or gbs_sort_pairs_workspace_size (pairs).  Pairs: stable by key, as
 * gbs_sort_pairs.  On GBS_ERROR_CUDA the buffers' contents are unspecified. */
typedef enum { GBS_KEY_U32 = 0, GBS_KEY_I32 = 1, GBS_KEY_F32 = 2 } gbs_key_type_t;
gbs_status_t gbs_sort_keys_typed(void* d_keys, size_t n, int key_type, void* d_ws, size_t ws_bytes,
                                 gbs_stream_t stream);
gbs_status_t gbs_sort_pairs_typed(void* d_keys, uint32_t* d_vals, size_t n, int key_type, void* d_ws,
                                  size_t ws_bytes, gbs_stream_t stream);

/* 64-bit keys (the paper never fixes the item type, R1).
 * GBS_KEY64_U64 unsigned, GBS_KEY64_I64 two's complement, GBS_KEY64_F64 IEEE-754 binary64
 * in totalOrder (-NaN < -inf < ... < -0 < +0 < ... < +inf < +NaN).  The key's
 * order-preserving u64 image is sorted as the composite (high half, low half) by two
 * stable u32 passes of the pairs GBS (low half first, each with the item index as the
 * value), then the original 8-byte keys (and the values) are gathered by the final index
 * permutation: ascending, stable (equals std::stable_sort by numeric key).  d_keys: n
 * 8-byte keys, 8-byte aligned, sorted in place; d_vals (pairs): n u32 values, not
 * overlapping the keys.  Workspace from gbs_sort64_workspace_size(n, pairs).  n <= 2^31. */
typedef enum { GBS_KEY64_U64 = 0, GBS_KEY64_I64 = 1, GBS_KEY64_F64 = 2 } gbs_key64_type_t;
gbs_status_t gbs_sort64_workspace_size(size_t n, int pairs, size_t* bytes);
gbs_status_t gbs_sort_keys64(void* d_keys, size_t n, int key_type, void* d_ws, size_t ws_bytes,
                             gbs_stream_t stream);
gbs_status_t gbs_sort_pairs64(void* d_keys, uint32_t* d_vals, size_t n, int key_type, void* d_ws,
                              size_t ws_bytes, gbs_stream_t stream);

/* End to end from HOST buffers: copy h_keys (pinned host, n keys) to d_keys, sort,
 * copy back to h_keys; all three enqueued on `stream` (H2D + sort + D2H).  Large inputs
 * are pipelined: the H2D copy is chunked by sublists so Step 2 sorts each chunk as it
 * lands, and (one-level plans) the final output is copied back bucket group by bucket
 * group while later groups sort (R18).  d_keys: device buffer of n keys
 * (scratch + result); workspace as gbs_sort_keys_workspace_size. */
gbs_status_t gbs_sort_keys_host(uint32_t* h_keys, size_t n, uint32_t* d_keys, void* d_ws,
                                size_t ws_bytes, gbs_stream_t stream);
/* The same for key-value pairs (stable by key, as gbs_sort_pairs): h_keys/h_vals pinned
 * host arrays of n items (in and out), d_keys/d_vals device buffers of n items, workspace
 * as gbs_sort_pairs_workspace_size. */
gbs_status_t gbs_sort_pairs_host(uint32_t* h_keys, uint32_t* h_vals, size_t n, uint32_t* d_keys,
                                 uint32_t* d_vals, void* d_ws, size_t ws_bytes, gbs_stream_t stream);

/* ------------------------------------------------------------ plans, stages */

/* Optional explicit level-1 parameters: sublist size L (= n/m of Step 1)
 * and sample count s (Steps 3/5).  L, s powers of two, 1 <= s <= L,
 * L <= tile capacity (32768 keys, 16384 pairs).  {0, 0} = automatic plan. */
typedef struct {
    uint32_t L;
    uint32_t s;
} gbs_config_t;

#define GBS_MAX_LEVELS 4
/* The static plan (depends on n, item kind and config only -- never on the data).
 * Level k+1, if present, sorts the buckets of level k (its problem capacity is
 * level k's tight bucket bound, cap[k+1] = bucket_bound[k]). */
typedef struct {
    int levels;                            /* 0 = a single on-chip sort */
    uint32_t L[GBS_MAX_LEVELS];
    uint32_t s[GBS_MAX_LEVELS];
    uint32_t m[GBS_MAX_LEVELS];            /* sublists per problem */
    uint64_t cap[GBS_MAX_LEVELS];          /* problem capacity at this level */
    uint64_t bucket_bound[GBS_MAX_LEVELS]; /* n'/s + (m-1)(d-1) */
    size_t ws_bytes;
    int kernels_per_sort;                  /* launches one call enqueues */
} gbs_plan_t;

/* pairs = 0: keys only; 1: key-value pairs.  cfg may be NULL. */
gbs_status_t gbs_plan(size_t n, int pairs, const gbs_config_t* cfg, gbs_plan_t* out);

gbs_status_t gbs_workspace_size_ex(size_t n, int pairs, const gbs_config_t* cfg, size_t* bytes);

/* Where the level-1 intermediates live inside the workspace (byte offsets), for
 * stage parity (tests).  Matrices are row-major [i*s + j] with m rows, s columns.
 *   samples:   m*s uint64 (key << 32 | tag); sorted in place by Step 4
 *   splitters: s uint64 (Step 5 global samples)
 *   a, l:      m*s uint32 (Step 6 bucket sizes, Step 7 offsets)
 *   relocated: n uint32 keys (Step 8 array R = B_1..B_s); pairs: values follow at
 *              relocated_vals.  Offsets are (size_t)-1 for a single-level-0 plan. */
typedef struct {
    size_t samples, splitters, a, l, relocated, relocated_vals;
} gbs_layout_t;
gbs_status_t gbs_debug_layout(size_t n, int pairs, const gbs_config_t* cfg, gbs_layout_t* out);

/* Like gbs_sort_keys / gbs_sort_pairs (d_vals may be NULL) with an explicit config,
 * stopping after level-1 Step `stop_after_step` (2..8; 0 = run to completion). */
gbs_status_t gbs_sort_ex(uint32_t* d_keys, uint32_t* d_vals, size_t n, const gbs_config_t* cfg,
                         int stop_after_step, void* d_ws, size_t ws_bytes, gbs_stream_t stream);

/* Per-step device time (CUDA events recorded on the call's stream between the steps'
 * launches; the Fig. 4 breakdown) for every complete sort this thread
 * enqueues between begin and end.  ms[2] = Steps 2-3 (local sort + local sampling),
 * ms[4] = Step 4 (sample sort), ms[5..8] = Steps 5-8, ms[9] = Step 9 (bucket sort, or
 * the whole nested level) of the top level, summed over `calls` sorts; ms_level[k][.]
 * the same for level k (k = 0 top, k >= 1 the k-th nested Step 9 level, whose steps run
 * over all buckets of the level above at once), `levels` of them.
 * gbs_profile_end synchronises the recorded events. */
typedef struct {
    float ms[10];
    int calls;
    int levels;
    float ms_level[GBS_MAX_LEVELS][10];
} gbs_step_times_t;
gbs_status_t gbs_profile_begin(void);
gbs_status_t gbs_profile_end(gbs_step_times_t* out);

const char* gbs_status_string(gbs_status_t s);
const char* gbs_last_error(void); /* thread-local */

/* ------------------------------------------------------------ multi GPU */
/* One process per GPU; a collective over all ranks of `comm`:
 * Alg. 1 once more as an outer level with one sublist per rank.  Every rank sorts its
 * shard with the single-GPU path (E1, the outer Step 2), takes s_r regular samples (E2,
 * Step 3), every rank receives all samples (E3), sorts them identically and picks the p
 * splitters G_k = sorted[(k+1) s_r - 1] (E4-E5, Steps 4-5), counts for every sorted
 * sample how many of its items are <= it (E6, Step 6), every rank receives that p x p s_r
 * matrix F (E7, Step 7), the buckets are relocated straight into their owners' receive
 * buffers at offsets derived from F (E8: the relocation of P:235-239 as the exchange) and
 * every rank merges the p sorted runs it received in one pass (E9, Step 9).
 * Transport: NVLink peer memory -- the communicator maps every rank's window (receive
 * buffer, sample slots, F, barrier flags) into every peer with CUDA IPC and E3/E7/E8 are
 * stores from the library's kernels into the peers' windows, ordered by device-side
 * barriers; where a peer cannot be mapped (or gbs_comm_set_exchange(comm, 1)), NCCL
 * allgathers and grouped send/recv carry the same data. */
typedef struct gbs_comm* gbs_comm_t;
#define GBS_UNIQUE_ID_BYTES 128 /* == sizeof(ncclUniqueId) */

gbs_status_t gbs_get_unique_id(uint8_t id[GBS_UNIQUE_ID_BYTES]);
/* Uses the current CUDA device.  Collective: every rank calls it with the same id.  At
 * most 16 ranks.  The communicator owns device memory: NCCL's, a 64 KB scratch and (from
 * the first multi-rank sort on) the peer-mapped window, sized for the largest n_local
 * sorted so far (~4.1 n_local + 8 p^2 s_r bytes). */
gbs_status_t gbs_comm_init(gbs_comm_t* comm, const uint8_t id[GBS_UNIQUE_ID_BYTES], int nranks,
                           int rank);
/* The same without NCCL: the communicator's one host-side collective -- exchanging the
 * window's IPC handles (and agreeing that every peer mapped) -- goes through `allgather`,
 * a caller-supplied blocking host allgather (each rank passes `bytes` at send, receives
 * nranks * bytes in rank order at recv; returns 0 on success).  The exchange is then
 * peer memory only (GBS_ERROR_UNSUPPORTED when a peer cannot be mapped).  This lets
 * several processes share one GPU (NCCL refuses two ranks on one device): tests run the
 * real multi-process path -- IPC windows, cross-process barriers, pushes -- on one B200. */
typedef int (*gbs_host_allgather_fn)(const void* send, void* recv, size_t bytes, void* ctx);
gbs_status_t gbs_comm_init_host(gbs_comm_t* comm, int nranks, int rank, gbs_host_allgather_fn allgather,
                                void* ctx);
/* Exchange transport: 0 = peer memory when every peer maps (default), 1 = NCCL.
 * Collective (every rank sets the same mode). */
gbs_status_t gbs_comm_set_exchange(gbs_comm_t comm, int mode);
gbs_status_t gbs_comm_destroy(gbs_comm_t comm);

/* ws_bytes: the rank's local workspace; out_capacity = n_local + (p-1)(n_local/s_r - 1),
 * the tight receive bound (s_r = the largest power of two <= 1024 dividing n_local;
 * out_capacity = n_local when nranks = 1).  N = nranks * n_local <= 2^32. */
gbs_status_t gbs_sort_keys_dist_workspace_size(size_t n_local, int nranks, size_t* ws_bytes,
                                               size_t* out_capacity);

/* Every rank passes the same n_local (>= 2 s_r when nranks > 1).  d_in (n_local keys,
 * device) is read only; d_out (out_capacity keys) receives this rank's part of the
 * global order and *n_out (host) its length.  Concatenating d_out[0:n_out] in rank order
 * gives sorted(concatenation of the inputs in rank order).  With nranks > 1 the call
 * synchronises `stream` once, at its end (to return *n_out); nranks = 1 is the
 * single-GPU sort of d_in into d_out (no synchronisation).  A rank that does not join
 * makes the others fail with GBS_ERROR_NCCL after a ~20 s timeout instead of hanging. */
gbs_status_t gbs_sort_keys_dist(gbs_comm_t comm, const uint32_t* d_in, size_t n_local,
                                uint32_t* d_out, size_t out_capacity, size_t* n_out, void* d_ws,
                                size_t ws_bytes, gbs_stream_t stream);

/* Phase times of the multi-GPU calls this thread enqueued between gbs_profile_begin()
 * and this call (which ends the profile, like gbs_profile_end): ms[0] E1 local sort,
 * ms[1] E2-E7 (samples, cuts and their exchange), ms[2] E8 exchange (incl. its barrier),
 * ms[3] E9 merge, ms[5] the whole call; exchange_bytes = keys bytes this rank sent to
 * other ranks; path 1 = peer memory, 2 = NCCL, 0 = one rank, 3 = the emulation
 * (gbs_sort_keys_dist_emulated; phases summed over its ranks). */
typedef struct {
    float ms[6];
    double exchange_bytes;
    int calls;
    int path;
} gbs_dist_times_t;
gbs_status_t gbs_dist_profile_end(gbs_dist_times_t* out);

/* The p-rank path of gbs_sort_keys_dist on ONE GPU, for testing: the same per-rank
 * kernels (E1-E9, peer-memory transport) run for ranks 0..p-1 in turn, with the p
 * windows as regions of the workspace and stream order in place of the barriers.
 * d_keys holds the p shards back to back (p*n_local keys, read only), d_out p regions of
 * out_capacity keys (rank k's part at d_out + k*out_capacity), n_out a host array of p
 * lengths, d_ws one workspace of gbs_sort_keys_dist_emulated_workspace_size bytes
 * (256-byte aligned).  Synchronises `stream` once. */
gbs_status_t gbs_sort_keys_dist_emulated_workspace_size(size_t n_local, int p, size_t* bytes);
gbs_status_t gbs_sort_keys_dist_emulated(int p, const uint32_t* d_keys, size_t n_local,
                                         uint32_t* d_out, size_t out_capacity, size_t* n_out,
                                         void* d_ws, size_t ws_bytes, gbs_stream_t stream);

/* Host-only exchange plan (E7-E8 counts from the splitters' cuts), exported so the
 * protocol can be tested without a GPU.  cuts: p x p row-major, cuts[r*p + k] = cut_{r,k}
 * (#items of rank r's sorted shard <= splitter k; cuts[r*p + p-1] = n_local).  For
 * `rank`, fills send_off/send_cnt (into its shard) and recv_off/recv_cnt (into its
 * receive buffer, source order) for each peer, and *n_out.  GBS_ERROR_INVALID_VALUE on
 * inconsistent cuts. */
gbs_status_t gbs_exchange_plan(const uint64_t* cuts, int p, int rank, uint64_t* send_off,
                               uint64_t* send_cnt, uint64_t* recv_off, uint64_t* recv_cnt,
                               uint64_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* GBS_H_ */
