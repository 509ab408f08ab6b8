"""GPU Bucket Sort for B200 -- Python binding of libgbs.so (include/gbs.h).

Argument marshalling only: every step of the sort runs in the sm_100a kernels of
``libgbs.so`` (csrc/).  PyTorch supplies device memory, streams and process
groups.  There is no CPU fallback: if the library is missing or no sm_100 device
is present, every call raises.

    import paper_1002_4464_b200 as gbs
    gbs.sort_keys(t)              # t: CUDA int32/uint32 tensor, sorted in place (unsigned)
    gbs.sort_pairs(k, v)          # stable by key, in place
    gbs.sort_keys_typed(f)        # int32 / float32 keys by value (floats: IEEE-754 totalOrder)
    gbs.sort_keys64(x)            # uint64 / int64 / float64 keys; sort_pairs64(k, v) with values
    gbs.sort_pairs_host(hk, hv, dk, dv)   # pinned host buffers in and out (copies inside)
    part = gbs.sort_keys_dist(t, gbs.Comm())   # one process per GPU (torch.distributed up)
"""
from __future__ import annotations

import ctypes as C
import functools
import os

__all__ = ["lib", "GbsError", "plan", "workspace_size", "debug_layout", "sort_keys", "sort_pairs",
           "sort_ex", "sort_keys_host", "sort_pairs_host", "sort_keys64", "sort_pairs64", "Workspace", "get_unique_id", "Comm", "sort_keys_dist",
           "exchange_plan", "dist_workspace_size", "dist_profile_end", "sort_keys_dist_emulated"]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgbs.so")
MAX_LEVELS = 4
UNIQUE_ID_BYTES = 128


class GbsError(RuntimeError):
    pass


class Config(C.Structure):
    _fields_ = [("L", C.c_uint32), ("s", C.c_uint32)]


class PlanT(C.Structure):
    _fields_ = [("levels", C.c_int), ("L", C.c_uint32 * MAX_LEVELS), ("s", C.c_uint32 * MAX_LEVELS),
                ("m", C.c_uint32 * MAX_LEVELS), ("cap", C.c_uint64 * MAX_LEVELS),
                ("bucket_bound", C.c_uint64 * MAX_LEVELS), ("ws_bytes", C.c_size_t),
                ("kernels_per_sort", C.c_int)]


class StepTimes(C.Structure):
    _fields_ = [("ms", C.c_float * 10), ("calls", C.c_int), ("levels", C.c_int),
                ("ms_level", (C.c_float * 10) * MAX_LEVELS)]


class DistTimes(C.Structure):
    _fields_ = [("ms", C.c_float * 6), ("exchange_bytes", C.c_double), ("calls", C.c_int), ("path", C.c_int)]


class LayoutT(C.Structure):
    _fields_ = [(f, C.c_size_t) for f in ("samples", "splitters", "a", "l", "relocated", "relocated_vals")]


_lib = None


def lib():
    """Load libgbs.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GbsError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        p, sz, u32 = C.c_void_p, C.c_size_t, C.c_uint32
        sigs = {
            "gbs_sort_keys_workspace_size": [sz, C.POINTER(sz)],
            "gbs_sort_pairs_workspace_size": [sz, C.POINTER(sz)],
            "gbs_sort_keys": [p, sz, p, sz, p],
            "gbs_sort_pairs": [p, p, sz, p, sz, p],
            "gbs_sort_keys_host": [p, sz, p, p, sz, p],
            "gbs_sort_pairs_host": [p, p, sz, p, p, p, sz, p],
            "gbs_sort_keys_typed": [p, sz, C.c_int, p, sz, p],
            "gbs_sort_pairs_typed": [p, p, sz, C.c_int, p, sz, p],
            "gbs_plan": [sz, C.c_int, C.POINTER(Config), C.POINTER(PlanT)],
            "gbs_workspace_size_ex": [sz, C.c_int, C.POINTER(Config), C.POINTER(sz)],
            "gbs_debug_layout": [sz, C.c_int, C.POINTER(Config), C.POINTER(LayoutT)],
            "gbs_sort_ex": [p, p, sz, C.POINTER(Config), C.c_int, p, sz, p],
            "gbs_get_unique_id": [p],
            "gbs_comm_init": [C.POINTER(p), p, C.c_int, C.c_int],
            "gbs_comm_destroy": [p],
            "gbs_sort_keys_dist_workspace_size": [sz, C.c_int, C.POINTER(sz), C.POINTER(sz)],
            "gbs_sort_keys_dist": [p, p, sz, p, sz, C.POINTER(sz), p, sz, p],
            "gbs_sort_keys_dist_emulated": [C.c_int, p, sz, p, sz, p, p, sz, p],
            "gbs_exchange_plan": [p, C.c_int, C.c_int, p, p, p, p, p],
            "gbs_profile_begin": [],
            "gbs_profile_end": [C.POINTER(StepTimes)],
            "gbs_comm_set_exchange": [p, C.c_int],
            "gbs_comm_init_host": [C.POINTER(p), C.c_int, C.c_int, p, p],
            "gbs_sort64_workspace_size": [sz, C.c_int, C.POINTER(sz)],
            "gbs_sort_keys64": [p, sz, C.c_int, p, sz, p],
            "gbs_sort_pairs64": [p, p, sz, C.c_int, p, sz, p],
            "gbs_dist_profile_end": [p],
            "gbs_sort_keys_dist_emulated_workspace_size": [sz, C.c_int, C.POINTER(sz)],
        }
        for name, args in sigs.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.gbs_status_string.argtypes = [C.c_int]
        L.gbs_status_string.restype = C.c_char_p
        L.gbs_last_error.argtypes = []
        L.gbs_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        L = lib()
        raise GbsError(f"{L.gbs_status_string(rc).decode()} ({rc}): {L.gbs_last_error().decode()}")


def _cfg(cfg):
    if cfg is None:
        return None
    L, s = cfg
    return C.byref(Config(L, s))


# ----------------------------------------------------------------- plans

@functools.lru_cache(maxsize=256)
def _plan_cached(n: int, pairs: bool, cfg):
    out = PlanT()
    _check(lib().gbs_plan(n, int(pairs), _cfg(cfg), C.byref(out)))
    k = out.levels
    return dict(levels=[(out.L[i], out.s[i]) for i in range(k)], m=list(out.m[:k]), cap=list(out.cap[:k]),
                bucket_bound=list(out.bucket_bound[:k]), ws_bytes=out.ws_bytes,
                kernels_per_sort=out.kernels_per_sort)


def plan(n: int, pairs: bool = False, cfg=None) -> dict:
    """The static plan for n items (depends on n, kind and cfg only)."""
    return dict(_plan_cached(int(n), bool(pairs), tuple(cfg) if cfg is not None else None))


def workspace_size(n: int, pairs: bool = False, cfg=None) -> int:
    return _plan_cached(int(n), bool(pairs), tuple(cfg) if cfg is not None else None)["ws_bytes"]


def debug_layout(n: int, pairs: bool = False, cfg=None) -> dict:
    out = LayoutT()
    _check(lib().gbs_debug_layout(n, int(pairs), _cfg(cfg), C.byref(out)))
    return {f: getattr(out, f) for f, _ in LayoutT._fields_}


def profile_begin():
    _check(lib().gbs_profile_begin())


def profile_end() -> dict:
    """{step: total ms} of the top level over the sorts enqueued since profile_begin(),
    'calls', and 'level' = a list of such dicts per level (0 = top, k = k-th nested Step 9)."""
    out = StepTimes()
    _check(lib().gbs_profile_end(C.byref(out)))
    d = {k: out.ms[k] for k in (2, 4, 5, 6, 7, 8, 9)}
    d["calls"] = out.calls
    d["level"] = [{k: out.ms_level[l][k] for k in (2, 4, 5, 6, 7, 8, 9)} for l in range(out.levels)]
    return d


# ----------------------------------------------------------------- tensors

def _torch():
    import torch
    return torch


def _dev_ptr(t, name, device=None):
    torch = _torch()
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise GbsError(f"{name} must be a CUDA tensor")
    if t.dtype not in (torch.int32, torch.uint32):
        raise GbsError(f"{name} must be int32/uint32 (bits read as unsigned)")
    if not t.is_contiguous():
        raise GbsError(f"{name} must be contiguous")
    if device is not None and t.device != device:
        raise GbsError(f"{name} is on {t.device}, expected {device}")
    return t.data_ptr()


class _On:
    """Run a library call on `device` (current device = the tensors' device, which is where
    libgbs launches) with `stream` (default: that device's current stream).  Owns the
    temporary workspace of the call: allocated with `stream` current, so the caching
    allocator hands its block to later work only in stream order after the sort; a
    caller's Workspace used on another stream is marked with record_stream."""

    def __init__(self, device, stream=None):
        torch = _torch()
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        if self.stream.device != device:
            raise GbsError(f"stream is on {self.stream.device}, the tensors on {device}")
        self.keep = []

    def __enter__(self):
        torch = _torch()
        self._dg = torch.cuda.device(self.device)
        self._dg.__enter__()
        self._sg = torch.cuda.stream(self.stream)
        self._sg.__enter__()
        return self

    def __exit__(self, *a):
        self._sg.__exit__(*a)
        self._dg.__exit__(*a)
        self.keep.clear()

    @property
    def s(self):
        return C.c_void_p(self.stream.cuda_stream)

    def ws(self, nbytes: int, ws=None):
        """(pointer, bytes) of a workspace of >= nbytes, alive until the call returns."""
        torch = _torch()
        if ws is None:
            buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        else:
            buf = ws.get(nbytes, self.device)
            buf.record_stream(self.stream)
        self.keep.append(buf)
        return C.c_void_p(buf.data_ptr()), buf.numel()


class Workspace:
    """A reusable device workspace (uint8 tensor) grown on demand."""

    def __init__(self, device=None):
        self.device = device
        self.buf = None

    def get(self, nbytes: int, device=None):
        torch = _torch()
        dev = device if device is not None else (self.device if self.device is not None else torch.cuda.current_device())
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != torch.device(dev):
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
        return self.buf


def sort_keys(keys, ws: Workspace | None = None, stream=None):
    """Sort a CUDA int32/uint32 tensor in place, ascending as unsigned 32-bit."""
    n = keys.numel()
    kp = _dev_ptr(keys, "keys")
    with _On(keys.device, stream) as on:
        wp, wb = on.ws(workspace_size(n), ws)
        _check(lib().gbs_sort_keys(C.c_void_p(kp), n, wp, wb, on.s))
    return keys


def sort_pairs(keys, vals, ws: Workspace | None = None, stream=None):
    """Sort (key, value) pairs by key in place, stable (std::stable_sort by key)."""
    n = keys.numel()
    if vals.numel() != n:
        raise GbsError("keys and vals must have the same length")
    kp, vp = _dev_ptr(keys, "keys"), _dev_ptr(vals, "vals", keys.device)
    with _On(keys.device, stream) as on:
        wp, wb = on.ws(workspace_size(n, pairs=True), ws)
        _check(lib().gbs_sort_pairs(C.c_void_p(kp), C.c_void_p(vp), n, wp, wb, on.s))
    return keys, vals


KEY_TYPES = {"uint32": 0, "int32": 1, "float32": 2}


def _key_type(t, key_type):
    torch = _torch()
    if key_type is None:
        key_type = {torch.uint32: "uint32", torch.int32: "int32", torch.float32: "float32"}.get(t.dtype)
        if key_type is None:
            raise GbsError("keys must be uint32, int32 or float32")
    if key_type not in KEY_TYPES:
        raise GbsError(f"key_type must be one of {sorted(KEY_TYPES)}")
    if not isinstance(t, torch.Tensor) or not t.is_cuda or not t.is_contiguous() or t.element_size() != 4:
        raise GbsError("keys must be a contiguous CUDA tensor of 4-byte elements")
    return KEY_TYPES[key_type]


def sort_keys_typed(keys, key_type=None, ws: Workspace | None = None, stream=None):
    """Sort a CUDA tensor in place by its value as uint32, int32 or float32 (default: the
    tensor's dtype; floats in IEEE-754 totalOrder, -0 before +0, NaNs at the ends by sign)."""
    kt = _key_type(keys, key_type)
    n = keys.numel()
    with _On(keys.device, stream) as on:
        wp, wb = on.ws(workspace_size(n), ws)
        _check(lib().gbs_sort_keys_typed(C.c_void_p(keys.data_ptr()), n, kt, wp, wb, on.s))
    return keys


def sort_pairs_typed(keys, vals, key_type=None, ws: Workspace | None = None, stream=None):
    """Stable (key, value) sort in place with uint32 / int32 / float32 keys (as sort_keys_typed)."""
    kt = _key_type(keys, key_type)
    n = keys.numel()
    if vals.numel() != n:
        raise GbsError("keys and vals must have the same length")
    vp = _dev_ptr(vals, "vals", keys.device)
    with _On(keys.device, stream) as on:
        wp, wb = on.ws(workspace_size(n, pairs=True), ws)
        _check(lib().gbs_sort_pairs_typed(C.c_void_p(keys.data_ptr()), C.c_void_p(vp), n, kt, wp, wb, on.s))
    return keys, vals


KEY64_TYPES = {"uint64": 0, "int64": 1, "float64": 2}


def _key64_type(t, key_type):
    torch = _torch()
    if key_type is None:
        key_type = {torch.uint64: "uint64", torch.int64: "int64", torch.float64: "float64"}.get(t.dtype)
        if key_type is None:
            raise GbsError("keys must be uint64, int64 or float64")
    if key_type not in KEY64_TYPES:
        raise GbsError(f"key_type must be one of {sorted(KEY64_TYPES)}")
    if not isinstance(t, torch.Tensor) or not t.is_cuda or not t.is_contiguous() or t.element_size() != 8:
        raise GbsError("keys must be a contiguous CUDA tensor of 8-byte elements")
    return KEY64_TYPES[key_type]


def sort64_workspace_size(n: int, pairs: bool = False) -> int:
    b = C.c_size_t()
    _check(lib().gbs_sort64_workspace_size(n, int(pairs), C.byref(b)))
    return b.value


def sort_keys64(keys, key_type=None, ws: Workspace | None = None, stream=None):
    """Sort a CUDA uint64 / int64 / float64 tensor in place by its numeric value (floats in
    IEEE-754 totalOrder).  Two stable 32-bit GBS passes + a gather (gbs_sort_keys64)."""
    kt = _key64_type(keys, key_type)
    n = keys.numel()
    with _On(keys.device, stream) as on:
        wp, wb = on.ws(sort64_workspace_size(n), ws)
        _check(lib().gbs_sort_keys64(C.c_void_p(keys.data_ptr()), n, kt, wp, wb, on.s))
    return keys


def sort_pairs64(keys, vals, key_type=None, ws: Workspace | None = None, stream=None):
    """Stable sort of (64-bit key, 32-bit value) pairs by key, in place."""
    kt = _key64_type(keys, key_type)
    n = keys.numel()
    if vals.numel() != n:
        raise GbsError("keys and vals must have the same length")
    vp = _dev_ptr(vals, "vals", keys.device)
    with _On(keys.device, stream) as on:
        wp, wb = on.ws(sort64_workspace_size(n, True), ws)
        _check(lib().gbs_sort_pairs64(C.c_void_p(keys.data_ptr()), C.c_void_p(vp), n, kt, wp, wb, on.s))
    return keys, vals


def sort_ex(keys, vals=None, cfg=None, stop_after_step: int = 0, ws=None, stream=None):
    """Debug/experiment entry: explicit level-1 (L, s) and early stop after a step.
    ``ws`` may be a raw uint8 CUDA tensor (to read intermediates at debug_layout offsets)."""
    torch = _torch()
    n = keys.numel()
    kp = _dev_ptr(keys, "keys")
    vp = _dev_ptr(vals, "vals", keys.device) if vals is not None else None
    need = workspace_size(n, vals is not None, cfg)
    with _On(keys.device, stream) as on:
        if isinstance(ws, torch.Tensor):
            if ws.numel() < need or ws.device != keys.device:
                raise GbsError("workspace tensor too small or on another device")
            wp, wb = C.c_void_p(ws.data_ptr()), ws.numel()
        else:
            wp, wb = on.ws(need, ws)
        _check(lib().gbs_sort_ex(C.c_void_p(kp), C.c_void_p(vp) if vp else None, n, _cfg(cfg),
                                 stop_after_step, wp, wb, on.s))
    return keys


def sort_keys_host(h_keys, d_buf, ws: Workspace | None = None, stream=None):
    """End-to-end: pinned host int32/uint32 tensor -> device -> sort -> host (in place)."""
    if h_keys.is_cuda or not h_keys.is_pinned():
        raise GbsError("h_keys must be a pinned host tensor")
    n = h_keys.numel()
    dp = _dev_ptr(d_buf, "d_buf")
    if d_buf.numel() < n:
        raise GbsError("d_buf too small")
    with _On(d_buf.device, stream) as on:
        wp, wb = on.ws(workspace_size(n), ws)
        _check(lib().gbs_sort_keys_host(C.c_void_p(h_keys.data_ptr()), n, C.c_void_p(dp), wp, wb, on.s))
    return h_keys


def sort_pairs_host(h_keys, h_vals, d_keys, d_vals, ws: Workspace | None = None, stream=None):
    """End-to-end stable pairs sort: pinned host keys/values -> device -> sort -> host (in place)."""
    for t, nm in ((h_keys, "h_keys"), (h_vals, "h_vals")):
        if t.is_cuda or not t.is_pinned():
            raise GbsError(f"{nm} must be a pinned host tensor")
    n = h_keys.numel()
    if h_vals.numel() != n or d_keys.numel() < n or d_vals.numel() < n:
        raise GbsError("size mismatch")
    dk, dv = _dev_ptr(d_keys, "d_keys"), _dev_ptr(d_vals, "d_vals", d_keys.device)
    with _On(d_keys.device, stream) as on:
        wp, wb = on.ws(workspace_size(n, pairs=True), ws)
        _check(lib().gbs_sort_pairs_host(C.c_void_p(h_keys.data_ptr()), C.c_void_p(h_vals.data_ptr()), n,
                                         C.c_void_p(dk), C.c_void_p(dv), wp, wb, on.s))
    return h_keys, h_vals


# ----------------------------------------------------------------- multi GPU

def get_unique_id() -> bytes:
    buf = (C.c_uint8 * UNIQUE_ID_BYTES)()
    _check(lib().gbs_get_unique_id(buf))
    return bytes(buf)


def dist_workspace_size(n_local: int, nranks: int):
    w, cap = C.c_size_t(), C.c_size_t()
    _check(lib().gbs_sort_keys_dist_workspace_size(n_local, nranks, C.byref(w), C.byref(cap)))
    return w.value, cap.value


def exchange_plan(cuts, rank: int):
    """Host-only exchange plan (E7-E8) from the p x p cut matrix (numpy uint64)."""
    import numpy as np
    cuts = np.ascontiguousarray(cuts, dtype=np.uint64)
    p = cuts.shape[0]
    so, sc, ro, rc = (np.zeros(p, np.uint64) for _ in range(4))
    n_out = np.zeros(1, np.uint64)
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)
    _check(lib().gbs_exchange_plan(ptr(cuts), p, rank, ptr(so), ptr(sc), ptr(ro), ptr(rc), ptr(n_out)))
    return dict(send_off=so, send_cnt=sc, recv_off=ro, recv_cnt=rc, n_out=int(n_out[0]))


HOST_ALLGATHER = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class Comm:
    """libgbs communicator (NCCL + peer-mapped windows), bootstrapped over a
    torch.distributed group: rank 0 creates the NCCL unique id, the group broadcasts it.
    bootstrap="host": no NCCL -- the window handles are exchanged with the group's own
    all_gather (any backend, e.g. gloo), so several processes may share one GPU."""

    def __init__(self, group=None, exchange: str = "p2p", bootstrap: str = "nccl"):
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        if bootstrap == "host":
            def allgather(send, recv, nbytes, _ctx):
                try:
                    mine = C.string_at(send, nbytes)
                    out = [None] * self.nranks
                    dist.all_gather_object(out, mine, group=group)
                    C.memmove(recv, b"".join(out), nbytes * self.nranks)
                    return 0
                except Exception:  # noqa: BLE001
                    return 1
            self._cb = HOST_ALLGATHER(allgather)             # kept alive with the communicator
            h = C.c_void_p()
            _check(lib().gbs_comm_init_host(C.byref(h), self.nranks, self.rank, C.cast(self._cb, C.c_void_p), None))
            self.handle = h
            return
        obj = [get_unique_id() if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        idbuf = (C.c_uint8 * UNIQUE_ID_BYTES).from_buffer_copy(obj[0])
        h = C.c_void_p()
        _check(lib().gbs_comm_init(C.byref(h), idbuf, self.nranks, self.rank))
        self.handle = h
        if exchange != "p2p":
            self.set_exchange(exchange)

    def set_exchange(self, exchange: str):
        """'p2p' (peer memory, default) or 'nccl'; collective."""
        _check(lib().gbs_comm_set_exchange(self.handle, {"p2p": 0, "nccl": 1}[exchange]))

    def close(self):
        if self.handle:
            _check(lib().gbs_comm_destroy(self.handle))
            self.handle = None


def sort_keys_dist(keys, comm: Comm, out=None, ws: Workspace | None = None, stream=None):
    """Every rank passes an equal-length shard (read only); returns the rank's part of the
    global order (a view of ``out``, allocated if missing or too small)."""
    torch = _torch()
    n = keys.numel()
    kp = _dev_ptr(keys, "keys")
    need, cap = dist_workspace_size(n, comm.nranks)
    if out is None or out.numel() < cap:
        out = torch.empty(cap, dtype=keys.dtype, device=keys.device)
    n_out = C.c_size_t()
    with _On(keys.device, stream) as on:
        wp, wb = on.ws(need, ws)
        _check(lib().gbs_sort_keys_dist(comm.handle, C.c_void_p(kp), n, C.c_void_p(out.data_ptr()), out.numel(),
                                        C.byref(n_out), wp, wb, on.s))
    return out[:n_out.value]


def dist_profile_end() -> dict:
    """Phase times (ms, summed over the calls) of the multi-GPU sorts since profile_begin()."""
    out = DistTimes()
    _check(lib().gbs_dist_profile_end(C.byref(out)))
    names = ["local_sort_ms", "samples_cuts_ms", "exchange_ms", "merge_ms", "_", "total_ms"]
    c = max(out.calls, 1)
    d = {nm: out.ms[i] / c for i, nm in enumerate(names) if nm != "_"}
    d.update(calls=out.calls, exchange_bytes=out.exchange_bytes / c,
             path={0: "one rank", 1: "peer memory (NVLink stores)", 2: "nccl",
                   3: "emulated (all ranks on one GPU, phases summed over ranks)"}.get(out.path))
    return d


def sort_keys_dist_emulated(shards, p: int, stream=None):
    """Testing aid: the p-rank multi-GPU path on one GPU (the same kernels, the p windows
    as regions of one workspace).  ``shards``: p*n_local keys, rank r's shard at
    [r n_local, (r+1) n_local) (read only).  Returns the list of the p ranks' parts."""
    torch = _torch()
    assert shards.numel() % p == 0
    n = shards.numel() // p
    kp = _dev_ptr(shards, "shards")
    _, cap = dist_workspace_size(n, p)
    tot = C.c_size_t()
    _check(lib().gbs_sort_keys_dist_emulated_workspace_size(n, p, C.byref(tot)))
    out = torch.empty(p * cap, dtype=shards.dtype, device=shards.device)
    n_out = (C.c_size_t * p)()
    with _On(shards.device, stream) as on:
        ws = torch.empty(tot.value + 256, dtype=torch.uint8, device=shards.device)
        wp = (ws.data_ptr() + 255) // 256 * 256
        _check(lib().gbs_sort_keys_dist_emulated(p, C.c_void_p(kp), n, C.c_void_p(out.data_ptr()), cap, n_out,
                                                 C.c_void_p(wp), tot.value, on.s))
    return [out[r * cap:r * cap + n_out[r]] for r in range(p)]
