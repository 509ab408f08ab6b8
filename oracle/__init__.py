"""CPU oracle for GPU Bucket Sort (arXiv 1002.4464, Algorithm 1).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product (``paper_1002_4464_b200``) never imports it; the two share
no code.  The arithmetic lives in ``gbs_oracle.c`` (plain single-threaded C);
this module is argument marshalling over ctypes plus the plan arithmetic the
tests use to state plans independently of the CUDA library.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gbs_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, single-threaded, no OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC",
                               "-o", _LIB, _SRC])
    return _LIB


class Trace(C.Structure):
    _fields_ = [("sorted_keys", C.c_void_p), ("samples", C.c_void_p),
                ("sorted_samples", C.c_void_p), ("splitters", C.c_void_p),
                ("a", C.c_void_p), ("l", C.c_void_p), ("relocated", C.c_void_p),
                ("bucket_total", C.c_void_p)]


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_LIB)
        u64, p = C.c_uint64, C.c_void_p
        lib.oracle_gbs_sort.argtypes = [p, p, u64, p, p, C.c_int, p]
        lib.oracle_gbs_sort_batch.argtypes = [p, u64, u64, p, p, C.c_int]
        lib.oracle_psrs.argtypes = [p, u64, C.c_int, C.c_uint32, p, p, p]
        lib.oracle_bucket_bound.argtypes = [u64, C.c_uint32, C.c_uint32, p, p, p, p, p]
        lib.oracle_bucket_bound.restype = None
        lib.oracle_local_samples.argtypes = [p, u64, C.c_uint32, C.c_uint32, p]
        lib.oracle_local_samples.restype = None
        lib.oracle_global_samples.argtypes = [p, u64, C.c_uint32, p]
        lib.oracle_global_samples.restype = None
        lib.oracle_sample_index.argtypes = [p, u64, C.c_uint32, C.c_uint32, p, C.c_uint32, p, p]
        lib.oracle_sample_index.restype = None
        lib.oracle_offsets.argtypes = [p, u64, C.c_uint32, p]
        lib.oracle_offsets.restype = None
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _plan_arrays(plan):
    Ls = np.array([lv[0] for lv in plan] or [0], dtype=np.uint32)
    ss = np.array([lv[1] for lv in plan] or [0], dtype=np.uint32)
    return Ls, ss


class OracleError(RuntimeError):
    pass


def _check(rc):
    if rc != 0:
        raise OracleError({-1: "allocation failed", -2: "invalid plan or size",
                           -3: "bucket bound violated"}.get(rc, f"rc={rc}"))


def bucket_bound(cap: int, L: int, s: int):
    """(m, n', hi, lo, last) of one level -- see gbs_oracle.c:oracle_bucket_bound."""
    out = [C.c_uint64() for _ in range(5)]
    _load().oracle_bucket_bound(cap, L, s, *[C.byref(o) for o in out])
    return tuple(int(o.value) for o in out)


def gbs_sort(keys, vals=None, plan=(), trace: bool = False):
    """Oracle GBS of ``keys`` (uint32) [and ``vals``] with plan [(L, s), ...] (level 1
    first; empty plan = one local sort).  Returns (keys, vals, trace_dict|None)."""
    lib = _load()
    k = np.ascontiguousarray(keys, dtype=np.uint32).copy()
    v = None if vals is None else np.ascontiguousarray(vals, dtype=np.uint32).copy()
    n = k.size
    Ls, ss = _plan_arrays(plan)
    tr_d = None
    tr_p = None
    if trace and plan and n > 1:
        L, s = plan[0]
        m = (n + L - 1) // L
        tr_d = dict(sorted_keys=np.zeros(n, np.uint32), samples=np.zeros(m * s, np.uint64),
                    sorted_samples=np.zeros(m * s, np.uint64), splitters=np.zeros(s, np.uint64),
                    a=np.zeros(m * s, np.uint32), l=np.zeros(m * s, np.uint32),
                    relocated=np.zeros(n, np.uint32), bucket_total=np.zeros(s, np.uint64))
        tr = Trace(*[_ptr(tr_d[f]) for f, _ in Trace._fields_])
        tr_p = C.byref(tr)
    _check(lib.oracle_gbs_sort(_ptr(k), _ptr(v), n, _ptr(Ls), _ptr(ss), len(plan), tr_p))
    if tr_d is not None:
        m = tr_d["a"].size // plan[0][1]
        tr_d["a"] = tr_d["a"].reshape(m, plan[0][1])
        tr_d["l"] = tr_d["l"].reshape(m, plan[0][1])
    return k, v, tr_d


def gbs_sort_batch(rows, plan):
    """Sort every row of a 2-D uint32 array independently (brute-force helper)."""
    lib = _load()
    x = np.ascontiguousarray(rows, dtype=np.uint32).copy()
    Ls, ss = _plan_arrays(plan)
    _check(lib.oracle_gbs_sort_batch(_ptr(x), x.shape[0], x.shape[1], _ptr(Ls), _ptr(ss), len(plan)))
    return x


def psrs(keys, p: int, s_r: int):
    """Multi-GPU outer level simulated on one host.  ``keys`` is the
    concatenation of p equal shards.  Returns (out, counts[p], cuts[p, p])."""
    lib = _load()
    k = np.ascontiguousarray(keys, dtype=np.uint32)
    n_local = k.size // p
    out = np.zeros(k.size, np.uint32)
    counts = np.zeros(p, np.uint64)
    cuts = np.zeros(p * p, np.uint64)
    _check(lib.oracle_psrs(_ptr(k), n_local, p, s_r, _ptr(out), _ptr(counts), _ptr(cuts)))
    return out, counts, cuts.reshape(p, p)


# --- per-step functions, exposed so tests can pin each against SPEC examples ---

def local_samples(sorted_keys, tag0: int, L: int, s: int):
    k = np.ascontiguousarray(sorted_keys, dtype=np.uint32)
    out = np.zeros(s, np.uint64)
    _load().oracle_local_samples(_ptr(k), tag0, L, s, _ptr(out))
    return out


def global_samples(sorted_samples, m: int, s: int):
    x = np.ascontiguousarray(sorted_samples, dtype=np.uint64)
    g = np.zeros(s, np.uint64)
    _load().oracle_global_samples(_ptr(x), m, s, _ptr(g))
    return g


def sample_index(sorted_keys, tag0: int, valid: int, splitters):
    k = np.ascontiguousarray(sorted_keys, dtype=np.uint32)
    g = np.ascontiguousarray(splitters, dtype=np.uint64)
    a = np.zeros(g.size, np.uint32)
    tot = np.zeros(g.size, np.uint64)
    _load().oracle_sample_index(_ptr(k), tag0, k.size, valid, _ptr(g), g.size, _ptr(a), _ptr(tot))
    return a, tot


def offsets(a):
    a = np.ascontiguousarray(a, dtype=np.uint32)
    m, s = a.shape
    l = np.zeros_like(a)
    _load().oracle_offsets(_ptr(a), m, s, _ptr(l))
    return l


def composite(key: int, tag: int) -> int:
    return (int(key) << 32) | int(tag)


# --- 64-bit keys: the plain definition of the result ---------------
# The paper's problem statement sorts "an array A with n data items" and never
# fixes the item type (R1).  For 64-bit keys the oracle is the definition the
# method must reach exactly: a stable sort by the key's numeric order.
# u64 / i64: the integer order.  f64: IEEE-754 totalOrder (IEEE 754-2008 section 5.10),
# written out: -NaN (larger payload first) < -inf < negative finite < -0 < +0 < positive
# finite < +inf < +NaN (larger payload last).

def _f64_total_order_key(bits: int):
    sign = bits >> 63
    exp = (bits >> 52) & 0x7FF
    frac = bits & ((1 << 52) - 1)
    if exp == 0x7FF and frac:                       # NaN: ordered by sign, then payload
        return (3, frac) if not sign else (-3, -frac)
    value = np.array([bits], dtype=np.uint64).view(np.float64)[0]
    zero_rank = (0 if sign else 1) if value == 0 else 0
    return (0, float(value), zero_rank)


def sort64(keys, vals=None, key_type: str = "uint64"):
    """Stable sort of 64-bit keys (uint64 / int64 / float64 as raw 8-byte items) [and u32
    values] by numeric key; pure Python ordering (small inputs).  Returns (keys, vals)."""
    k = np.ascontiguousarray(keys)
    bits = k.view(np.uint64)
    if key_type == "uint64":
        keyf = [int(b) for b in bits]
    elif key_type == "int64":
        keyf = [int(b) for b in bits.view(np.int64)]
    elif key_type == "float64":
        keyf = [_f64_total_order_key(int(b)) for b in bits]
    else:
        raise ValueError(key_type)
    order = sorted(range(k.size), key=lambda i: keyf[i])        # Python's sort is stable
    order = np.array(order, dtype=np.int64)
    return k[order], (None if vals is None else np.ascontiguousarray(vals)[order])
