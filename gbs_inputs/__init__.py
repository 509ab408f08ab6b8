"""Seeded synthetic inputs for GPU Bucket Sort tests and benchmarks.

This module holds NONE of the method's arithmetic: it only generates keys.  It
serves both the oracle (``oracle/``) and the CUDA path (``paper_1002_4464_b200``)
so the two sort identical bytes.

Generator: counter-based SplitMix64,
``u(c) = hi32(mix(seed + (c+1) * 0x9E3779B97F4A7C15))`` -- the c-th output of a
standard SplitMix64(seed) -- so any rank or host can generate any slice.

The seven distributions are the Helman-Bader-JaJa benchmark family the north
star names (uniform, gaussian, bucket-sorted, staggered, sorted, zero,
det-duplicates); the paper itself measured only uniform.  With
P_v = 256 virtual blocks of b = n // P_v items, element e has q = e // b (capped
at P_v - 1) and o = e - q b.

Two implementations: ``numpy`` (canonical, exact uint64 wrap-around) and
``torch`` (same formulas on int64 tensors, usable on a CUDA device for large n);
tests check they agree bit for bit.
"""
from __future__ import annotations

import numpy as np

DISTRIBUTIONS = ("uniform", "gaussian", "bucket_sorted", "staggered", "sorted", "zero",
                 "det_duplicates")
GAMMA = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
PV = 256


# ----------------------------------------------------------------- numpy (canonical)

def _mix_np(z):
    z = z.copy()
    z ^= z >> np.uint64(30)
    z *= np.uint64(M1)
    z ^= z >> np.uint64(27)
    z *= np.uint64(M2)
    z ^= z >> np.uint64(31)
    return z


def _u_np(seed: int, c):
    """u(c) for an array of counters c (uint64)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (c.astype(np.uint64) + np.uint64(1)) * np.uint64(GAMMA)
        return (_mix_np(z) >> np.uint64(32)).astype(np.uint32)


def _blocks(n: int, e):
    b = max(1, n // PV)
    q = np.minimum(e // b, PV - 1)
    o = e - q * b
    return b, q, o


def _floor_log2(x):
    """floor(log2(x)) for integer x >= 1 (elementwise)."""
    x = np.asarray(x, dtype=np.int64)
    out = np.zeros(x.shape, np.int64)
    y = x.copy()
    for sh in (32, 16, 8, 4, 2, 1):
        m = y >= (1 << sh)
        out[m] += sh
        y[m] >>= sh
    return out


def generate(dist: str, n: int, seed: int = 0, start: int = 0, count: int | None = None):
    """Keys [start, start+count) of distribution ``dist`` over a global array of n."""
    if count is None:
        count = n - start
    e = np.arange(start, start + count, dtype=np.int64)
    if dist == "uniform":
        return _u_np(seed, e)
    if dist == "gaussian":
        acc = np.zeros(count, np.uint64)
        for t in range(4):
            acc += _u_np(seed, 4 * e + t).astype(np.uint64)
        return (acc >> np.uint64(2)).astype(np.uint32)
    if dist == "zero":
        return np.zeros(count, np.uint32)
    if dist == "sorted":
        if start != 0 or count != n:
            raise ValueError("sorted is defined on the whole array only")
        return np.sort(_u_np(seed, e))
    b, q, o = _blocks(n, e)
    low = (_u_np(seed, e) >> np.uint32(8)).astype(np.int64)
    if dist == "bucket_sorted":
        bs = max(1, b // PV)
        g = np.minimum(o // bs, PV - 1)
        return (g * (1 << 24) + low).astype(np.uint32)
    if dist == "staggered":
        base = np.where(q < PV // 2, 2 * q + 1, 2 * q - PV) * (1 << 24)
        return (base + low).astype(np.uint32)
    if dist == "det_duplicates":
        lg = int(_floor_log2(max(n, 1)))
        t = 1 + _floor_log2(PV // np.maximum(PV - q, 1))
        ob = np.maximum(b - o, 1)
        u = 1 + _floor_log2(np.maximum(b // ob, 1))
        v = np.where(q < PV - 1, lg - t + 1, lg - 8 - u + 1)
        return np.maximum(v, 0).astype(np.uint32)
    raise ValueError(f"unknown distribution {dist!r}")


def pair_values(n: int, start: int = 0, count: int | None = None):
    """Pair values v_e = e (makes stability and permutation checks trivial)."""
    if count is None:
        count = n - start
    return np.arange(start, start + count, dtype=np.int64).astype(np.uint32)


# ----------------------------------------------------------------- torch twin

def _mix_t(z):
    import torch
    def srl(x, k):  # logical shift right of a 64-bit pattern held in int64
        return (x >> k) & ((1 << (64 - k)) - 1)
    z = z ^ srl(z, 30)
    z = z * torch.tensor(M1 - (1 << 64), dtype=torch.int64, device=z.device)
    z = z ^ srl(z, 27)
    z = z * torch.tensor(M2 - (1 << 64), dtype=torch.int64, device=z.device)
    z = z ^ srl(z, 31)
    return z


def _u_t(seed: int, c):
    import torch
    g = torch.tensor(GAMMA - (1 << 64), dtype=torch.int64, device=c.device)
    sd = torch.tensor(seed if seed < (1 << 63) else seed - (1 << 64), dtype=torch.int64, device=c.device)
    z = sd + (c + 1) * g
    return (_mix_t(z) >> 32) & 0xFFFFFFFF   # int64 in [0, 2^32)


def _floor_log2_t(x):
    import torch
    out = torch.zeros_like(x)
    y = x.clone()
    for sh in (32, 16, 8, 4, 2, 1):
        m = y >= (1 << sh)
        out = out + m.to(torch.int64) * sh
        y = torch.where(m, y >> sh, y)
    return out


def generate_torch(dist: str, n: int, seed: int = 0, device="cpu", start: int = 0,
                   count: int | None = None, chunk: int = 1 << 26):
    """Same keys as :func:`generate`, as an int32 torch tensor holding the uint32 bits
    (torch has no general uint32 arithmetic).  Generated in chunks to bound memory."""
    import torch
    if count is None:
        count = n - start
    out = torch.empty(count, dtype=torch.int32, device=device)
    for c0 in range(0, count, chunk):
        c1 = min(count, c0 + chunk)
        e = torch.arange(start + c0, start + c1, dtype=torch.int64, device=device)
        if dist in ("uniform", "sorted"):
            v = _u_t(seed, e)
        elif dist == "gaussian":
            v = sum(_u_t(seed, 4 * e + t) for t in range(4)) >> 2
        elif dist == "zero":
            v = torch.zeros_like(e)
        else:
            b = max(1, n // PV)
            q = torch.clamp(e // b, max=PV - 1)
            o = e - q * b
            low = _u_t(seed, e) >> 8
            if dist == "bucket_sorted":
                bs = max(1, b // PV)
                v = torch.clamp(o // bs, max=PV - 1) * (1 << 24) + low
            elif dist == "staggered":
                v = torch.where(q < PV // 2, 2 * q + 1, 2 * q - PV) * (1 << 24) + low
            elif dist == "det_duplicates":
                lg = int(_floor_log2(max(n, 1)))
                t = 1 + _floor_log2_t(PV // torch.clamp(PV - q, min=1))
                ob = torch.clamp(b - o, min=1)
                u = 1 + _floor_log2_t(torch.clamp(b // ob, min=1))
                v = torch.clamp(torch.where(q < PV - 1, lg - t + 1, lg - 8 - u + 1), min=0)
            else:
                raise ValueError(f"unknown distribution {dist!r}")
        out[c0:c1] = (v - ((v >> 31) << 32)).to(torch.int32)   # uint32 bits -> int32
    if dist == "sorted":
        if start != 0 or count != n:
            raise ValueError("sorted is defined on the whole array only")
        u = out.to(torch.int64) & 0xFFFFFFFF
        u, _ = torch.sort(u)
        out = (u - ((u >> 31) << 32)).to(torch.int32)
    return out
