"""CPU (-m "not gpu"): DESIGN.md R28, the packed pairs tile, restated in numpy and checked
against the plain definition of the stable sort (np.argsort(kind="stable"), R7).

The GPU tile sorts P = (prefix << POSB) | position with prefix = (key - min) >> shift (the
top 32 - POSB bits of the tile's key range), then runs odd-even transposition rounds in
which neighbours of equal prefix swap iff the later key is strictly smaller.  The claims
checked here, on tiles built to stress them:
  1. the result is the stable order (key, position) for every input;
  2. a group of g items is sorted after g rounds, so a fixed round count equal to the
     largest prefix group suffices (the fixed-round path of the fix-up);
  3. shift = 0 (key range below 2^(32 - POSB)) makes the packed order itself the stable
     order (MODE_EXACT: no fix-up)."""
import numpy as np
import pytest

POSB = 14


def packed_order(keys):
    """Positions in the order of the packed sort (P distinct: ties cannot occur)."""
    keys = keys.astype(np.uint64)
    lo, hi = int(keys.min()), int(keys.max())
    bits = (hi - lo).bit_length()
    shift = max(0, bits - (32 - POSB))
    pre = (keys - lo) >> np.uint64(shift)
    P = (pre << np.uint64(POSB)) | np.arange(keys.size, dtype=np.uint64)
    order = np.argsort(P, kind="stable")
    return order, pre[order], shift


def transpose_rounds(order, pre, keys, rounds=None):
    """Odd-even transposition restricted to equal-prefix neighbours; stops after `rounds`
    rounds, or (None) after the first round pair without a swap.  Returns (order, rounds run)."""
    o = order.copy()
    k = keys[o].astype(np.int64)
    n, r = o.size, 0
    while True:
        swapped = False
        for parity in (0, 1):
            if rounds is not None and r >= rounds:
                return o, r
            i = np.arange(parity, n - 1, 2)
            sw = (pre[i] == pre[i + 1]) & (k[i + 1] < k[i])
            a, b = i[sw], i[sw] + 1
            o[a], o[b] = o[b].copy(), o[a].copy()
            k[a], k[b] = k[b].copy(), k[a].copy()
            swapped |= bool(sw.any())
            r += 1
        if rounds is None and not swapped:
            return o, r


def largest_group(pre):
    if pre.size == 0:
        return 0
    edges = np.flatnonzero(np.diff(pre.astype(np.int64)) != 0)
    bounds = np.concatenate(([-1], edges, [pre.size - 1]))
    return int(np.diff(bounds).max())


def tiles(seed):
    r = np.random.default_rng(seed)
    n = 1 << POSB
    yield r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)                # uniform, full range
    yield (r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32) % 1000)        # small range: exact
    g = r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    for s0 in range(0, n - 40, 997):                                                   # prefix clusters
        g[s0:s0 + 40] = (r.integers(0, (1 << 32) - (1 << 14)) + r.integers(0, 1 << 14, 40) // 3 * 3)
    yield g
    z = np.zeros(n, dtype=np.uint32)
    z[::5000] = 0xFFFFFFFF                                                             # range 2^32, equal keys
    yield z
    yield np.sort(r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32))[::-1].copy()  # reversed


@pytest.mark.parametrize("seed", [0, 1])
def test_packed_then_transposition_is_the_stable_sort(seed):
    for keys in tiles(seed):
        order, pre, shift = packed_order(keys)
        fixed, _ = transpose_rounds(order, pre, keys)
        assert np.array_equal(fixed, np.argsort(keys, kind="stable"))


@pytest.mark.parametrize("seed", [2, 3])
def test_largest_group_rounds_suffice(seed):
    for keys in tiles(seed):
        order, pre, shift = packed_order(keys)
        g = largest_group(pre)
        fixed, r = transpose_rounds(order, pre, keys, rounds=g)
        assert r <= g
        assert np.array_equal(fixed, np.argsort(keys, kind="stable"))


def test_small_range_needs_no_fixup():
    r = np.random.default_rng(4)
    keys = (r.integers(0, 1 << 18, 1 << POSB, dtype=np.uint64)).astype(np.uint32) + np.uint32(123456789)
    order, pre, shift = packed_order(keys)
    assert shift == 0
    assert np.array_equal(order, np.argsort(keys, kind="stable"))
