"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Every test names what fixes the expected value: a naive sort (brute force), a
closed form, an invariant with its derivation, the paper's worked parameters, or
a SPEC per-operation example.  A plausible slip in the oracle -- a dropped
sentinel, an off-by-one sample index, a transposed scan order, an inclusive/
exclusive bucket rule swap, an unstable tie -- fails at least one of them.
"""
import itertools

import numpy as np
import pytest

import gbs_inputs as gi
import oracle
from plans import TILE_KEYS, TILE_PAIRS, hi_bound, plan

ALPHA = np.array([0, 1, 2, 0xFFFFFFFF], dtype=np.uint32)
SMALL_PLANS = [(4, [(2, 2)]), (4, [(4, 2)]), (4, [(4, 4)]), (6, [(2, 2)]), (8, [(2, 2)]),
               (8, [(4, 2)]), (8, [(4, 4)]), (8, [(8, 2)]), (8, [(8, 4)]), (8, [(2, 1)]),
               (5, [(2, 2)]), (7, [(4, 2)]), (8, [(2, 2), (2, 2)]), (7, [(2, 2), (2, 1)])]


def _all_words(n):
    idx = np.array(list(itertools.product(range(4), repeat=n)), dtype=np.int64)
    return ALPHA[idx]


# ------------------------------------------------------------ brute force

@pytest.mark.parametrize("n,pl", SMALL_PLANS)
def test_bruteforce_all_small_inputs(n, pl):
    """Every input of length n over {0,1,2,0xFFFFFFFF} (sentinel-colliding key
    included): oracle == naive sort."""
    rows = _all_words(n)
    got = oracle.gbs_sort_batch(rows, pl)
    assert np.array_equal(got, np.sort(rows, axis=1))


def test_bruteforce_all_permutations():
    rows = np.array(list(itertools.permutations(range(8))), dtype=np.uint32) * 7 + 3
    for pl in ([(4, 2)], [(2, 2)], [(8, 4)], [(2, 2), (2, 2)]):
        assert np.array_equal(oracle.gbs_sort_batch(rows, pl), np.sort(rows, axis=1))


def test_random_medium_against_numpy():
    rng = np.random.default_rng(1)
    for n, pl in [(1000, [(64, 8)]), (4097, [(256, 16)]), (3000, [(64, 8), (64, 4)]),
                  (5000, [(128, 4)]), (20000, [(1024, 64), (256, 16)])]:
        for hi_key in (4, 1000, 1 << 32):
            k = rng.integers(0, hi_key, n, dtype=np.uint64).astype(np.uint32)
            out, _, _ = oracle.gbs_sort(k, plan=pl)
            assert np.array_equal(out, np.sort(k)), (n, pl, hi_key)


@pytest.mark.parametrize("dist", gi.DISTRIBUTIONS)
@pytest.mark.parametrize("n", [0, 1, 2, 1023, 2048, 2049, 65536])
def test_distributions_paper_and_default_plan(dist, n):
    """SPEC acceptance S:439 sizes; paper plan (L=2K, s=64)
    and the default plan of DESIGN.md section 5."""
    k = gi.generate(dist, n, seed=n % 5)
    for pl in (plan(n, cfg=(2048, 64)) if n > 1 else [], plan(n), [(256, 32)] if n > 1 else []):
        out, _, _ = oracle.gbs_sort(k, plan=pl)
        assert np.array_equal(out, np.sort(k)), (dist, n, pl)


# ------------------------------------------------------------ stability (pairs)

def test_pairs_stable_with_90pct_duplicates():
    """stable by key; values = index so the expected permutation is the
    stable argsort (a library sort with a documented stable mode)."""
    rng = np.random.default_rng(7)
    for n, pl in [(10000, [(256, 16)]), (10000, [(512, 8), (256, 8)]), (3001, [(64, 2)])]:
        k = np.where(rng.random(n) < 0.9, 5, rng.integers(0, 1 << 32, n)).astype(np.uint32)
        v = np.arange(n, dtype=np.uint32)
        ko, vo, _ = oracle.gbs_sort(k, v, plan=pl)
        perm = np.argsort(k, kind="stable")
        assert np.array_equal(ko, k[perm]) and np.array_equal(vo, v[perm])


# ------------------------------------------------------------ invariants

def _trace(k, pl):
    return oracle.gbs_sort(k, plan=pl, trace=True)[2]


def test_bucket_bound_tight_and_attained():
    """|B_j| (sentinels included) within the tight bound for j < s-1 and <= n'/s for
    the last bucket; the upper bound is reached (it is tight, not just valid)."""
    rng = np.random.default_rng(3)
    n, L, s = 16, 4, 2
    m, npr, hi, lo, last = oracle.bucket_bound(n, L, s)
    assert (m, npr, hi, lo, last) == (4, 16, 11, 5, 8)
    best = 0
    for _ in range(4000):
        k = rng.integers(0, 4, n).astype(np.uint32)
        tot = _trace(k, [(L, s)])["bucket_total"]
        assert tot.sum() == npr
        assert all(lo <= t <= hi for t in tot[:-1]) and tot[-1] <= last
        best = max(best, int(tot.max()))
    assert best == hi


@pytest.mark.parametrize("n,L,s", [(1 << 14, 1024, 64), (1 << 16, 2048, 64), (12288, 4096, 256)])
def test_bucket_bound_random(n, L, s):
    rng = np.random.default_rng(n)
    m, npr, hi, lo, last = oracle.bucket_bound(n, L, s)
    for keyspace in (2, 50, 1 << 32):
        k = rng.integers(0, keyspace, n, dtype=np.uint64).astype(np.uint32)
        tot = _trace(k, [(L, s)])["bucket_total"]
        assert all(lo <= t <= hi for t in tot[:-1]) and tot[-1] <= last
        assert tot.max() <= 2 * n / s            # the paper's form


@pytest.mark.parametrize("dist", ["zero", "sorted"])
def test_closed_form_equal_buckets(dist):
    """All-equal and sorted inputs: tag order == index order and splitter tags are
    (k+1) m d - 1, so every bucket holds exactly n/s items."""
    n, L, s = 1 << 15, 1024, 32
    k = gi.generate(dist, n, seed=1)
    tr = _trace(k, [(L, s)])
    assert np.all(tr["bucket_total"] == n // s)
    assert np.all(tr["a"].sum(axis=0) == n // s)


def test_conservation_and_offsets():
    """Sum a = n; row i sums to its real items; l = column-major exclusive scan
    (P:231-233): l_00 = 0 and l_{m-1,s-1} + a_{m-1,s-1} = n."""
    rng = np.random.default_rng(11)
    n, L, s = 10000, 512, 16          # ragged tail: 10000 = 19*512 + 272
    k = rng.integers(0, 1000, n).astype(np.uint32)
    tr = _trace(k, [(L, s)])
    a, l = tr["a"].astype(np.int64), tr["l"].astype(np.int64)
    m = a.shape[0]
    assert a.sum() == n
    valid = np.minimum(np.maximum(n - np.arange(m) * L, 0), L)
    assert np.array_equal(a.sum(axis=1), valid)
    colmajor = a.T.reshape(-1)
    excl = np.concatenate([[0], np.cumsum(colmajor)[:-1]])
    assert np.array_equal(l.T.reshape(-1), excl)
    assert l[-1, -1] + a[-1, -1] == n


def test_stage_intermediates_by_definition():
    """Re-derive each intermediate from its definition with plain numpy:
    Step 2 sorted sublists, Step 3 indices (k+1)d-1 with tags iL+r, Step 4 sort,
    Step 5 indices (k+1)m-1, Step 6 by LINEAR count over (key, tag) (pins the
    bisection), Step 8 relocation from a and l, R8 sentinels (key 2^32-1, tag>=n)."""
    rng = np.random.default_rng(5)
    n, L, s = 3000, 256, 8
    k = rng.integers(0, 300, n).astype(np.uint32)
    tr = _trace(k, [(L, s)])
    m, d = -(-n // L), L // s
    pad = np.concatenate([k, np.full(m * L - n, 0xFFFFFFFF, np.uint32)])
    A = np.concatenate([np.sort(pad[i * L:(i + 1) * L]) for i in range(m)])
    assert np.array_equal(tr["sorted_keys"], A[:n])
    tags = np.arange(m * L, dtype=np.uint64)
    comp = (A.astype(np.uint64) << np.uint64(32)) | tags
    S = np.concatenate([comp[i * L + (np.arange(s) + 1) * d - 1] for i in range(m)])
    assert np.array_equal(tr["samples"], S)
    assert np.array_equal(tr["sorted_samples"], np.sort(S))
    g = np.sort(S)[(np.arange(s) + 1) * m - 1]
    assert np.array_equal(tr["splitters"], g)
    a = np.zeros((m, s), np.int64)
    for i in range(m):
        v = min(max(n - i * L, 0), L)
        row = comp[i * L:(i + 1) * L][:v]
        prev = 0
        for j in range(s):
            c = int(np.count_nonzero(row <= g[j]))
            a[i, j] = c - prev
            prev = c
    assert np.array_equal(tr["a"], a)
    R = np.zeros(n, np.uint32)
    for i in range(m):
        st = 0
        for j in range(s):
            R[tr["l"][i, j]:tr["l"][i, j] + a[i, j]] = A[i * L + st:i * L + st + a[i, j]]
            st += a[i, j]
    assert np.array_equal(tr["relocated"], R)


def test_determinism_repeatable():
    k = gi.generate("det_duplicates", 1 << 15, seed=2)
    t1, t2 = _trace(k, [(1024, 32)]), _trace(k, [(1024, 32)])
    for f in t1:
        assert np.array_equal(t1[f], t2[f]), f


# ------------------------------------------------------------ paper + SPEC examples

def test_paper_worked_parameters():
    """P:249-259 (n=32M, n/m=2K, m=16K, 512 threads x 4 items), P:269-274 (s=64,
    sm=1M), P:299-300 (log s = 6 rounds), P:318-319 (|B_j| <= 2n/s = 1M)."""
    n, L, s = 32 * 2**20, 2048, 64
    m, npr, hi, lo, last = oracle.bucket_bound(n, L, s)
    assert m == 16 * 1024 and 512 * 4 == L and m * s == 2**20
    assert s.bit_length() - 1 == 6
    assert 2 * n // s == 2**20
    assert hi == 1032161 and hi <= 2 * n // s and last == n // s


def test_spec_local_samples_S105_S107():
    out = oracle.local_samples(np.arange(1, 9), 0, 8, 4)
    assert [int(x) >> 32 for x in out] == [2, 4, 6, 8]
    out = oracle.local_samples(np.arange(2048), 0, 2048, 64)
    assert [int(x) & 0xFFFFFFFF for x in out] == list(range(31, 2048, 32))


def test_spec_global_samples_S123():
    g = oracle.global_samples(np.arange(8, dtype=np.uint64) * 10, 2, 4)
    assert list(g) == [10, 30, 50, 70]


def test_spec_sample_index_S132():
    big = 1 << 31
    a, _ = oracle.sample_index([10, 20, 30, 40], 0, 4,
                               [oracle.composite(25, big), oracle.composite(100, big)])
    assert list(a) == [2, 2]
    # upper-bucket inclusive rule (R4): an item equal to g_j in (key, tag) is in bucket j
    a, _ = oracle.sample_index([10, 20, 30, 40], 0, 4,
                               [oracle.composite(20, 1), oracle.composite(40, 3)])
    assert list(a) == [2, 2]
    a, _ = oracle.sample_index([10, 20, 30, 40], 0, 4,
                               [oracle.composite(20, 0), oracle.composite(40, 3)])
    assert list(a) == [1, 3]


def test_spec_offsets_S141():
    assert oracle.offsets(np.array([[1, 3], [2, 2]])).tolist() == [[0, 3], [1, 6]]
    assert oracle.offsets(np.zeros((3, 4))).tolist() == np.zeros((3, 4)).tolist()
    assert oracle.offsets(np.array([[3, 1, 4, 1]])).tolist() == [[0, 3, 4, 8]]


def test_spec_relocate_single_row_identity_S150():
    rng = np.random.default_rng(2)
    k = rng.integers(0, 1 << 32, 1024, dtype=np.uint64).astype(np.uint32)
    tr = _trace(k, [(1024, 16)])          # m = 1
    assert np.array_equal(tr["relocated"], tr["sorted_keys"])


# ------------------------------------------------------------ plans + multi-GPU outer level

def test_plan_rule_table_P():
    """DESIGN.md section 5 plans for the five configs."""
    assert plan(1 << 16, cfg=(2048, 64)) == [(2048, 64)]
    assert plan(1 << 25) == [(TILE_KEYS, 2048)] and hi_bound(1 << 25, TILE_KEYS, 2048) == 31729
    # one tile would need d = 8 here: sublists of two tiles (CTA pairs), buckets one tile
    assert plan(1 << 26) == [(2 * TILE_KEYS, 4096)] and hi_bound(1 << 26, 2 * TILE_KEYS, 4096) == 31729
    assert hi_bound(1 << 26, TILE_KEYS, 4096) == 30713
    assert plan(3 << 24) == [(2 * TILE_KEYS, 4096)] and plan((1 << 25) + 1) == [(TILE_KEYS, 2048)]
    assert all(hi_bound(n, *plan(n)[0]) <= TILE_KEYS for n in (1 << 22, 3 << 24, 1 << 26))
    assert plan(1 << 30, TILE_PAIRS) == [(TILE_PAIRS, 512), (TILE_PAIRS, 512)]
    assert hi_bound(1 << 30, TILE_PAIRS, 512) == 4128737
    assert hi_bound(4128737, TILE_PAIRS, 512) == 15845


@pytest.mark.parametrize("p", [1, 2, 4, 8])
@pytest.mark.parametrize("dist", ["uniform", "zero", "det_duplicates", "staggered"])
def test_psrs_outer_level(p, dist):
    n_local, s_r = 4096, 64
    k = gi.generate(dist, n_local * p, seed=p)
    out, counts, cuts = oracle.psrs(k, p, s_r)
    assert np.array_equal(out, np.sort(k))
    assert counts.sum() == k.size
    assert counts.max() <= n_local + (p - 1) * (n_local // s_r - 1)
    assert np.all(np.diff(cuts, axis=1) >= 0) and np.all(cuts[:, -1] == n_local)


# --- 64-bit keys: the oracle's plain definition, pinned ----------------------------------

def test_sort64_pins():
    """oracle.sort64 against hand values (IEEE-754 totalOrder, section 5.10) and numpy."""
    f = np.array([1.0, -0.0, 0.0, -np.inf, np.inf, -1.0, 0.0, -0.0], np.float64)
    nan_pos = np.array([0x7FF8000000000001], np.uint64).view(np.float64)[0]
    nan_neg = np.array([0xFFF8000000000001], np.uint64).view(np.float64)[0]
    x = np.concatenate([f, [nan_pos, nan_neg]])
    vals = np.arange(x.size, dtype=np.uint32)
    k, v = oracle.sort64(x, vals, "float64")
    # -NaN, -inf, -1, -0 (input 1), -0 (input 7), +0 (2), +0 (6), 1, inf, +NaN
    assert list(v) == [9, 3, 5, 1, 7, 2, 6, 0, 4, 8]
    rng = np.random.default_rng(0)
    u = rng.integers(0, 1 << 63, 5000, dtype=np.uint64) * 2 + rng.integers(0, 2, 5000, dtype=np.uint64)
    u[::7] = u[0]
    ks, vs = oracle.sort64(u, np.arange(u.size, dtype=np.uint32), "uint64")
    order = np.argsort(u, kind="stable")
    assert np.array_equal(ks, u[order]) and np.array_equal(vs, order.astype(np.uint32))
    i = u.view(np.int64)
    ks, vs = oracle.sort64(i, np.arange(i.size, dtype=np.uint32), "int64")
    order = np.argsort(i, kind="stable")
    assert np.array_equal(ks, i[order]) and np.array_equal(vs, order.astype(np.uint32))
    g = rng.standard_normal(3000) * 1e300
    ks, _ = oracle.sort64(g, None, "float64")
    assert np.array_equal(ks, np.sort(g))
