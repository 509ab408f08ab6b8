"""GPU parity (-m gpu): the CUDA path through the C-ABI vs the CPU oracle, bit-exact.

Integer sort: the final output is unique, every intermediate is fixed
by the plan and the readings of DESIGN.md section 3, so every comparison is exact
equality.  Inputs: gbs_inputs (seeded, the seven distributions of the north star)."""
import numpy as np
import pytest

import gbs_inputs as gi
import oracle
from plans import TILE_KEYS, TILE_PAIRS, plan

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1002_4464_b200 as gbs  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1002_4464_b200 import _build
    _build.build()
    return torch.device("cuda:0")


def to_dev(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).to(dev)


def to_np(t):
    return t.cpu().numpy().view(np.uint32)


def gpu_sort(keys, dev, vals=None, cfg=None, stop=0, ws=None):
    k = to_dev(keys, dev)
    v = to_dev(vals, dev) if vals is not None else None
    gbs.sort_ex(k, v, cfg=cfg, stop_after_step=stop, ws=ws)
    torch.cuda.synchronize()
    return to_np(k), (to_np(v) if v is not None else None)


SIZES = [0, 1, 2, 3, 31, 1023, 2048, 2049, 32768, 32769, 65536, 100003, 1 << 20, 3 * (1 << 20) + 17,
         (1 << 22) + 12345]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("dist", gi.DISTRIBUTIONS)
def test_keys_default_plan(dev, n, dist):
    keys = gi.generate(dist, n, seed=n % 5)
    got, _ = gpu_sort(keys, dev)
    exp, _, _ = oracle.gbs_sort(keys, plan=plan(n, TILE_KEYS))
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("n,cfg", [((1 << 22) + 12345, (1 << 16, 256)), (5_000_003, (1 << 16, 1024)),
                                   (70_000, (1 << 16, 16))])
@pytest.mark.parametrize("dist", gi.DISTRIBUTIONS)
def test_keys_cta_pair_plan(dev, n, cfg, dist):
    """Sublists of two tiles sorted by a CTA pair (NEXT-2): ragged last sublists whose
    second half is empty or partial."""
    keys = gi.generate(dist, n, seed=n % 5)
    got, _ = gpu_sort(keys, dev, cfg=cfg)
    exp, _, _ = oracle.gbs_sort(keys, plan=plan(n, TILE_KEYS, cfg))
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("seed", range(5))
@pytest.mark.parametrize("dist", gi.DISTRIBUTIONS)
def test_keys_C1_paper_plan(dev, seed, dist):
    """C1: 2^16 keys with the paper's L = 2K, s = 64."""
    n = 1 << 16
    keys = gi.generate(dist, n, seed=seed)
    got, _ = gpu_sort(keys, dev, cfg=(2048, 64))
    exp, _, _ = oracle.gbs_sort(keys, plan=plan(n, cfg=(2048, 64)))
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("cfg,n", [((2048, 64), 1 << 16), (None, 1 << 16), (None, 3 * (1 << 20) + 17),
                                   ((4096, 256), 500_000), ((1024, 32), 300_001),
                                   ((1 << 16, 512), 3_000_017), ((1 << 16, 64), 100_000)])
@pytest.mark.parametrize("dist", ["uniform", "zero", "det_duplicates", "staggered"])
def test_stage_parity(dev, cfg, n, dist):
    """Every level-1 intermediate equals the oracle's: sorted sublists (Step 2), samples
    (3), sorted samples (4), splitters (5), a (6), l (7), R (8)."""
    keys = gi.generate(dist, n, seed=3)
    pl = plan(n, TILE_KEYS, cfg)
    _, _, tr = oracle.gbs_sort(keys, plan=pl, trace=True)
    lay = gbs.debug_layout(n, cfg=cfg)
    m, s = tr["a"].shape
    ws = torch.zeros(gbs.workspace_size(n, cfg=cfg), dtype=torch.uint8, device=dev)

    def view(off, count, dtype):
        nb = count * np.dtype(dtype).itemsize
        return ws[off:off + nb].cpu().numpy().view(dtype)

    got, _ = gpu_sort(keys, dev, cfg=cfg, stop=2, ws=ws)
    assert np.array_equal(got, tr["sorted_keys"])
    assert np.array_equal(view(lay["samples"], m * s, np.uint64), tr["samples"])
    gpu_sort(keys, dev, cfg=cfg, stop=5, ws=ws)
    assert np.array_equal(view(lay["samples"], m * s, np.uint64), tr["sorted_samples"])
    assert np.array_equal(view(lay["splitters"], s, np.uint64), tr["splitters"])
    gpu_sort(keys, dev, cfg=cfg, stop=8, ws=ws)
    assert np.array_equal(view(lay["a"], m * s, np.uint32).reshape(m, s), tr["a"])
    assert np.array_equal(view(lay["l"], m * s, np.uint32).reshape(m, s), tr["l"])
    assert np.array_equal(view(lay["relocated"], n, np.uint32), tr["relocated"])


@pytest.mark.parametrize("cfg,n", [(None, 1 << 25), (None, 3 * (1 << 20) + 17), ((4096, 256), 500_000),
                                   ((1 << 16, 512), 3_000_017), ((2048, 64), (1 << 20) + 3),
                                   ((32768, 4096), 7 * (1 << 20) + 5)])
@pytest.mark.parametrize("dist", ["uniform", "zero", "det_duplicates", "sorted"])
def test_step4_splitter_selection(dev, cfg, n, dist):
    """Step 4 as a merge tree with selection (R22; every plan here has more
    than one tile of samples, some an odd number of sample runs): the splitters the
    production path selects (stop after Step 6, not the full-merge stage-parity form of
    stop 4/5) equal the oracle's g_k = sorted[(k+1)m - 1], and so do the counts a."""
    keys = gi.generate(dist, n, seed=11)
    pl = plan(n, TILE_KEYS, cfg)
    _, _, tr = oracle.gbs_sort(keys, plan=pl, trace=True)
    m, s = tr["a"].shape
    assert m * s > (1 << 14)
    lay = gbs.debug_layout(n, cfg=cfg)
    ws = torch.zeros(gbs.workspace_size(n, cfg=cfg), dtype=torch.uint8, device=dev)
    gpu_sort(keys, dev, cfg=cfg, stop=6, ws=ws)
    spl = ws[lay["splitters"]:lay["splitters"] + 8 * s].cpu().numpy().view(np.uint64)
    assert np.array_equal(spl, tr["splitters"])
    a = ws[lay["a"]:lay["a"] + 4 * m * s].cpu().numpy().view(np.uint32).reshape(m, s)
    assert np.array_equal(a, tr["a"])


@pytest.mark.parametrize("n", [2, 1000, 16384, 16385, 65536, 1 << 20, 2_000_003])
@pytest.mark.parametrize("dist", ["uniform", "zero", "det_duplicates", "sorted", "gaussian"])
def test_pairs_stable(dev, n, dist):
    keys = gi.generate(dist, n, seed=1)
    if dist == "uniform":
        keys = keys % 1000                         # many duplicates: stability is observable
    vals = gi.pair_values(n)
    gk, gv = gpu_sort(keys, dev, vals=vals)
    ek, ev, _ = oracle.gbs_sort(keys, vals, plan=plan(n, TILE_PAIRS))
    assert np.array_equal(gk, ek) and np.array_equal(gv, ev)


def test_nested_level_keys(dev):
    """A plan with a nested Step 9 (paper's L = 2K, s = 64 at n = 2^21: bucket bound
    > one tile) -- the batched level over all buckets."""
    n = (1 << 21) + 5
    for dist in ("uniform", "zero", "det_duplicates"):
        keys = gi.generate(dist, n, seed=2)
        pl = plan(n, TILE_KEYS, (2048, 64))
        assert len(pl) == 2
        got, _ = gpu_sort(keys, dev, cfg=(2048, 64))
        exp, _, _ = oracle.gbs_sort(keys, plan=pl)
        assert np.array_equal(got, exp)


def test_nested_level_pairs(dev):
    n = (1 << 20) + 3
    keys = gi.generate("uniform", n, seed=4) % 5000
    vals = gi.pair_values(n)
    pl = plan(n, TILE_PAIRS, (1024, 16))
    assert len(pl) == 2
    gk, gv = gpu_sort(keys, dev, vals=vals, cfg=(1024, 16))
    ek, ev, _ = oracle.gbs_sort(keys, vals, plan=pl)
    assert np.array_equal(gk, ek) and np.array_equal(gv, ev)


def test_determinism_intermediates(dev):
    n = 1 << 20
    keys = gi.generate("det_duplicates", n, seed=0)
    lay = gbs.debug_layout(n)
    outs = []
    for _ in range(3):
        ws = torch.zeros(gbs.workspace_size(n), dtype=torch.uint8, device=dev)
        got, _ = gpu_sort(keys, dev, stop=8, ws=ws)
        outs.append(ws[lay["a"]:lay["relocated"]].cpu().numpy().copy())
    assert all(np.array_equal(outs[0], o) for o in outs[1:])


def test_host_e2e_entry(dev):
    n = 1 << 20
    keys = gi.generate("uniform", n, seed=7)
    h = torch.from_numpy(keys.view(np.int32).copy()).pin_memory()
    d = torch.empty(n, dtype=torch.int32, device=dev)
    gbs.sort_keys_host(h, d)
    torch.cuda.synchronize()
    assert np.array_equal(h.numpy().view(np.uint32), np.sort(keys))


@pytest.mark.parametrize("n,dist", [((1 << 21) + 1, "uniform"), ((1 << 22) + 12345, "det_duplicates"),
                                    (1 << 25, "uniform"), (1 << 25, "zero"), (1 << 25, "sorted"),
                                    ((1 << 25) - 777, "staggered"), (1 << 24, "gaussian")])
def test_host_e2e_pipelined(dev, n, dist):
    """gbs_sort_keys_host above 2^21 keys: H2D in chunks of sublists overlapping Step 2,
    Step 9 in bucket groups whose guaranteed-final output prefix is copied back while
    the next groups sort (R18).  Output = the plain sort of the input."""
    keys = gi.generate(dist, n, seed=5)
    h = torch.from_numpy(keys.view(np.int32).copy()).pin_memory()
    d = torch.empty(n, dtype=torch.int32, device=dev)
    for _ in range(2):                               # twice: the second reuses the streams
        h.copy_(torch.from_numpy(keys.view(np.int32)))
        gbs.sort_keys_host(h, d)
        torch.cuda.synchronize()
        assert np.array_equal(h.numpy().view(np.uint32), np.sort(keys))


@pytest.mark.parametrize("dist", gi.DISTRIBUTIONS)
def test_C2_C3_full_size(dev, dist):
    """C2 (2^25 uniform) and C3 (2^26, all seven distributions) in the launch
    configuration bench.py times; compared with the plain definition (a library sort)."""
    n = 1 << 26
    keys = gi.generate_torch(dist, n, seed=0, device=dev)
    exp = np.sort(keys.cpu().numpy().view(np.uint32))
    gbs.sort_keys(keys)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(keys), exp)
    if dist == "uniform":
        k2 = gi.generate_torch(dist, 1 << 25, seed=0, device=dev)
        exp2, _, _ = oracle.gbs_sort(to_np(k2), plan=plan(1 << 25))
        gbs.sort_keys(k2)
        torch.cuda.synchronize()
        assert np.array_equal(to_np(k2), exp2)


def test_dist_single_rank_nccl(dev):
    """The multi-GPU entry with p = 1 (one NCCL rank): the out-of-place local sort is the
    whole job; output == sort, the input is left unchanged (read only)."""
    import ctypes as C
    L = gbs.lib()
    uid = gbs.get_unique_id()
    h = C.c_void_p()
    idbuf = (C.c_uint8 * 128).from_buffer_copy(uid)
    assert L.gbs_comm_init(C.byref(h), idbuf, 1, 0) == 0

    class _C:
        handle, nranks, rank = h, 1, 0
    n = 1 << 20
    keys = gi.generate("staggered", n, seed=1)
    d = to_dev(keys, dev)
    for _ in range(2):
        out = gbs.sort_keys_dist(d, _C)
        torch.cuda.synchronize()
        assert np.array_equal(to_np(out), np.sort(keys))
        assert np.array_equal(to_np(d), keys)
    assert L.gbs_comm_destroy(h) == 0


def test_C4_pairs_full_size(dev):
    """C4: 2^30 u32 -> u32 pairs (nested Step 9) in the bench's launch configuration.
    Too large for the oracle; checked by properties that define a stable sort:
    keys nondecreasing, values a permutation, keys_out == keys_in[values_out]
    (values are input positions), equal keys keep increasing values."""
    n = 1 << 30
    keys_in = gi.generate_torch("uniform", n, seed=0, device=dev)
    keys = keys_in.clone()
    vals = torch.arange(n, dtype=torch.int32, device=dev)
    assert len(gbs.plan(n, pairs=True)["levels"]) == 2
    gbs.sort_pairs(keys, vals)
    torch.cuda.synchronize()
    k64 = keys.to(torch.int64) & 0xFFFFFFFF
    assert bool((k64[1:] >= k64[:-1]).all())
    seen = torch.zeros(n, dtype=torch.bool, device=dev)
    seen[vals.long()] = True
    assert bool(seen.all())
    del seen
    assert torch.equal(keys_in[vals.long()], keys)
    eq = k64[1:] == k64[:-1]
    assert bool((vals[1:][eq] > vals[:-1][eq]).all())


@pytest.mark.parametrize("args", [("67108864", "32768", "64"), ("16777216", "32768", "512"),
                                  ("33554432", "16384", "128")])
def test_nested_invariants_debug_mode(dev, args):
    """Nested Step 9 with many empty trailing sublists per problem (capacity = bound,
    actual buckets ~half), run with GBS_DEBUG_SYNC=1: every launch synchronised and the
    invariants of Steps 4 (sorted samples) and 6 (sum of a row = real items)
    checked on device at every level; output == the plain definition."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "scripts", "debug_nested.py"), *args],
                       capture_output=True, text=True, env=dict(os.environ, GBS_DEBUG_SYNC="1"), timeout=600)
    assert "ok equal: True" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("n,dist", [(1 << 27, "uniform"), (1 << 27, "zero"), (1 << 27, "staggered"),
                                    ((1 << 27) + 12345, "det_duplicates"), (100_000_000, "gaussian")])
def test_pair_buckets_one_level(dev, n, dist):
    """Sizes whose one-tile buckets would need a nested Step 9 run one level with Step 9 on
    CTA pairs (NEXT-2: buckets of up to 2^16 keys over DSMEM); == the plain definition."""
    p = gbs.plan(n)
    assert len(p["levels"]) == 1 and 1 << 15 < p["bucket_bound"][0] <= 1 << 16
    keys = gi.generate_torch(dist, n, seed=2, device=dev)
    ref = torch.sort(keys.to(torch.int64) & 0xFFFFFFFF).values
    gbs.sort_keys(keys)
    torch.cuda.synchronize()
    assert torch.equal(keys.to(torch.int64) & 0xFFFFFFFF, ref)


def test_pair_buckets_vs_oracle(dev):
    """2^27 uniform keys, the pair-bucket plan [(65536, 4096)], against the CPU oracle run
    with the same plan (element by element)."""
    n = 1 << 27
    keys = gi.generate("uniform", n, seed=9)
    pl = plan(n)
    assert pl == [(65536, 4096)]
    exp, _, _ = oracle.gbs_sort(keys, plan=pl)
    d = to_dev(keys, dev)
    gbs.sort_keys(d)
    torch.cuda.synchronize()
    assert np.array_equal(to_np(d), exp)


@pytest.mark.parametrize("n,dist,pairs", [((1 << 25) + 7, "uniform", True), ((1 << 25) + 7, "det_duplicates", True),
                                          ((1 << 25) + 7, "staggered", True), (1 << 28, "zero", False),
                                          ((1 << 28) + 3, "uniform", False)])
def test_host_e2e_nested(dev, n, dist, pairs):
    """gbs_sort_{keys,pairs}_host with a nested plan: the nested level runs in groups of
    the top level's buckets and each group's guaranteed-final output prefix (R18) is
    copied back while the next groups sort.  Output = the plain (stable) sort."""
    keys = gi.generate(dist, n, seed=6)
    h = torch.from_numpy(keys.view(np.int32).copy()).pin_memory()
    d = torch.empty(n, dtype=torch.int32, device=dev)
    if pairs:
        vals = gi.pair_values(n)
        hv = torch.from_numpy(vals.view(np.int32).copy()).pin_memory()
        dv = torch.empty(n, dtype=torch.int32, device=dev)
        gbs.sort_pairs_host(h, hv, d, dv)
        torch.cuda.synchronize()
        order = np.argsort(keys, kind="stable")
        assert np.array_equal(h.numpy().view(np.uint32), keys[order])
        assert np.array_equal(hv.numpy().view(np.uint32), vals[order])
    else:
        gbs.sort_keys_host(h, d)
        torch.cuda.synchronize()
        assert np.array_equal(h.numpy().view(np.uint32), np.sort(keys))


def test_pair_buckets_host_pipeline(dev):
    """gbs_sort_keys_host with the pair-bucket plan: chunked H2D + Step 2, bucket-group
    D2H of the final prefix while later CTA-pair groups sort."""
    n = (1 << 27) + 77
    keys = gi.generate("bucket_sorted", n, seed=4)
    h = torch.from_numpy(keys.view(np.int32).copy()).pin_memory()
    d = torch.empty(n, dtype=torch.int32, device=dev)
    gbs.sort_keys_host(h, d)
    torch.cuda.synchronize()
    assert np.array_equal(h.numpy().view(np.uint32), np.sort(keys))
