"""Host-side checks of libgbs.so that need no GPU (-m "not gpu"): the library loads
and exports every symbol include/gbs.h declares; the planner matches the plan rule
of DESIGN.md section 5 (restated independently in tests/plans.py); argument
validation happens before any device work; the multi-GPU exchange plan."""
import os
import re

import numpy as np
import pytest

import paper_1002_4464_b200 as gbs
from plans import TILE_KEYS, TILE_PAIRS, hi_bound, plan

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1002_4464_b200 import _build
    _build.build()


def test_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "gbs.h")).read()
    declared = set(re.findall(r"\b(gbs_[a-z_]+)\s*\(", hdr))
    assert len(declared) >= 17
    L = gbs.lib()
    for name in sorted(declared):
        assert hasattr(L, name), name


@pytest.mark.parametrize("n", [2, 100, 2048, 32768, 32769, 65536, 100000, 1 << 20, 3 * (1 << 20) + 7,
                               1 << 25, 1 << 26, 100_000_000, 1 << 27, (1 << 27) + 12345, 1 << 28, 1 << 29,
                               1 << 31])
def test_plan_matches_rule_keys(n):
    p = gbs.plan(n)
    exp = plan(n, TILE_KEYS)
    assert p["levels"] == exp
    cap = n
    for k, (L, s) in enumerate(exp):
        assert p["cap"][k] == cap and p["bucket_bound"][k] == hi_bound(cap, L, s)
        assert p["m"][k] == -(-cap // L)
        cap = hi_bound(cap, L, s)
    # Step 9 buckets fit one CTA tile, or -- a one-level top plan only -- a CTA pair's two
    assert cap <= TILE_KEYS or (len(exp) == 1 and cap <= 2 * TILE_KEYS)


@pytest.mark.parametrize("n", [2, 16384, 16385, 1 << 20, 1 << 26, 1 << 30])
def test_plan_matches_rule_pairs(n):
    assert gbs.plan(n, pairs=True)["levels"] == plan(n, TILE_PAIRS)


def test_plan_paper_config():
    """The paper's parameters (L = 2K items, s = 64) at C1."""
    p = gbs.plan(1 << 16, cfg=(2048, 64))
    assert p["levels"] == [(2048, 64)] and p["m"] == [32] and p["bucket_bound"] == [1985]
    p = gbs.plan(32 << 20, cfg=(2048, 64))        # paper's n = 32M: needs a nested Step 9
    assert p["levels"][0] == (2048, 64) and p["bucket_bound"][0] == 1032161


def test_plan_is_data_independent_and_small_n():
    assert gbs.plan(0)["levels"] == [] and gbs.plan(1)["ws_bytes"] == 0
    assert gbs.workspace_size(1 << 25) == gbs.plan(1 << 25)["ws_bytes"] > 4 * (1 << 25)


def test_validation_before_device_work():
    L = gbs.lib()
    import ctypes as C
    # NULL keys with n > 1 -> INVALID_VALUE (rejected before any device query)
    assert L.gbs_sort_keys(None, 10, None, 0, None) == 1
    # bad configs
    for cfg in [(3000, 64), (2048, 4096), (1 << 17, 64), (64, 128)]:
        with pytest.raises(gbs.GbsError):
            gbs.plan(1 << 16, cfg=cfg)
    # sublists of two tiles (CTA-pair local sort) are keys-only
    assert gbs.plan(1 << 20, cfg=(1 << 16, 64))["levels"][0] == (1 << 16, 64)
    with pytest.raises(gbs.GbsError):
        gbs.plan(1 << 20, pairs=True, cfg=(1 << 15, 64))
    with pytest.raises(gbs.GbsError):
        gbs.plan((1 << 31) + 1)
    # workspace too small is reported, not crashed on
    assert L.gbs_sort_keys(C.c_void_p(16), 1 << 20, C.c_void_p(256), 10, None) == 2
    assert L.gbs_sort_keys(None, 0, None, 0, None) == 0 and L.gbs_sort_keys(None, 1, None, 0, None) == 0
    # typed keys: a bad key type, NULL keys, a short workspace -- all rejected before the
    # in-place key transform is enqueued
    assert L.gbs_sort_keys_typed(C.c_void_p(16), 100, 7, None, 0, None) == 1
    assert L.gbs_sort_keys_typed(None, 100, 2, None, 0, None) == 1
    assert L.gbs_sort_keys_typed(C.c_void_p(16), 1 << 20, 1, C.c_void_p(256), 10, None) == 2
    assert L.gbs_sort_pairs_typed(C.c_void_p(16), None, 100, 2, None, 0, None) == 1
    assert L.gbs_sort_keys_typed(None, 1, 2, None, 0, None) == 0


def test_exchange_plan_against_direct_definition():
    """E7-E8: rank k receives S_r[cut_{r,k-1}, cut_{r,k}) from every r, in rank order."""
    rng = np.random.default_rng(0)
    for p in (1, 2, 3, 8):
        n_local = 1000
        cuts = np.sort(rng.integers(0, n_local + 1, (p, p)), axis=1).astype(np.uint64)
        cuts[:, -1] = n_local
        total = 0
        for rank in range(p):
            e = gbs.exchange_plan(cuts, rank)
            lo = np.concatenate([[0], cuts[rank, :-1]])
            assert np.array_equal(e["send_off"], lo) and np.array_equal(e["send_cnt"], cuts[rank] - lo)
            rc = np.array([cuts[r, rank] - (cuts[r, rank - 1] if rank else 0) for r in range(p)], np.uint64)
            assert np.array_equal(e["recv_cnt"], rc)
            assert np.array_equal(e["recv_off"], np.concatenate([[0], np.cumsum(rc)[:-1]]).astype(np.uint64))
            total += e["n_out"]
        assert total == p * n_local
    bad = np.array([[5, 3], [1, 10]], np.uint64)
    with pytest.raises(gbs.GbsError):
        gbs.exchange_plan(bad, 0)
