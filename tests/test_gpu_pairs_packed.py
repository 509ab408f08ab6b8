"""GPU (-m gpu): the pairs tile sort on packed (prefix, position) items and its exact
fix-up (gbs_kernels.cuh, Seg<KIND_PAIRS>): inputs built to hit each of its paths, compared
with the oracle (stable pairs, R7) element by element.

- full-range uniform keys: prefix groups of 1-4 items, a few transposition round pairs;
- clusters of 2-300 keys sharing a prefix, written in random order: the fixed round count
  (groups of at most 32, within one thread or across one thread boundary), the voting
  loop (longer groups) and the composite fallback;
- a tile whose keys span 0 .. 2^32-1 while almost all of them lie below 2^14: one prefix
  group of the whole tile, unsorted -> the composite fallback;
- equal keys inside a prefix group (stability inside the fix-up)."""
import numpy as np
import pytest

import gbs_inputs as gi
import oracle
from plans import TILE_PAIRS, plan

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


def run_pairs(keys, dev):
    n = len(keys)
    vals = gi.pair_values(n)
    k = torch.from_numpy(keys.astype(np.uint32).view(np.int32)).to(dev)
    v = torch.from_numpy(vals.view(np.int32)).to(dev)
    gbs.sort_pairs(k, v)
    torch.cuda.synchronize()
    ek, ev, _ = oracle.gbs_sort(keys.astype(np.uint32), vals, plan=plan(n, TILE_PAIRS))
    assert np.array_equal(k.cpu().numpy().view(np.uint32), ek)
    assert np.array_equal(v.cpu().numpy().view(np.uint32), ev)


def rng_u32(seed, n, hi=1 << 32):
    return np.random.default_rng(seed).integers(0, hi, n, dtype=np.uint64).astype(np.uint32)


@pytest.mark.parametrize("n", [16384, 16385, 1 << 20, (1 << 20) + 77])
def test_full_range_uniform(dev, n):
    run_pairs(gi.generate("uniform", n, seed=7), dev)


@pytest.mark.parametrize("n", [16384, (1 << 20) + 5])
@pytest.mark.parametrize("cluster", [2, 3, 8, 16, 31, 32, 33, 40, 64, 300])
def test_prefix_clusters(dev, n, cluster):
    """Uniform keys plus, every 4096 positions, `cluster` keys from one window of 2^14
    values (they share a prefix at full range) in random order, some of them equal."""
    keys = rng_u32(11, n)
    r = np.random.default_rng(cluster)
    for s0 in range(0, n - cluster, 4096):
        base = r.integers(0, (1 << 32) - (1 << 14))
        keys[s0:s0 + cluster] = base + r.integers(0, 1 << 14, cluster) // 3 * 3
    run_pairs(keys, dev)


@pytest.mark.parametrize("n", [16384, 3 * 16384 + 11, (1 << 20) + 9])
def test_whole_tile_group_fallback(dev, n):
    """Every 16K tile holds 0 and 2^32 - 1 and otherwise keys below 2^14 (many equal): the
    prefix is key >> 14 = 0 for nearly the whole tile, in random key order."""
    keys = rng_u32(3, n, 1 << 14)
    keys[::16384] = 0xFFFFFFFF
    keys[1::16384] = 0
    run_pairs(keys, dev)


def test_equal_keys_in_groups(dev):
    """Few distinct keys spread over the full range, each repeated many times: equal keys
    share a prefix group, their order must stay the input order."""
    n = (1 << 20) + 3
    distinct = rng_u32(5, 97)
    keys = distinct[np.random.default_rng(6).integers(0, 97, n)]
    run_pairs(keys, dev)
