"""GPU parity of the multi-GPU path at p > 1 on ONE GPU (-m gpu).

`gbs_sort_keys_dist_emulated` runs the same per-rank kernels as `gbs_sort_keys_dist`
with the peer-memory transport -- E1 local sort, E2-E3 samples stored into every rank's
window, E4-E7 sample sort + fine cuts stored into every window, E8 relocation of the
runs straight into the owners' receive buffers, E9 one-pass k-way merge -- for ranks
0..p-1 in turn, with the p windows as regions of one workspace and stream order in
place of the device barriers.  Compared with the CPU oracle's PSRS outer level
(oracle/gbs_oracle.c): every rank's part bit-exact, the receive counts
equal, the receive bound n_l + (p-1)(n_l/s_r - 1) respected, the input unchanged."""
import numpy as np
import pytest

import gbs_inputs as gi
import oracle

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


def s_r_of(n_local: int) -> int:
    """E2: the largest power of two <= 1024 dividing n_local."""
    s = 1
    while s < 1024 and n_local % (2 * s) == 0:
        s *= 2
    return s


def check_emulated(dev, p, n_local, dist, seed):
    keys = gi.generate(dist, p * n_local, seed=seed)
    shards = torch.from_numpy(keys.view(np.int32).copy()).to(dev)
    parts = gbs.sort_keys_dist_emulated(shards, p)
    torch.cuda.synchronize()
    assert np.array_equal(shards.cpu().numpy().view(np.uint32), keys), "input modified"
    s_r = s_r_of(n_local)
    exp, counts, _ = oracle.psrs(keys, p, s_r)
    got_counts = [t.numel() for t in parts]
    assert got_counts == [int(c) for c in counts]
    assert max(got_counts) <= n_local + (p - 1) * (n_local // s_r - 1)
    got = np.concatenate([t.cpu().numpy().view(np.uint32) for t in parts])
    assert np.array_equal(got, exp)
    assert np.array_equal(exp, np.sort(keys))


@pytest.mark.parametrize("p", [2, 3, 4, 8, 16])
@pytest.mark.parametrize("n_local", [1 << 16, (1 << 20) + 64, 3 * 4099])
@pytest.mark.parametrize("dist", ["uniform", "zero", "det_duplicates", "staggered", "sorted", "gaussian",
                                  "bucket_sorted"])
def test_dist_emulated_matches_oracle_psrs(dev, p, n_local, dist):
    check_emulated(dev, p, n_local, dist, seed=p)


def test_dist_emulated_2_27_per_rank(dev):
    """One case at C5-like shard size: 2^27 keys per rank, p = 2 (the oracle sorts 2^28)."""
    check_emulated(dev, 2, 1 << 27, "uniform", seed=5)
