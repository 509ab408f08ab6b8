"""GPU parity of the multi-GPU path at p > 1 on ONE GPU (-m gpu).

`gbs_sort_keys_dist_emulated` runs the same per-rank phases as `gbs_sort_keys_dist`
(E1-E2 local sort + regular samples, E4-E6 sample sort + cut points, E9 p-way merge)
for ranks 0..p-1 in turn, with the collectives (E3/E7 allgathers, E8 all-to-all)
replaced by device copies.  Compared with the CPU oracle's PSRS outer level
(oracle/gbs_oracle.c): every rank's part bit-exact, the receive counts
equal, and the receive bound n_l + (p-1)(n_l/s_r - 1) respected."""
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


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("n_local", [1 << 16, (1 << 20) + 64])
@pytest.mark.parametrize("dist", ["uniform", "zero", "det_duplicates", "staggered", "sorted"])
def test_dist_emulated_matches_oracle_psrs(dev, p, n_local, dist):
    keys = gi.generate(dist, p * n_local, seed=p)
    shards = torch.from_numpy(keys.view(np.int32).copy()).to(dev)
    parts = gbs.sort_keys_dist_emulated(shards, p)
    torch.cuda.synchronize()
    s_r = s_r_of(n_local)
    exp, counts, _ = oracle.psrs(keys, p, s_r)
    got_counts = [t.numel() for t in parts]
    assert got_counts == [int(c) for c in counts]
    assert max(got_counts) <= n_local + (p - 1) * (n_local // s_r - 1)
    got = np.concatenate([t.cpu().numpy().view(np.uint32) for t in parts])
    assert np.array_equal(got, exp)
    assert np.array_equal(exp, np.sort(keys))
