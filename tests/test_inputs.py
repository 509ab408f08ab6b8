"""Input generator pins (gbs_inputs): SplitMix64 known value, twin agreement, shapes."""
import numpy as np
import pytest

import gbs_inputs as gi


def test_splitmix64_known_first_output():
    # The first output of SplitMix64 seeded with 0 is 0xE220A8397B1DCDAF
    # (Steele, Lea, Flood 2014 reference generator; widely tabulated).
    z = gi._mix_np(np.array([gi.GAMMA], dtype=np.uint64))
    assert int(z[0]) == 0xE220A8397B1DCDAF
    assert int(gi.generate("uniform", 1, seed=0)[0]) == 0xE220A839


@pytest.mark.parametrize("dist", gi.DISTRIBUTIONS)
@pytest.mark.parametrize("n", [1, 255, 1000, 1 << 16, 100003])
def test_torch_twin_matches_numpy(dist, n):
    a = gi.generate(dist, n, seed=4)
    b = gi.generate_torch(dist, n, seed=4, chunk=1 << 14).numpy().view(np.uint32)
    assert np.array_equal(a, b)


def test_slices_compose():
    n = 1 << 16
    for dist in ("uniform", "gaussian", "bucket_sorted", "staggered", "det_duplicates"):
        full = gi.generate(dist, n, seed=9)
        parts = np.concatenate([gi.generate(dist, n, 9, start=s, count=n // 4)
                                for s in range(0, n, n // 4)])
        assert np.array_equal(full, parts)


def test_distribution_shapes():
    n = 1 << 16
    assert np.all(gi.generate("zero", n) == 0)
    s = gi.generate("sorted", n, 1)
    assert np.all(np.diff(s.astype(np.int64)) >= 0)
    assert np.array_equal(np.sort(gi.generate("uniform", n, 1)), s)
    bs = gi.generate("bucket_sorted", n).astype(np.int64)
    b = n // 256
    assert np.all(bs[:b] >> 24 == np.arange(b) // (b // 256))   # block 0 walks 256 sub-buckets
    st = gi.generate("staggered", n).astype(np.int64) >> 24
    assert st[0] == 1 and st[128 * b] == 0 and st[255 * b] == 254
    dd = gi.generate("det_duplicates", n)
    assert len(np.unique(dd)) <= 17 and dd.max() == 16
    g = gi.generate("gaussian", n).astype(np.float64)
    assert abs(g.mean() / 2**32 - 0.5) < 0.01 and g.std() / 2**32 < 0.2
