"""GPU (-m gpu): signed and float keys (gbs_sort_keys_typed / gbs_sort_pairs_typed, SURVEY
8(f) NEXT-4) against numpy's sorts of the same values.

int32 keys: the result equals np.sort exactly.  float32 keys: for non-NaN values the result
equals np.sort by value (numpy treats -0 == +0), every -0 precedes every +0 (IEEE-754
totalOrder), the output is a permutation of the input bit patterns, and NaNs sit at the
ends by sign.  Pairs: equal to numpy's stable argsort by key (inputs without -0, where
numpy's value order and totalOrder agree)."""
import numpy as np
import pytest

import gbs_inputs as gi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_1002_4464_b200 as gbs  # noqa: E402

SIZES = [2, 1000, (1 << 16) + 3, (1 << 20) + 5, 1 << 22]


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1002_4464_b200 import _build
    _build.build()
    return torch.device("cuda:0")


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("dist", ["uniform", "gaussian", "staggered", "det_duplicates", "zero"])
def test_int32_keys(dev, n, dist):
    keys = gi.generate(dist, n, seed=3).view(np.int32)
    t = torch.from_numpy(keys.copy()).to(dev)
    gbs.sort_keys_typed(t)
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy(), np.sort(keys))


def _floats(n, seed, nan=False):
    bits = gi.generate("uniform", n, seed=seed)
    f = bits.view(np.float32).copy()
    if not nan:
        f[np.isnan(f)] = 1.5
    if n >= 8:
        f[:4] = [0.0, -0.0, np.inf, -np.inf]
        f[n // 2:n // 2 + 4] = [-0.0, 0.0, -0.0, 0.0]
    return f


@pytest.mark.parametrize("n", SIZES)
def test_float32_keys_total_order(dev, n):
    f = _floats(n, seed=5)
    t = torch.from_numpy(f.copy()).to(dev)
    gbs.sort_keys_typed(t)
    torch.cuda.synchronize()
    got = t.cpu().numpy()
    assert np.array_equal(got, np.sort(f))                          # by value
    zeros = got[got == 0]
    nneg = int(np.signbit(zeros).sum())
    assert not np.signbit(zeros[nneg:]).any() and np.signbit(zeros[:nneg]).all()   # -0 before +0
    assert np.array_equal(np.sort(got.view(np.uint32)), np.sort(f.view(np.uint32)))  # permutation


@pytest.mark.parametrize("n", [1000, (1 << 20) + 5])
def test_float32_keys_with_nans(dev, n):
    f = _floats(n, seed=7, nan=True)
    isn = np.isnan(f)
    assert isn.any()
    neg_nan = int((isn & np.signbit(f)).sum())
    pos_nan = int((isn & ~np.signbit(f)).sum())
    t = torch.from_numpy(f.copy()).to(dev)
    gbs.sort_keys_typed(t)
    torch.cuda.synchronize()
    got = t.cpu().numpy()
    assert np.isnan(got[:neg_nan]).all() and np.signbit(got[:neg_nan]).all()
    assert np.isnan(got[n - pos_nan:]).all() and not np.signbit(got[n - pos_nan:]).any()
    assert np.array_equal(got[neg_nan:n - pos_nan], np.sort(f[~isn]))
    assert np.array_equal(np.sort(got.view(np.uint32)), np.sort(f.view(np.uint32)))


@pytest.mark.parametrize("n", [1000, (1 << 16) + 3, (1 << 20) + 5])
@pytest.mark.parametrize("kind", ["int32", "float32"])
def test_typed_pairs_stable(dev, n, kind):
    u = gi.generate("uniform", n, seed=9)
    if kind == "int32":
        keys = ((u % 2001).astype(np.int64) - 1000).astype(np.int32)   # many duplicates
    else:
        keys = ((u % 2001).astype(np.float32) - 1000.0) / 8.0          # no -0 (x - 1000 is +0 at 1000)
    vals = gi.pair_values(n)
    kt = torch.from_numpy(keys.copy()).to(dev)
    vt = torch.from_numpy(vals.view(np.int32).copy()).to(dev)
    gbs.sort_pairs_typed(kt, vt)
    torch.cuda.synchronize()
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(kt.cpu().numpy(), keys[order])
    assert np.array_equal(vt.cpu().numpy().view(np.uint32), vals[order])
