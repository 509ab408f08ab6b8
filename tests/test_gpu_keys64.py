"""GPU (-m gpu): 64-bit keys (gbs_sort_keys64 / gbs_sort_pairs64).

The result has a plain definition: the stable sort by numeric key
(oracle.sort64: u64 / i64 integer order, f64 IEEE-754 totalOrder).  Compared bit for bit
with the oracle up to 2^16 + 3 items (every distribution of the 32-bit family, widened),
and at 2^20 / 2^24 with numpy's stable argsort (the same definition, a library routine)."""
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


def keys64(dist, n, seed, key_type):
    """64-bit keys from two 32-bit draws of the input family: hi from `dist`, lo uniform
    (so equal hi words, duplicates and the structured shapes reach both passes)."""
    hi = gi.generate(dist, n, seed=seed).astype(np.uint64)
    lo = gi.generate("uniform", n, seed=seed + 101).astype(np.uint64)
    if dist in ("zero", "det_duplicates"):
        lo %= np.uint64(7)                           # many fully equal 64-bit keys
    u = (hi << np.uint64(32)) | lo
    if key_type == "uint64":
        return u
    if key_type == "int64":
        return u.view(np.int64)
    f = u.view(np.float64).copy()
    if n >= 16:
        f[:8] = [0.0, -0.0, np.inf, -np.inf, 1.0, -1.0, -0.0, 0.0]
    return f


def to_dev(a, dev):
    t = torch.from_numpy(a.copy())
    return t.to(dev)


@pytest.mark.parametrize("n", [0, 1, 2, 1000, (1 << 16) + 3])
@pytest.mark.parametrize("key_type", ["uint64", "int64", "float64"])
@pytest.mark.parametrize("dist", ["uniform", "zero", "det_duplicates", "staggered", "sorted"])
def test_keys64_vs_oracle(dev, n, key_type, dist):
    k = keys64(dist, n, seed=n % 97, key_type=key_type)
    t = to_dev(k, dev)
    gbs.sort_keys64(t)
    torch.cuda.synchronize()
    exp, _ = oracle.sort64(k, None, key_type)
    assert np.array_equal(t.cpu().numpy().view(np.uint64), exp.view(np.uint64))


@pytest.mark.parametrize("n", [2, 1000, (1 << 16) + 3])
@pytest.mark.parametrize("key_type", ["uint64", "int64", "float64"])
def test_pairs64_vs_oracle(dev, n, key_type):
    k = keys64("det_duplicates", n, seed=7, key_type=key_type)
    v = np.arange(n, dtype=np.uint32)
    tk, tv = to_dev(k, dev), to_dev(v.view(np.int32), dev)
    gbs.sort_pairs64(tk, tv)
    torch.cuda.synchronize()
    ek, ev = oracle.sort64(k, v, key_type)
    assert np.array_equal(tk.cpu().numpy().view(np.uint64), ek.view(np.uint64))
    assert np.array_equal(tv.cpu().numpy().view(np.uint32), ev)


@pytest.mark.parametrize("n", [(1 << 20) + 5, 1 << 24])
@pytest.mark.parametrize("key_type", ["uint64", "int64"])
def test_keys64_large_vs_library(dev, n, key_type):
    k = keys64("uniform", n, seed=11, key_type=key_type)
    k[::5] = k[0]
    v = np.arange(n, dtype=np.uint32)
    tk, tv = to_dev(k, dev), to_dev(v.view(np.int32), dev)
    gbs.sort_pairs64(tk, tv)
    torch.cuda.synchronize()
    order = np.argsort(k, kind="stable")
    assert np.array_equal(tk.cpu().numpy(), k[order])
    assert np.array_equal(tv.cpu().numpy().view(np.uint32), order.astype(np.uint32))


def test_keys64_float_large(dev):
    n = (1 << 20) + 5
    f = keys64("gaussian", n, seed=13, key_type="float64")
    f[np.isnan(f)] = 2.5
    f[f == 0] = 0.0                                   # one zero sign: numpy value order == totalOrder
    t = to_dev(f, dev)
    gbs.sort_keys64(t)
    torch.cuda.synchronize()
    assert np.array_equal(t.cpu().numpy(), np.sort(f))


def test_keys64_rejects_bad_args(dev):
    t = torch.zeros(9, dtype=torch.int64, device=dev)
    with pytest.raises(gbs.GbsError):
        gbs.sort_keys64(t, key_type="int32")
    with pytest.raises(gbs.GbsError):
        gbs.sort_pairs64(t, torch.zeros(8, dtype=torch.int32, device=dev))
