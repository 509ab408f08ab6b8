"""GPU (-m gpu): a sort is a fixed, host-sync-free launch sequence (static plan),
so it can be captured into a CUDA graph and replayed on new data -- including plans whose
Step 9 size tiers fork onto side streams and join back (fork/join events) and nested
levels.  Each replay is compared with the plain definition."""
import numpy as np
import pytest

import gbs_inputs as gi

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


@pytest.mark.parametrize("n,pairs", [(1 << 16, False), (1 << 25, False), (1 << 26, False), (1 << 28, False),
                                     ((1 << 20) + 5, True)])
def test_graph_capture_and_replay(dev, n, pairs):
    keys = torch.empty(n, dtype=torch.int32, device=dev)
    vals = torch.empty(n, dtype=torch.int32, device=dev) if pairs else None
    ws = gbs.Workspace(dev)
    ws.get(gbs.workspace_size(n, pairs=pairs), dev)
    s = torch.cuda.Stream(dev)
    # warm-up outside the capture (one-time kernel attribute setup, side streams)
    keys.copy_(gi.generate_torch("uniform", n, seed=1, device=dev))
    s.wait_stream(torch.cuda.current_stream(dev))   # the input is written on the current stream
    with torch.cuda.stream(s):
        if pairs:
            vals.copy_(torch.arange(n, dtype=torch.int32, device=dev))
            gbs.sort_pairs(keys, vals, ws=ws, stream=s)
        else:
            gbs.sort_keys(keys, ws=ws, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        if pairs:
            gbs.sort_pairs(keys, vals, ws=ws, stream=s)
        else:
            gbs.sort_keys(keys, ws=ws, stream=s)
    for seed, dist in ((2, "gaussian"), (3, "staggered")):
        src = gi.generate_torch(dist, n, seed=seed, device=dev)
        keys.copy_(src)
        if pairs:
            vals.copy_(torch.arange(n, dtype=torch.int32, device=dev))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        if pairs:
            order = np.argsort(src.cpu().numpy().view(np.uint32), kind="stable")
            assert np.array_equal(vals.cpu().numpy(), order.astype(np.int32))
        else:
            ref = torch.sort(src.to(torch.int64) & 0xFFFFFFFF).values
            assert torch.equal(keys.to(torch.int64) & 0xFFFFFFFF, ref)


@pytest.mark.parametrize("n,pairs", [(1000, False), (1 << 16, False), (1 << 20, False), ((1 << 16) + 3, True),
                                     (1 << 20, True)])
def test_graph_cache_replay(dev, n, pairs):
    """Latency-bound sizes (<= 2^20 items): the first call on given buffers runs directly
    and records its launch sequence into a cached graph; later calls on the same buffers
    replay it.  Every call, on new data, equals the plain (stable) sort."""
    keys = torch.empty(n, dtype=torch.int32, device=dev)
    vals = torch.empty(n, dtype=torch.int32, device=dev) if pairs else None
    ws = gbs.Workspace(dev)
    ws.get(gbs.workspace_size(n, pairs=pairs), dev)
    for seed, dist in enumerate(("uniform", "zero", "gaussian", "staggered", "det_duplicates")):
        src = gi.generate_torch(dist, n, seed=seed, device=dev)
        keys.copy_(src)
        if pairs:
            vals.copy_(torch.arange(n, dtype=torch.int32, device=dev))
            gbs.sort_pairs(keys, vals, ws=ws)
        else:
            gbs.sort_keys(keys, ws=ws)
        torch.cuda.synchronize()
        if pairs:
            order = np.argsort(src.cpu().numpy().view(np.uint32), kind="stable")
            assert np.array_equal(vals.cpu().numpy(), order.astype(np.int32))
        else:
            ref = torch.sort(src.to(torch.int64) & 0xFFFFFFFF).values
            assert torch.equal(keys.to(torch.int64) & 0xFFFFFFFF, ref)
