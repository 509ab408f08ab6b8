"""GPU (-m gpu): the multi-GPU entry with several real processes sharing one GPU.

Each rank is its own process on cuda:0 (tests/dist_ipc_worker.py); the communicator is
bootstrapped through the gloo group's allgather (NCCL refuses two ranks on one device), so
the exchange is the product's peer-memory path end to end: windows exported and opened with
CUDA IPC across processes, samples / fine cuts / buckets stored into the other processes'
windows, device barriers over system-scope flags.  The rank parts are compared bit for bit
with the oracle's PSRS and the receive counts with its counts."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import gbs_inputs as gi
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1002_4464_b200 import _build
    _build.build()
    return torch.device("cuda:0")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def s_r_of(n_local: int) -> int:
    s = 1
    while s < 1024 and n_local % (2 * s) == 0:
        s *= 2
    return s


@pytest.mark.parametrize("world,n_local,dist", [(2, 1 << 20, "uniform"), (3, (1 << 18) + 40, "det_duplicates"),
                                                (4, 1 << 19, "staggered")])
def test_multiprocess_peer_exchange(dev, tmp_path, world, n_local, dist):
    port = free_port()
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "dist_ipc_worker.py"), str(r), str(world),
                               str(port), str(n_local), dist, str(tmp_path)], cwd=ROOT,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(out)
    assert all(p.returncode == 0 for p in procs), "\n".join(outs)
    keys = gi.generate(dist, world * n_local, seed=world)
    exp, counts, _ = oracle.psrs(keys, world, s_r_of(n_local))
    parts = [np.load(os.path.join(tmp_path, f"part{r}.npy")) for r in range(world)]
    assert [p.size for p in parts] == [int(c) for c in counts]
    assert np.array_equal(np.concatenate(parts), exp)
