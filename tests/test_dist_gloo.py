"""Multi-GPU protocol (E1-E9) with world_size 2 on CPU over gloo (-m "not gpu").

The NCCL data path cannot run here (one GPU per run, none in the sandbox), so this test
drives the same protocol with torch.distributed/gloo collectives and numpy local steps,
using libgbs's host exchange plan (`gbs_exchange_plan`), and checks it against the oracle's
PSRS simulation (identical per-rank counts) and the plain definition (global sort)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def s_r_of(n_local, cap=1024):
    s = 1
    while s < cap and n_local % (2 * s) == 0:
        s *= 2
    return s


def _worker(rank, world, port, n_local, dist_name, q):
    import sys
    sys.path.insert(0, ROOT)
    import gbs_inputs as gi
    import paper_1002_4464_b200 as gbs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = gi.generate(dist_name, n_local * world, seed=5, start=rank * n_local, count=n_local)
        S = np.sort(shard)                                                        # E1
        s_r = s_r_of(n_local)
        d = n_local // s_r
        pos = (np.arange(s_r) + 1) * d - 1
        gpos = rank * n_local + np.arange(n_local, dtype=np.uint64)
        comp = (S.astype(np.uint64) << np.uint64(32)) | gpos                       # (key, global position)
        samples = torch.from_numpy(comp[pos].view(np.int64))                      # E2
        gathered = [torch.empty_like(samples) for _ in range(world)]
        dist.all_gather(gathered, samples)                                        # E3
        allS = np.sort(torch.cat(gathered).numpy().view(np.uint64))               # E4
        G = allS[(np.arange(world) + 1) * s_r - 1]                                # E5
        cuts = np.searchsorted(comp, G, side="right").astype(np.uint64)          # E6
        allc = [torch.empty(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allc, torch.from_numpy(cuts.view(np.int64)))              # E7
        C = torch.stack(allc).numpy().view(np.uint64)
        plan = gbs.exchange_plan(C, rank)                                         # host plan (libgbs)
        out = np.zeros(plan["n_out"], np.uint32)
        reqs = []
        for k in range(world):                                                    # E8
            so, sc = int(plan["send_off"][k]), int(plan["send_cnt"][k])
            ro, rc = int(plan["recv_off"][k]), int(plan["recv_cnt"][k])
            if k == rank:
                out[ro:ro + rc] = S[so:so + sc]
                continue
            if sc:
                reqs.append(dist.isend(torch.from_numpy(S[so:so + sc].view(np.int32).copy()), k))
            if rc:
                buf = torch.empty(rc, dtype=torch.int32)
                reqs.append((dist.irecv(buf, k), buf, ro, rc))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                out[r[2]:r[2] + r[3]] = r[1].numpy().view(np.uint32)
            else:
                r.wait()
        out = np.sort(out)                                                        # E9
        q.put((rank, out, plan["n_out"]))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dist_name", ["uniform", "zero", "det_duplicates"])
def test_protocol_world2_matches_oracle(dist_name):
    import gbs_inputs as gi
    import oracle
    from paper_1002_4464_b200 import _build
    _build.build()
    world, n_local = 2, 1 << 14
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_local, dist_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(world):
        r, out, n_out = q.get(timeout=120)
        res[r] = (out, n_out)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([res[r][0] for r in range(world)])
    full = gi.generate(dist_name, n_local * world, seed=5)
    assert np.array_equal(got, np.sort(full))
    s_r = s_r_of(n_local)
    _, counts, _ = oracle.psrs(full, world, s_r)
    assert [res[r][1] for r in range(world)] == [int(c) for c in counts]
    assert max(res[r][1] for r in range(world)) <= n_local + (world - 1) * (n_local // s_r - 1)
