"""One rank of the multi-process peer-memory test (tests/test_gpu_dist_ipc.py): every rank
runs on cuda:0, the group is gloo, the libgbs communicator is host-bootstrapped, so the
real multi-process path runs -- IPC-mapped windows, cross-process device barriers, pushes
into the peers' receive buffers, the k-way merge.

usage: python tests/dist_ipc_worker.py RANK WORLD PORT N_LOCAL DIST OUTDIR"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import gbs_inputs as gi  # noqa: E402
import paper_1002_4464_b200 as gbs  # noqa: E402


def main():
    rank, world, port, n_local = (int(a) for a in sys.argv[1:5])
    dist_name, outdir = sys.argv[5], sys.argv[6]
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    comm = gbs.Comm(bootstrap="host")
    keys = gi.generate(dist_name, world * n_local, seed=world)
    shard = torch.from_numpy(keys[rank * n_local:(rank + 1) * n_local].view(np.int32).copy()).to("cuda:0")
    parts = []
    for _ in range(2):                      # the second call reuses the mapped windows
        part = gbs.sort_keys_dist(shard, comm)
        torch.cuda.synchronize()
        parts.append(part.cpu().numpy().view(np.uint32).copy())
    assert np.array_equal(parts[0], parts[1])
    assert np.array_equal(shard.cpu().numpy().view(np.uint32), keys[rank * n_local:(rank + 1) * n_local])
    np.save(os.path.join(outdir, f"part{rank}.npy"), parts[0])
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
