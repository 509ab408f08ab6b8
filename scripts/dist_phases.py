"""Phase times of the multi-GPU kernels in the single-GPU emulation (all ranks' phases run
one after another on one GPU; the E8 push is local copies here, so only E1, E2-E7 and E9 are
representative): keys/s of the one-pass k-way merge (E9) and of the other phases.

usage: python scripts/dist_phases.py [p] [log2 n_local]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gbs_inputs as gi  # noqa: E402
import paper_1002_4464_b200 as gbs  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 26)
dev = torch.device("cuda:0")
keys = gi.generate_torch("uniform", p * n, seed=0, device=dev)
gbs.sort_keys_dist_emulated(keys, p)
torch.cuda.synchronize()
gbs.profile_begin()
reps = 3
for _ in range(reps):
    gbs.sort_keys_dist_emulated(keys, p)
torch.cuda.synchronize()
ph = gbs.dist_profile_end()
tot = p * n
out = {"p": p, "n_local": n, "path": ph["path"], "per_call_ms": {k: v for k, v in ph.items() if k.endswith("_ms")}}
out["E9_merge_Gkeys_s"] = tot / (ph["merge_ms"] / 1e3) / 1e9
out["E1_local_sort_Gkeys_s"] = tot / (ph["local_sort_ms"] / 1e3) / 1e9
out["E9_alg_GBps"] = 8 * tot / (ph["merge_ms"] / 1e3) / 1e9
print(json.dumps(out, indent=1))
