import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gbs_inputs as gi, paper_1002_4464_b200 as gbs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 30
pairs = len(sys.argv) <= 2 or sys.argv[2] == "pairs"
dev = torch.device("cuda:0")
k = gi.generate_torch("uniform", n, seed=0, device=dev)
print(gbs.plan(n, pairs=pairs), flush=True)
try:
    if pairs:
        v = torch.arange(n, dtype=torch.int32, device=dev)
        gbs.sort_pairs(k, v)
    else:
        gbs.sort_keys(k)
    torch.cuda.synchronize()
    k64 = k.to(torch.int64) & 0xFFFFFFFF
    print("ok sorted:", bool((k64[1:] >= k64[:-1]).all()))
except Exception as e:
    print("ERROR", e)
