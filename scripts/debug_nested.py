import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gbs_inputs as gi, paper_1002_4464_b200 as gbs
n = int(sys.argv[1]); L = int(sys.argv[2]); s = int(sys.argv[3])
dev = torch.device("cuda:0")
k = gi.generate_torch("uniform", n, seed=0, device=dev)
ref = np.sort(k.cpu().numpy().view(np.uint32))
print(gbs.plan(n, cfg=(L, s)), flush=True)
try:
    gbs.sort_ex(k, None, cfg=(L, s))
    torch.cuda.synchronize()
    print("ok equal:", np.array_equal(k.cpu().numpy().view(np.uint32), ref))
except Exception as e:
    print("ERROR", e)
