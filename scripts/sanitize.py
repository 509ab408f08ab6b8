"""compute-sanitizer driver: runs the library's code paths at small sizes, each
result checked against the plain definition, so a memcheck / racecheck / synccheck run
covers them.  Prints one line per case; exits non-zero on a wrong result.

    compute-sanitizer --tool racecheck python scripts/sanitize.py [--big] [case ...]

Paths covered: the 2K-tile plan (2^16), the one-tile CTA sort with fused Step 8+9 (2^20),
CTA-pair sublists (explicit (65536, 4096) plan), Step 9 size tiers (3*2^20+7), a nested
Step 9 (explicit (2048, 8) plan), stable pairs (with their fused Step 8+9), typed float
keys, 64-bit keys, the host-buffer pipeline, the multi-GPU kernels (P2P transport and the
k-way merge, emulated p = 4), and with --big the CTA-pair buckets (10^8 keys)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gbs_inputs as gi  # noqa: E402
import paper_1002_4464_b200 as gbs  # noqa: E402

dev = torch.device("cuda:0")


def keys_case(n, dist="uniform", cfg=None):
    k = gi.generate_torch(dist, n, seed=1, device=dev)
    ref = torch.sort(k.to(torch.int64) & 0xFFFFFFFF).values
    if cfg:
        gbs.sort_ex(k, None, cfg=cfg)
    else:
        gbs.sort_keys(k)
    torch.cuda.synchronize()
    return torch.equal(k.to(torch.int64) & 0xFFFFFFFF, ref)


def pairs_case(n):
    k = gi.generate_torch("det_duplicates", n, seed=2, device=dev)
    v = torch.arange(n, dtype=torch.int32, device=dev)
    kin = k.clone()
    gbs.sort_pairs(k, v)
    torch.cuda.synchronize()
    order = np.argsort(kin.cpu().numpy().view(np.uint32), kind="stable")
    return bool(np.array_equal(v.cpu().numpy(), order.astype(np.int32)))


def float_case(n):
    f = torch.randn(n, generator=torch.Generator().manual_seed(3)).to(dev)
    ref = torch.sort(f).values
    gbs.sort_keys_typed(f)
    torch.cuda.synchronize()
    return torch.equal(f, ref)


def k64_case(n):
    x = torch.randint(-2**62, 2**62, (n,), generator=torch.Generator().manual_seed(4), dtype=torch.int64).to(dev)
    ref = torch.sort(x).values
    gbs.sort_keys64(x)
    torch.cuda.synchronize()
    return torch.equal(x, ref)


def host_case(n):
    keys = gi.generate("staggered", n, seed=5)
    h = torch.from_numpy(keys.view(np.int32).copy()).pin_memory()
    d = torch.empty(n, dtype=torch.int32, device=dev)
    gbs.sort_keys_host(h, d)
    torch.cuda.synchronize()
    return bool(np.array_equal(h.numpy().view(np.uint32), np.sort(keys)))


def dist_case(p, n_local):
    keys = gi.generate("uniform", p * n_local, seed=6)
    shards = torch.from_numpy(keys.view(np.int32).copy()).to(dev)
    parts = gbs.sort_keys_dist_emulated(shards, p)
    torch.cuda.synchronize()
    got = np.concatenate([t.cpu().numpy().view(np.uint32) for t in parts])
    return bool(np.array_equal(got, np.sort(keys)))


CASES = {
    "small_2k_plan": lambda: keys_case(1 << 16),
    "one_tile_fused_8_9": lambda: keys_case(1 << 20),
    "cta_pair_sublists": lambda: keys_case(1 << 20, "gaussian", cfg=(65536, 4096)),
    "step9_tiers": lambda: keys_case(3 * (1 << 20) + 7, "staggered"),
    "nested_step9": lambda: keys_case(1 << 18, "det_duplicates", cfg=(2048, 8)),
    "pairs": lambda: pairs_case((1 << 18) + 3),
    "typed_float": lambda: float_case(1 << 18),
    "keys64": lambda: k64_case(1 << 16),
    "host_pipeline": lambda: host_case(1 << 21),
    "multi_gpu_emulated_p4": lambda: dist_case(4, 1 << 16),
}
BIG = {"cta_pair_buckets": lambda: keys_case(100_000_000, "uniform")}


def main():
    from paper_1002_4464_b200 import _build
    _build.build()
    sel = [a for a in sys.argv[1:] if not a.startswith("--")]
    cases = dict(CASES, **(BIG if "--big" in sys.argv else {}))
    bad = 0
    for name, fn in cases.items():
        if sel and name not in sel:
            continue
        ok = fn()
        print(f"{name}: {'ok' if ok else 'WRONG RESULT'}", flush=True)
        bad += not ok
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
