"""The paper's experiments on one B200, through the C-ABI:

  Fig. 3 analogue: device time and keys/s vs n, uniform u32 keys, default plan.
  Fig. 4 analogue: per-step time at n = 2^25 (the library's step events).
  Fig. 5 analogue: device time vs the sample count s at n = 2^25 and 2^26 with
      one-tile sublists (L = 2^15); small s gives buckets above one tile, i.e. a nested
      Step 9 (the plan reports it).
  Pairs: the Fig. 3 analogue for stable (u32 key, u32 value) pairs, the headline's item
      type (C4 = 2^30), checked against a stable library sort.

Timing: input restored from a pristine copy outside the CUDA-event window, 3 warm-ups,
median of `--reps` sorts.  Every sorted output is checked against torch.sort.

usage: python scripts/experiments.py [--reps 10] [--out profiles/r02/experiments]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gbs_inputs as gi  # noqa: E402
import paper_1002_4464_b200 as gbs  # noqa: E402


def time_sort(keys_np, cfg=None, reps=10, prof=False):
    dev = torch.device("cuda:0")
    n = keys_np.size
    pristine = torch.from_numpy(keys_np.view(np.int32)).to(dev)
    d = torch.empty_like(pristine)
    ws = gbs.Workspace(dev)
    st = torch.cuda.current_stream()
    times = []
    if prof:
        gbs.profile_begin()
    for r in range(3 + reps):
        d.copy_(pristine)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        if cfg is None:
            gbs.sort_keys(d, ws=ws)
        else:
            gbs.sort_ex(d, cfg=cfg, ws=ws)
        e1.record(st)
        torch.cuda.synchronize()
        if r >= 3:
            times.append(e0.elapsed_time(e1))
    steps = gbs.profile_end() if prof else None
    exp = torch.sort(pristine.view(torch.uint32).to(torch.int64))[0]
    ok = bool(torch.equal(d.view(torch.uint32).to(torch.int64), exp))
    ms = float(np.median(times))
    out = {"n": n, "ms": round(ms, 4), "ms_min": round(min(times), 4), "ms_max": round(max(times), 4),
           "gkeys_per_s": round(n / ms / 1e6, 3), "sorted_ok": ok,
           "plan": gbs.plan(n, cfg=cfg)["levels"]}
    if steps:
        calls = steps.pop("calls")
        steps.pop("level", None)
        out["steps_ms"] = {k: round(v / calls, 4) for k, v in steps.items()}
    return out


def time_sort_pairs(keys_np, reps=10):
    dev = torch.device("cuda:0")
    n = keys_np.size
    pristine = torch.from_numpy(keys_np.view(np.int32)).to(dev)
    pv = torch.arange(n, dtype=torch.int32, device=dev)
    d, dv = torch.empty_like(pristine), torch.empty_like(pv)
    ws = gbs.Workspace(dev)
    st = torch.cuda.current_stream()
    times = []
    for r in range(3 + reps):
        d.copy_(pristine)
        dv.copy_(pv)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        gbs.sort_pairs(d, dv, ws=ws)
        e1.record(st)
        torch.cuda.synchronize()
        if r >= 3:
            times.append(e0.elapsed_time(e1))
    k64 = pristine.view(torch.uint32).to(torch.int64)
    exp_k, exp_i = torch.sort(k64, stable=True)
    ok = bool(torch.equal(d.view(torch.uint32).to(torch.int64), exp_k)) and bool(torch.equal(dv.to(torch.int64), exp_i))
    del k64, exp_k, exp_i
    ms = float(np.median(times))
    return {"n": n, "ms": round(ms, 4), "ms_min": round(min(times), 4), "ms_max": round(max(times), 4),
            "gpairs_per_s": round(n / ms / 1e6, 3), "sorted_ok": ok, "plan": gbs.plan(n, pairs=True)["levels"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "experiments"))
    args = ap.parse_args()
    res = {"device": torch.cuda.get_device_name(0), "fig3_n_scaling": [], "fig5_s_sweep": []}
    for lg in (16, 18, 20, 22, 24, 25, 26, 27, 28, 29, 30):   # (2^31: bench.py c5_base)
        n = 1 << lg
        r = time_sort(gi.generate("uniform", n, seed=0), reps=args.reps)
        res["fig3_n_scaling"].append(r)
        print("n-scaling", r, flush=True)
    res["pairs_n_scaling"] = []
    for lg in (16, 20, 22, 24, 25, 26, 27, 28, 29, 30):
        r = time_sort_pairs(gi.generate("uniform", 1 << lg, seed=0), reps=args.reps)
        res["pairs_n_scaling"].append(r)
        print("pairs n-scaling", r, flush=True)
    res["fig4_steps_c2"] = time_sort(gi.generate("uniform", 1 << 25, seed=0), reps=args.reps, prof=True)
    print("steps", res["fig4_steps_c2"], flush=True)
    for lg in (25, 26):
        keys = gi.generate("uniform", 1 << lg, seed=0)
        for s in (256, 512, 1024, 2048, 4096):
            r = time_sort(keys, cfg=(1 << 15, s), reps=args.reps)
            r["s"] = s
            res["fig5_s_sweep"].append(r)
            print("s-sweep", r, flush=True)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    with open(args.out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    lines = [f"# Experiments on {res['device']} (scripts/experiments.py, median of {args.reps})", "",
             "## Fig. 3 analogue: keys/s vs n (uniform u32, default plan)", "",
             "| n | ms | Gkeys/s | plan (L, s) per level | sorted |", "|---|---|---|---|---|"]
    for r in res["fig3_n_scaling"]:
        lines.append(f"| 2^{int(np.log2(r['n']))} | {r['ms']} | {r['gkeys_per_s']} | {r['plan']} | {r['sorted_ok']} |")
    lines += ["", "## Pairs: Gpairs/s vs n (uniform u32 keys, values = index, stable)", "",
              "| n | ms | Gpairs/s | plan (L, s) per level | sorted |", "|---|---|---|---|---|"]
    for r in res["pairs_n_scaling"]:
        lines.append(f"| 2^{int(np.log2(r['n']))} | {r['ms']} | {r['gpairs_per_s']} | {r['plan']} | {r['sorted_ok']} |")
    lines += ["", "## Fig. 4 analogue: per-step ms at n = 2^25", "",
              "| step | ms |", "|---|---|"]
    for k, v in res["fig4_steps_c2"]["steps_ms"].items():
        lines.append(f"| {k} | {v} |")
    lines += ["", "## Fig. 5 analogue: ms vs s (L = 2^15)", "",
              "| n | s | ms | Gkeys/s | plan | sorted |", "|---|---|---|---|---|---|"]
    for r in res["fig5_s_sweep"]:
        lines.append(f"| 2^{int(np.log2(r['n']))} | {r['s']} | {r['ms']} | {r['gkeys_per_s']} | {r['plan']} | {r['sorted_ok']} |")
    with open(args.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
