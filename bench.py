#!/usr/bin/env python
"""Benchmark: GPU Bucket Sort (arXiv 1002.4464) on B200 -- sorted keys/s, device-timed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2|C3|C1]
                    [--dist uniform] [--impl gbs|reference]

One step = one complete sort (all nine steps of Alg. 1) of one batch of
synthetic keys already resident in HBM.  N = 1: the workload BASELINE.json's metric is
quoted on (configs[1], C2: n = 2^25 uniform u32 keys).  N > 1 (torchrun, one rank per
GPU, NCCL): every rank holds an n-key shard and the ranks run the multi-GPU sort
(sample allgather + bucket exchange) -- weak scaling, value = all keys
sorted / max-over-ranks device time.

Between timed steps the input is restored from a pristine copy and L2 is flushed
(a 256 MiB device memset), both outside the per-step CUDA-event window.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "C1": (1 << 16, "C1: n=2^16 uniform u32 keys"),
    "C2": (1 << 25, "C2: n=2^25 (32M) uniform u32 keys (configs[1]; the paper's largest GTX 285 size)"),
    "C3": (1 << 26, "C3: n=2^26 (64M) u32 keys"),
    "C4": (1 << 30, "C4: n=2^30 u32->u32 key-value pairs (stable; nested Step 9)"),
}
METRIC = "sorted keys/sec (device-timed)"
L2_FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C2", choices=sorted(WORKLOADS))
    ap.add_argument("--dist", default="uniform")
    ap.add_argument("--impl", default="gbs", choices=["gbs", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (profiling runs only)")
    ap.add_argument("--n", type=int, default=0, help="override the workload's size (experiments; not a bench line)")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the multi-GPU entry even with one rank (exercises E1-E9 on one GPU)")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks (NVML)

class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.nv = None
            self.err = str(e)
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        names = {getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
                 getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
                 getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
                 getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap"}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": self.err}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------- helpers

def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, b.copy_(a) read+write)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def traffic_from_profile(step_kernel: str):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d["kernels"][step_kernel]["dram_bytes_per_launch"]
    except Exception:  # noqa: BLE001
        return None


def limiter_from_profile(step_kernel: str):
    """What bounds the dominant kernel, from the committed ncu --set full summary: issue
    slots, ALU pipe, shared-memory wavefronts (percent of peak) and the top stall."""
    path = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    try:
        with open(path) as f:
            k = json.load(f)["kernels"][step_kernel]
        return {"issue_active_pct": round(k["smsp__issue_active.avg.pct_of_peak_sustained_active"], 1),
                "alu_pipe_pct": round(k["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"], 1),
                "smem_wavefronts_pct": round(
                    k["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"], 1),
                "top_stall": k["top_stalls"][0][0], "source": "profiles/ncu_full_summary.json (ncu --set full)"}
    except Exception:  # noqa: BLE001
        return None


def algorithmic_bytes(n: int, plan: dict, ib: int = 4):
    """Bytes each level-1 step must move; ib = 4 keys, 8 pairs."""
    L, s = plan["levels"][0]
    m = plan["m"][0]
    ms = m * s
    nested = len(plan["levels"]) > 1
    return {
        2: 2 * ib * n + 8 * ms,     # Steps 2-3: read + write every item, write the samples
        4: None,                    # Step 4: recursive sample sort (reported as time only)
        5: 16 * s,                  # Step 5: gather s splitters
        6: 4 * n + 8 * s * m + 4 * ms,  # Step 6: key reload, splitters per CTA, counts
        7: 12 * ms,                 # Step 7: read a twice, write l
        8: 2 * ib * n + 8 * ms,     # Step 8: read + write every item, a and l rows
        9: None if nested else 2 * ib * n + 4 * s,   # Step 9: read + write every item
    }


STEP_NAMES = {2: "k_local_sort (Steps 2-3)", 4: "Step 4 (sample sort: merge tree or u64 level)", 5: "k_global_samples (Step 5)",
              6: "k_sample_index (Step 6)", 7: "k_scan (Step 7)", 8: "k_relocate (Step 8)",
              9: "k_segment_sort (Step 9)"}


# ----------------------------------------------------------------- reference arm (the oracle)

def run_reference(args):
    import numpy as np
    import gbs_inputs as gi
    import oracle
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from plans import plan as plan_rule
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_full, wl = WORKLOADS[args.workload]
    n = min(n_full, 1 << 22)                        # bounded sample: ~1.5 s of CPU per step
    keys = gi.generate(args.dist, n, seed=0)
    pl = plan_rule(n)
    for _ in range(args.warmup):
        oracle.gbs_sort(keys, plan=pl)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        out, _, _ = oracle.gbs_sort(keys, plan=pl)
        ts.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.mean(ts)
    v = n / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "keys/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": wl, "n": n_full, "dist": args.dist},
            "cpu_baseline": {"value": v, "unit": "keys/s", "cores": 1, "kind": "oracle",
                             "sample": f"{n} keys of the {args.workload} workload per step "
                                       f"(oracle plan {pl}), single-threaded C"},
            "e2e": {"value": v, "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ----------------------------------------------------------------- GPU arm

def cpu_baseline_line(args, n):
    """The oracle as it stands, single-threaded, once on a bounded sample of the workload
    (the full C2 workload, ~10-15 s; C3/C4 are sampled at 2^25 items)."""
    import numpy as np
    import gbs_inputs as gi
    import oracle
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from plans import TILE_KEYS, TILE_PAIRS, plan as plan_rule
    pairs = args.workload == "C4"
    ns = min(n, 1 << 25)
    keys = gi.generate(args.dist, ns, seed=0)
    vals = gi.pair_values(ns) if pairs else None
    t0 = time.perf_counter()
    oracle.gbs_sort(keys, vals, plan=plan_rule(ns, TILE_PAIRS if pairs else TILE_KEYS))
    dt = time.perf_counter() - t0
    what = "full" if ns == n else f"2^{ns.bit_length() - 1}-item sample of the"
    return {"value": ns / dt, "unit": "keys/s", "cores": 1, "kind": "oracle",
            "sample": f"one {what} {args.workload} sort ({ns} {'pairs' if pairs else 'keys'}, {args.dist}) "
                      f"by the single-threaded C oracle, {dt:.1f} s"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import gbs_inputs as gi
    import paper_1002_4464_b200 as gbs
    from paper_1002_4464_b200 import _build

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    use_dist = world > 1 or args.force_dist
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    if rank == 0:
        _build.build()
    if use_dist:
        dist.barrier()

    n, wl = WORKLOADS[args.workload]
    if args.n:
        n, wl = args.n, f"{args.workload} shape at n={args.n} (size override)"
    stream = torch.cuda.current_stream()
    # rank r holds global elements [r n, (r+1) n) of an N = world*n array
    if args.dist == "sorted":
        pristine = gi.generate_torch("sorted", n * world, seed=0, device=dev)[n * rank:n * (rank + 1)].clone()
    else:
        pristine = gi.generate_torch(args.dist, n * world, seed=0, device=dev, start=n * rank, count=n)
    pairs = args.workload == "C4"
    if pairs and use_dist:
        raise SystemExit("the multi-GPU entry sorts keys (DESIGN.md 7); C4 is a single-GPU workload")
    keys = torch.empty_like(pristine)
    vals = torch.empty_like(pristine) if pairs else None
    pristine_v = torch.arange(n, dtype=torch.int32, device=dev) if pairs else None
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    ws = gbs.Workspace(dev)
    comm = gbs.Comm() if use_dist else None
    out = None
    if comm is not None:
        _, cap = gbs.dist_workspace_size(n, world)
        out = torch.empty(cap, dtype=torch.int32, device=dev)
    plan = gbs.plan(n, pairs=pairs)

    def restore():
        keys.copy_(pristine)
        if pairs:
            vals.copy_(pristine_v)

    def one_sort():
        if pairs:
            gbs.sort_pairs(keys, vals, ws=ws)
        elif comm is None:
            gbs.sort_keys(keys, ws=ws)
        else:
            gbs.sort_keys_dist(keys, comm, out=out, ws=ws)

    for _ in range(args.warmup):
        restore()
        one_sort()
    torch.cuda.synchronize()
    # correctness of the timed configuration (single GPU): compare with the plain definition
    if comm is None:
        restore()
        one_sort()
        if pairs:   # stable: keys_out == keys_in[vals_out], nondecreasing, ties by position
            k64 = keys.to(torch.int64) & 0xFFFFFFFF
            assert torch.equal(pristine[vals.long()], keys), "pairs mismatch"
            assert bool((k64[1:] >= k64[:-1]).all()), "pairs not sorted"
            eq = k64[1:] == k64[:-1]
            assert bool((vals[1:][eq] > vals[:-1][eq]).all()), "pairs not stable"
            del k64, eq
        else:
            ref = torch.sort(pristine.to(torch.int64) & 0xFFFFFFFF).values
            assert torch.equal(keys.to(torch.int64) & 0xFFFFFFFF, ref), "sort mismatch"
            del ref
    else:   # multi-GPU: every rank's part sorted, parts ordered across ranks, nothing lost
        restore()
        part = gbs.sort_keys_dist(keys, comm, out=out, ws=ws)
        p64 = part.to(torch.int64) & 0xFFFFFFFF
        ok = bool((p64[1:] >= p64[:-1]).all()) if part.numel() > 1 else True
        info = torch.tensor([part.numel(), int(p64[0]) if part.numel() else -1,
                             int(p64[-1]) if part.numel() else -1, int(ok)], dtype=torch.int64, device=dev)
        allinfo = [torch.empty_like(info) for _ in range(world)]
        dist.all_gather(allinfo, info)
        rows = [t.tolist() for t in allinfo]
        assert sum(r[0] for r in rows) == n * world, "multi-GPU sort lost keys"
        assert all(r[3] for r in rows), "a rank's part is not sorted"
        ends = [(r[1], r[2]) for r in rows if r[0] > 0]
        assert all(ends[k][1] <= ends[k + 1][0] for k in range(len(ends) - 1)), "parts out of order"
        del p64

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            restore()
            flush.zero_()                                   # L2 flush (256 MiB > 126 MB L2)
            starts[i].record(stream)
            one_sort()
            ends[i].record(stream)
        torch.cuda.synchronize()
    # Per-step kernel times (roofline, breakdown): a second timed pass of the same steps
    # with the library's per-step CUDA events on the call's stream.  Kept out of the
    # headline pass: an event between two kernels stops the programmatic dependent
    # launch at that boundary (~1-2 % per step).
    prof = None
    if comm is None:
        gbs.profile_begin()
        for i in range(min(args.steps, 10)):
            restore()
            flush.zero_()
            one_sort()
        torch.cuda.synchronize()
        prof = gbs.profile_end()
    if use_dist:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms = statistics.mean(step_ms)
    if use_dist:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_keys = n * world
    value = total_keys / (ms / 1e3)

    # ---- end to end through the C-ABI with host buffers (N = 1)
    e2e = None
    if comm is None and not pairs and not args.no_e2e:
        host = pristine.cpu().pin_memory()
        hbuf = torch.empty_like(host).pin_memory()
        dbuf = torch.empty_like(keys)
        for _ in range(2):
            hbuf.copy_(host)
            gbs.sort_keys_host(hbuf, dbuf, ws=ws)
        torch.cuda.synchronize()
        e_ms = []
        for i in range(max(3, args.steps // 2)):
            hbuf.copy_(host)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            gbs.sort_keys_host(hbuf, dbuf, ws=ws)
            b.record(stream)
            b.synchronize()
            e_ms.append(a.elapsed_time(b))
        em = statistics.mean(e_ms)
        e2e = {"value": n / (em / 1e3), "unit": "keys/s", "h2d_bytes_per_step": 4 * n,
               "d2h_bytes_per_step": 4 * n, "ms_per_step": em}
    elif comm is not None:
        # end to end per rank: pinned host shard -> device, multi-GPU sort, the rank's
        # part back to pinned host; max over ranks
        host = pristine.cpu().pin_memory()
        hout = torch.empty(out.numel(), dtype=torch.int32).pin_memory()
        e_ms, moved = [], 0
        for i in range(max(3, args.steps // 2) + 1):
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            keys.copy_(host, non_blocking=True)
            part = gbs.sort_keys_dist(keys, comm, out=out, ws=ws)
            hout[:part.numel()].copy_(part, non_blocking=True)
            b.record(stream)
            b.synchronize()
            if i:                                            # first iteration = warm-up
                e_ms.append(a.elapsed_time(b))
            moved = part.numel()
        t = torch.tensor([statistics.mean(e_ms), moved], dtype=torch.float64, device=dev)
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        em = float(tmax[0].item())
        e2e = {"value": n * world / (em / 1e3), "unit": "keys/s", "h2d_bytes_per_step": 4 * n * world,
               "d2h_bytes_per_step": 4 * n * world, "ms_per_step": em}

    if rank != 0:
        if use_dist:
            dist.destroy_process_group()
        return

    # our kernels per step: the plan's launches; multi-GPU adds E2 + E5/E6 + the E4
    # single-tile sample sort and the E9 re-sort of the received runs (~ n keys)
    launches_per_step = plan["kernels_per_sort"]
    if comm is not None:
        launches_per_step += 3 + gbs.plan(n)["kernels_per_sort"]
    peak, peak_src = peaks()
    roof = None
    steps = None
    if prof is not None and prof["calls"]:
        calls = prof["calls"]
        ab = algorithmic_bytes(n, plan, 8 if pairs else 4)
        steps = {}
        for k in (2, 4, 5, 6, 7, 8, 9):
            t_ms = prof[k] / calls
            gbps = (ab[k] / (t_ms / 1e3) / 1e9) if ab[k] and t_ms > 0 else None
            steps[STEP_NAMES[k]] = {"ms": round(t_ms, 4), "share": round(prof[k] / sum(prof[j] for j in (2, 4, 5, 6, 7, 8, 9)), 3),
                                    "alg_bytes": ab[k], "alg_GBps": round(gbps, 1) if gbps else None}
        dom = max((k for k in (2, 9, 8, 6) if ab[k]), key=lambda k: prof[k])
        t_ms = prof[dom] / calls
        ach = ab[dom] / (t_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": STEP_NAMES[dom], "achieved": round(ach, 1), "peak": peak,
                "unit": "GB/s", "frac": round(ach / peak, 4), "peak_source": peak_src,
                "traffic": traffic_from_profile(STEP_NAMES[dom].split()[0]),
                "alg_bytes_per_launch": ab[dom], "launch_ms": round(t_ms, 4),
                "limiter": limiter_from_profile(STEP_NAMES[dom].split()[0])}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line(args, n)

    line = {"metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32 pairs" if pairs else "u32", "data": "synthetic",
            "config": {"workload": wl, "n_per_gpu": n, "dist": args.dist,
                       "plan": plan["levels"], "bucket_bound": plan["bucket_bound"],
                       "l2": "flushed between steps (256 MiB memset) outside the event window",
                       "parallelism": f"dp{world}" if world > 1 else "single"},
            "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(), "roofline": roof, "cpu_baseline": cpu, "steps_breakdown": steps,
            "step_ms_min_max": [min(step_ms), max(step_ms)]}
    print(json.dumps(line))
    if use_dist:
        comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
