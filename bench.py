#!/usr/bin/env python
"""Benchmark: GPU Bucket Sort (arXiv 1002.4464) on B200 -- sorted keys/s, device-timed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C1..C5]
                    [--dist uniform] [--impl gbs|reference]

One step = one complete sort (all nine steps of Alg. 1) of one batch of
synthetic items already resident in HBM.

N = 1: the headline is C4 (configs[3]: 2^30 u32 -> u32 key-value pairs, stable), the
largest single-GPU config of BASELINE.json.  The same line carries, measured in the same
run: `c2` (configs[1], 2^25 uniform keys), `c3` (configs[2], 2^26 keys over the seven
distributions, each sort verified, with the spread (max - min)/mean the north star bounds
at 10 %), and `c5_base` (the C5 shape on one GPU at the largest single-call size, 2^31
keys: the N = 1 base point of the scaling runs).
N > 1 (torchrun, one rank per GPU): C5 (configs[4]): N = 2^32 uniform keys in total,
2^32/N per rank (strong scaling), sorted by the multi-GPU entry; verified by
a multiset fingerprint allreduced in vs out, per-rank order, rank-boundary order and the
receive bound; value = 2^32 / max-over-ranks device time.

Between timed steps the input is restored from a pristine copy and L2 is flushed (a
256 MiB device memset), both outside the per-step CUDA-event window.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "C1": dict(n=1 << 16, pairs=False, name="C1: n=2^16 uniform u32 keys (configs[0])"),
    "C2": dict(n=1 << 25, pairs=False,
               name="C2: n=2^25 (32M) uniform u32 keys (configs[1]; the paper's largest GTX 285 size)"),
    "C3": dict(n=1 << 26, pairs=False, name="C3: n=2^26 (64M) u32 keys (configs[2])"),
    "C4": dict(n=1 << 30, pairs=True,
               name="C4: n=2^30 u32->u32 key-value pairs, stable (configs[3]; the largest single-GPU config)"),
    "C5": dict(n=1 << 32, pairs=False,
               name="C5: N=2^32 uniform u32 keys sharded over the ranks (configs[4]); strong scaling"),
}
DISTS = ["uniform", "gaussian", "bucket_sorted", "staggered", "sorted", "zero", "det_duplicates"]
METRIC = "sorted keys/sec (device-timed)"
L2_FLUSH_BYTES = 256 << 20
C5_BASE_N = 1 << 31                 # largest single call (32-bit tags, R10)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: C4 on one GPU, C5 on several")
    ap.add_argument("--dist", default="uniform")
    ap.add_argument("--impl", default="gbs", choices=["gbs", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer leg (profiling runs only)")
    ap.add_argument("--no-extras", action="store_true", help="skip the c2/c3/c5_base legs (profiling runs only)")
    ap.add_argument("--size", type=int, default=0, help="override the workload's size (experiments; not a bench line)")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the multi-GPU entry even with one rank (exercises E1-E9 on one GPU)")
    ap.add_argument("--lib", default=None, help="tuning only: load this libgbs build instead of the in-tree one")
    ap.add_argument("--bootstrap", default="nccl", choices=["nccl", "host"],
                    help="testing only (C5): 'host' = gloo group + host-bootstrapped communicator, so several "
                         "ranks may share one GPU (exercises the multi-rank path on a one-GPU box)")
    ap.add_argument("--ncu-one", action="store_true",
                    help="profiling only: run exactly one sort of the workload (for ncu captures) and exit")
    a = ap.parse_args()
    if a.workload is None:
        a.workload = "C5" if (a.gpus > 1 or a.force_dist) else "C4"
    return a


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
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, b.copy_(a) read+write, burst)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_record(kernel_key: str):
    """The committed `ncu --set full` record of a kernel (profiles/ncu_full_summary.json):
    DRAM bytes per launch and what bounds it (issue slots, ALU pipe, shared-memory
    wavefronts, top stall)."""
    path = os.path.join(ROOT, "profiles", "ncu_full_summary.json")
    try:
        with open(path) as f:
            k = json.load(f)["kernels"][kernel_key]
    except Exception:  # noqa: BLE001
        return None, None
    lim = {"issue_active_pct": round(k["smsp__issue_active.avg.pct_of_peak_sustained_active"], 1),
           "alu_pipe_pct": round(k["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"], 1),
           "smem_wavefronts_pct": round(k["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"], 1),
           "top_stall": k["top_stalls"][0][0] if k.get("top_stalls") else None,
           "source": f"profiles/ncu_full_summary.json ({k.get('capture', 'ncu --set full')})"}
    return k.get("dram_bytes_one_launch"), lim


def s4_bytes(samples: int) -> int:
    """Step 4 of one problem: the merge tree (R22) reads and writes every 8-byte composite
    once in the tile merge and once per global merge level (L2-resident), or -- for a u64
    level -- ~56 B per composite."""
    tile = 16384
    if samples <= tile:
        return 16 * samples
    if samples <= (1 << 23):
        levels, r = 0, tile
        while 2 * r < samples:
            levels, r = levels + 1, 2 * r
        return 16 * samples * (1 + levels)
    return 56 * samples


def algorithmic_bytes(n: int, plan: dict, ib: int, level: int = 0):
    """Bytes each step of `level` must move; ib = 4 keys, 8 pairs.
    A nested level covers all n items at once (its problems are the buckets above)."""
    L, s = plan["levels"][level]
    m = plan["m"][level]
    probs = 1 if level == 0 else plan["levels"][level - 1][1]
    ms = m * s * probs
    nested = len(plan["levels"]) > level + 1
    return {
        2: 2 * ib * n + 8 * ms,            # Steps 2-3: read + write every item, write the samples
        4: s4_bytes(m * s) * probs,        # Step 4: sort the samples (per problem)
        5: 16 * s * probs,                 # Step 5: gather s splitters
        6: 4 * n + 8 * s * m * probs + 4 * ms,   # Step 6: key reload, splitters per CTA, counts
        7: 12 * ms,                        # Step 7: read a twice, write l
        8: 2 * ib * n + 8 * ms,            # Step 8: read + write every item, a and l rows
        9: None if nested else 2 * ib * n + 4 * s * probs,   # Step 9: read + write every item
    }


STEP_NAMES = {2: "Steps 2-3 local sort + samples", 4: "Step 4 sample sort", 5: "Step 5 global samples",
              6: "Step 6 sample indexing", 7: "Step 7 prefix sum", 8: "Step 8 relocation",
              9: "Step 9 bucket sort"}
STEP_KERNEL = {2: "k_local_sort", 6: "k_sample_index", 8: "k_relocate", 9: "k_segment_sort"}


def cpu_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count()


def pin_one_core():
    """Pin this process to one core (the single-threaded oracle's baseline)."""
    try:
        cores = sorted(os.sched_getaffinity(0))
        os.sched_setaffinity(0, {cores[0]})
        return cores[0]
    except (AttributeError, OSError):
        return None


def config_of(args, world: int) -> dict:
    """The workload's config dict -- identical for the GBS arm and the reference arm."""
    w = WORKLOADS[args.workload]
    n = args.size or w["n"]
    cfg = {"workload": w["name"] if not args.size else f"{args.workload} shape at n={args.size} (size override)",
           "n_total": n, "items": "u32 key -> u32 value pairs" if w["pairs"] else "u32 keys",
           "dist": args.dist, "parallelism": f"dp{world}" if world > 1 else "single",
           "l2": "inputs > L2 and flushed between steps (256 MiB memset) outside the event window"}
    if args.workload == "C5":
        cfg["n_per_rank"] = n // world
    return cfg


# ----------------------------------------------------------------- reference arm (the oracle)

def run_reference(args):
    """The reference is a paper (no code): this arm times the oracle (oracle/, plain
    single-threaded C) on the box's host cores, on the GBS arm's config, each step one
    bounded sample of the workload."""
    import gbs_inputs as gi
    import oracle
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from plans import TILE_KEYS, TILE_PAIRS, plan as plan_rule
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    core = pin_one_core()
    w = WORKLOADS[args.workload]
    n_full = args.size or w["n"]
    pairs = w["pairs"]
    n = min(n_full, 1 << 22)                        # bounded sample: ~1-2 s of CPU per step
    keys = gi.generate(args.dist, n, seed=0)
    vals = gi.pair_values(n) if pairs else None
    pl = plan_rule(n, TILE_PAIRS if pairs else TILE_KEYS)
    for _ in range(args.warmup):
        oracle.gbs_sort(keys, vals, plan=pl)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.gbs_sort(keys, vals, plan=pl)
        ts.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.mean(ts)
    v = n / (ms / 1e3)
    model, nproc = cpu_info()
    unit = "pairs/s" if pairs else "keys/s"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if args.workload == "C5" else "weak", "vs_baseline": None,
            "dtype": "u32 pairs" if pairs else "u32", "data": "synthetic",
            "config": config_of(args, world),
            "cpu_baseline": {"value": v, "unit": unit, "cores": 1, "kind": "oracle", "pinned_core": core,
                             "nproc": nproc, "cpu_model": model,
                             "sample": f"per step: the first {n} {'pairs' if pairs else 'keys'} of the "
                                       f"{args.workload} input ({args.dist}, seed 0), oracle plan {pl}, "
                                       f"single-threaded C pinned to one core"},
            "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def cpu_baseline_line(args, n: int, pairs: bool):
    """The oracle as it stands, single-threaded and pinned to one core, once on a bounded
    sample of the workload (2^25 items: ~10-15 s)."""
    import gbs_inputs as gi
    import oracle
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from plans import TILE_KEYS, TILE_PAIRS, plan as plan_rule
    ns = min(n, 1 << 25)
    keys = gi.generate(args.dist, ns, seed=0)
    vals = gi.pair_values(ns) if pairs else None
    saved = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    core = pin_one_core()
    try:
        t0 = time.perf_counter()
        oracle.gbs_sort(keys, vals, plan=plan_rule(ns, TILE_PAIRS if pairs else TILE_KEYS))
        dt = time.perf_counter() - t0
    finally:
        if saved:
            os.sched_setaffinity(0, saved)
    model, nproc = cpu_info()
    what = "full" if ns == n else f"2^{ns.bit_length() - 1}-item sample (the first items) of the"
    return {"value": ns / dt, "unit": "pairs/s" if pairs else "keys/s", "cores": 1, "kind": "oracle",
            "pinned_core": core, "nproc": nproc, "cpu_model": model,
            "sample": f"one {what} {args.workload} sort ({ns} {'pairs' if pairs else 'keys'}, {args.dist}) "
                      f"by the single-threaded C oracle, {dt:.1f} s"}


# ----------------------------------------------------------------- GPU arm

def timed_sorts(torch, one_sort, restore, flush, stream, steps, warmup, clk_index=None):
    """W untimed warm-ups, then K sorts each bracketed by CUDA events on `stream`, with
    the input restored and L2 flushed before each (outside the events)."""
    for _ in range(warmup):
        restore()
        one_sort()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    clk = ClockSampler(clk_index) if clk_index is not None else None
    if clk:
        clk.__enter__()
    for i in range(steps):
        restore()
        flush.zero_()
        starts[i].record(stream)
        one_sort()
        ends[i].record(stream)
    torch.cuda.synchronize()
    if clk:
        clk.__exit__()
    return [s.elapsed_time(e) for s, e in zip(starts, ends)], (clk.summary() if clk else None)


def breakdown(prof, plan, n, ib, peak):
    """Per-step ms, share and algorithmic GB/s of every level (from gbs_profile events)."""
    calls = prof["calls"]
    out, flat = {}, []
    for lev, times in enumerate(prof["level"]):
        ab = algorithmic_bytes(n, plan, ib, lev)
        tot = sum(times[k] for k in (2, 4, 5, 6, 7, 8, 9) if not (k == 9 and ab[9] is None))
        steps = {}
        for k in (2, 4, 5, 6, 7, 8, 9):
            t_ms = times[k] / calls
            if k == 9 and ab[9] is None:
                steps[STEP_NAMES[k]] = {"ms": round(t_ms, 4), "note": f"the nested level {lev + 1} (below)"}
                continue
            gbps = ab[k] / (t_ms / 1e3) / 1e9 if ab[k] and t_ms > 0 else None
            steps[STEP_NAMES[k]] = {"ms": round(t_ms, 4), "share_of_level": round(times[k] / tot, 3) if tot else None,
                                    "alg_bytes": ab[k], "alg_GBps": round(gbps, 1) if gbps else None,
                                    "frac": round(gbps / peak, 4) if gbps else None}
            flat.append((t_ms, lev, k, ab[k]))
        out[f"level{lev + 1}"] = steps
    return out, flat


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
    if args.bootstrap == "host":           # testing aid: ranks may share GPUs
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    multi = args.workload == "C5"
    if multi:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        if args.bootstrap == "host":
            dist.init_process_group("gloo", rank=rank, world_size=world)
        else:
            dist.init_process_group("nccl", device_id=dev, rank=rank, world_size=world)
    if args.lib:
        gbs.LIB_PATH = args.lib
    elif rank == 0:
        _build.build()
    if multi:
        dist.barrier()
    w = WORKLOADS[args.workload]
    pairs = w["pairs"]
    stream = torch.cuda.current_stream()
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    peak, peak_src = peaks()
    cfg = config_of(args, world)
    line = {"metric": METRIC}
    if multi:
        res = run_c5(args, torch, dist, gi, gbs, dev, world, rank, local, stream, flush, peak)
        if rank != 0:
            dist.destroy_process_group()
            return
        line.update(res)
        line["config"] = cfg
        print(json.dumps(line))
        dist.destroy_process_group()
        return

    # ---------------- headline (N = 1)
    n = args.size or w["n"]
    if args.ncu_one:
        keys = gi.generate_torch(args.dist, n, seed=0, device=dev)
        vals = torch.arange(n, dtype=torch.int32, device=dev) if pairs else None
        torch.cuda.synchronize()
        if pairs:
            gbs.sort_pairs(keys, vals)
        else:
            gbs.sort_keys(keys)
        torch.cuda.synchronize()
        print(json.dumps({"ncu_one": args.workload, "n": n}))
        return
    res = run_single(args, torch, gi, gbs, dev, stream, flush, peak, n, pairs, args.dist, args.steps, args.warmup,
                     headline=True)
    unit = "pairs/s" if pairs else "keys/s"
    line.update({"value": res["value"], "unit": unit, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                 "ms_per_step": res["ms"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                 "dtype": "u32 pairs" if pairs else "u32", "data": "synthetic", "config": cfg,
                 "e2e": res.get("e2e"), "gpu_launches": res["launches"], "clocks": res["clocks"],
                 "roofline": None, "verified": res["verified"], "step_ms_min_max": res["minmax"]})
    dom = res["dominant"]
    if dom is not None:
        t_ms, lev, k, ab = dom
        kern = STEP_KERNEL.get(k, STEP_NAMES[k])
        traffic, lim = ncu_record(f"{args.workload}:{kern}:level{lev + 1}")
        ach = ab / (t_ms / 1e3) / 1e9
        line["roofline"] = {"bound": "hbm", "kernel": f"{kern} (level {lev + 1}, {STEP_NAMES[k]})",
                            "achieved": round(ach, 1), "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4),
                            "peak_source": peak_src, "traffic": traffic, "alg_bytes_per_launch": ab,
                            "launch_ms": round(t_ms, 4), "limiter": lim,
                            "alg_bytes_rule": "2 x item bytes per item (load + store) + 8 B per sample written"}
    line["steps_breakdown"] = res["breakdown"]
    gc(torch, res)

    # ---------------- extras in the same run: C2, C3 x 7 distributions, the C5 base point
    if not args.no_extras and not args.size:
        c2 = run_single(args, torch, gi, gbs, dev, stream, flush, peak, WORKLOADS["C2"]["n"], False, "uniform",
                        args.steps, args.warmup)
        line["c2"] = {"workload": WORKLOADS["C2"]["name"], "value": c2["value"], "unit": "keys/s", "ms": c2["ms"],
                      "verified": c2["verified"], "roofline_frac": c2["dominant_frac"],
                      "steps_breakdown": c2["breakdown"]}
        gc(torch, c2)
        c3 = {}
        for d in DISTS:
            r = run_single(args, torch, gi, gbs, dev, stream, flush, peak, WORKLOADS["C3"]["n"], False, d,
                           max(5, args.steps // 2), args.warmup, profile=False)
            c3[d] = {"value": r["value"], "ms": r["ms"], "verified": r["verified"]}
            gc(torch, r)
        vals = [c3[d]["value"] for d in DISTS]
        line["c3"] = {"workload": WORKLOADS["C3"]["name"], "unit": "keys/s", "per_dist": c3,
                      "spread": (max(vals) - min(vals)) / statistics.mean(vals), "spread_def": "(max - min) / mean",
                      "all_verified": all(c3[d]["verified"] for d in DISTS)}
        cb = run_single(args, torch, gi, gbs, dev, stream, flush, peak, C5_BASE_N, False, "uniform",
                        max(3, args.steps // 4), args.warmup, profile=False)
        line["c5_base"] = {"workload": "C5 shape on one GPU: n=2^31 uniform u32 keys (the largest single call; "
                                       "the N=1 base point of the C5 scaling runs)",
                           "value": cb["value"], "unit": "keys/s", "ms": cb["ms"], "verified": cb["verified"]}
        gc(torch, cb)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_line(args, n, pairs)
    print(json.dumps(line))


def gc(torch, res):
    res.pop("_bufs", None)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def run_single(args, torch, gi, gbs, dev, stream, flush, peak, n, pairs, dist_name, steps, warmup,
               headline=False, profile=True):
    """One single-GPU workload: timed sorts, verification against the plain definition,
    per-step breakdown (second pass with the library's step events), e2e (headline)."""
    pristine = gi.generate_torch(dist_name, n, seed=0, device=dev)
    keys = torch.empty_like(pristine)
    vals = torch.empty_like(pristine) if pairs else None
    pristine_v = torch.arange(n, dtype=torch.int32, device=dev) if pairs else None
    ws = gbs.Workspace(dev)
    plan = gbs.plan(n, pairs=pairs)

    def restore():
        keys.copy_(pristine)
        if pairs:
            vals.copy_(pristine_v)

    def one_sort():
        if pairs:
            gbs.sort_pairs(keys, vals, ws=ws)
        else:
            gbs.sort_keys(keys, ws=ws)

    step_ms, clocks = timed_sorts(torch, one_sort, restore, flush, stream, steps, warmup,
                                  clk_index=dev.index if headline else None)
    ms = statistics.mean(step_ms)
    # verification of the timed configuration against the plain definition
    restore()
    one_sort()
    torch.cuda.synchronize()
    verified = verify_sorted(torch, pristine, keys, vals)
    res = {"value": n / (ms / 1e3), "ms": ms, "minmax": [min(step_ms), max(step_ms)], "clocks": clocks,
           "verified": verified, "launches": plan["kernels_per_sort"] * steps, "dominant": None,
           "dominant_frac": None, "breakdown": None}
    if profile:
        gbs.profile_begin()
        for _ in range(min(steps, 10)):
            restore()
            flush.zero_()
            one_sort()
        torch.cuda.synchronize()
        prof = gbs.profile_end()
        if prof["calls"]:
            res["breakdown"], flat = breakdown(prof, plan, n, 8 if pairs else 4, peak)
            cand = [f for f in flat if f[2] in STEP_KERNEL and f[3]]
            if cand:
                res["dominant"] = max(cand, key=lambda f: f[0])
                t_ms, _, _, ab = res["dominant"]
                res["dominant_frac"] = round(ab / (t_ms / 1e3) / 1e9 / peak, 4)
    if headline and not args.no_e2e:
        res["e2e"] = e2e_single(torch, gbs, stream, pristine, pristine_v, keys, vals, ws, steps, warmup)
    res["_bufs"] = (pristine, keys, vals, pristine_v, ws)
    return res


def verify_sorted(torch, pristine, keys, vals, chunk=1 << 28) -> bool:
    """Keys: equal to the sorted input (bit-exact); pairs: stable sort by key (keys equal to
    the input gathered at the values, nondecreasing, equal keys in value = position order)."""
    n = keys.numel()
    if vals is None and n > (1 << 28):
        # very large key sets (the C5 base point): sorted + multiset fingerprint in == out
        ok = fingerprint(torch, pristine).item() == fingerprint(torch, keys).item()
        for c0 in range(0, n - 1, chunk):
            k64 = keys[c0:c0 + chunk + 1].to(torch.int64) & 0xFFFFFFFF
            ok &= bool((k64[1:] >= k64[:-1]).all())
            del k64
        return bool(ok)
    if vals is None:
        ref = torch.sort(pristine.to(torch.int64) & 0xFFFFFFFF).values
        ok = torch.equal(keys.to(torch.int64) & 0xFFFFFFFF, ref)
        del ref
        return bool(ok)
    ok = True
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk + 1)
        k64 = keys[c0:c1].to(torch.int64) & 0xFFFFFFFF
        v = vals[c0:c1]
        ok &= torch.equal(pristine[v.long()], keys[c0:c1])
        ok &= bool((k64[1:] >= k64[:-1]).all())
        eq = k64[1:] == k64[:-1]
        ok &= bool((v[1:][eq] > v[:-1][eq]).all())
        del k64, eq
    # the values are a permutation of 0..n-1 (with the gather check: the multiset of keys)
    seen = torch.zeros(n, dtype=torch.bool, device=keys.device)
    seen[vals.long()] = True
    ok &= bool(seen.all())
    return bool(ok)


def e2e_single(torch, gbs, stream, pristine, pristine_v, keys, vals, ws, steps, warmup):
    """End to end through the C-ABI host-buffer entry: pinned host input -> H2D -> sort ->
    D2H, all inside the CUDA-event window (gbs_sort_keys_host / gbs_sort_pairs_host)."""
    pairs = vals is not None
    host = pristine.cpu()
    hk = torch.empty_like(host).pin_memory()
    hostv = pristine_v.cpu() if pairs else None
    hv = torch.empty_like(hostv).pin_memory() if pairs else None

    def go():
        if pairs:
            gbs.sort_pairs_host(hk, hv, keys, vals, ws=ws)
        else:
            gbs.sort_keys_host(hk, keys, ws=ws)

    for _ in range(max(1, min(2, warmup))):
        hk.copy_(host)
        if pairs:
            hv.copy_(hostv)
        go()
    torch.cuda.synchronize()
    e_ms = []
    for i in range(max(3, steps // 4)):
        hk.copy_(host)
        if pairs:
            hv.copy_(hostv)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        go()
        b.record(stream)
        b.synchronize()
        e_ms.append(a.elapsed_time(b))
    n = host.numel()
    ok = bool(torch.equal(hk, keys.cpu())) and (not pairs or bool(torch.equal(hv, vals.cpu())))
    em = statistics.mean(e_ms)
    nb = 4 * n * (2 if pairs else 1)
    return {"value": n / (em / 1e3), "unit": "pairs/s" if pairs else "keys/s", "h2d_bytes_per_step": nb,
            "d2h_bytes_per_step": nb, "ms_per_step": em, "matches_device_result": ok,
            "entry": "gbs_sort_pairs_host" if pairs else "gbs_sort_keys_host"}


# ----------------------------------------------------------------- C5 (multi-GPU)

def fingerprint(torch, t, chunk=1 << 27):
    """Multiset fingerprint: sum over items of a 64-bit mix of the key (mod 2^64) and the
    item count; order-independent, so input and output fingerprints match iff (with
    overwhelming probability) the multisets do."""
    c1 = 0x9E3779B97F4A7C15 - (1 << 64)
    c2 = 0xBF58476D1CE4E5B9 - (1 << 64)
    acc = torch.zeros((), dtype=torch.int64, device=t.device)
    for c0 in range(0, t.numel(), chunk):
        x = t[c0:c0 + chunk].to(torch.int64) & 0xFFFFFFFF
        x = (x + 1) * c1
        x = x ^ ((x >> 31) & ((1 << 33) - 1))
        x = x * c2
        x = x ^ ((x >> 29) & ((1 << 35) - 1))
        acc += x.sum()
    return acc


def run_c5(args, torch, dist, gi, gbs, dev, world, rank, local, stream, flush, peak):
    N = args.size or WORKLOADS["C5"]["n"]
    n = N // world
    pristine = gi.generate_torch(args.dist, N, seed=0, device=dev, start=n * rank, count=n)
    keys = pristine.clone()
    comm = gbs.Comm(bootstrap=args.bootstrap)
    # the group's collectives run on the device for NCCL, on the host for gloo
    cdev = dev if args.bootstrap == "nccl" else torch.device("cpu")
    ws = gbs.Workspace(dev)
    _, cap = gbs.dist_workspace_size(n, world)
    out = torch.empty(cap, dtype=torch.int32, device=dev)

    def one_sort():
        return gbs.sort_keys_dist(keys, comm, out=out, ws=ws)

    for _ in range(args.warmup):
        one_sort()
    torch.cuda.synchronize()
    # verification: fingerprint in vs out, per-rank sortedness, boundary order, bound
    part = one_sort()
    torch.cuda.synchronize()
    p64 = part.to(torch.int64) & 0xFFFFFFFF
    ok_sorted = bool((p64[1:] >= p64[:-1]).all()) if part.numel() > 1 else True
    fin, fout = fingerprint(torch, pristine), fingerprint(torch, part)
    info = torch.stack([fin, fout, torch.tensor(part.numel(), device=dev),
                        p64[0] if part.numel() else torch.tensor(-1, device=dev),
                        p64[-1] if part.numel() else torch.tensor(-1, device=dev),
                        torch.tensor(int(ok_sorted), device=dev)]).to(cdev)
    allinfo = [torch.empty_like(info) for _ in range(world)]
    dist.all_gather(allinfo, info)
    rows = [t.tolist() for t in allinfo]
    del p64
    total_in = sum(r[0] for r in rows) & ((1 << 64) - 1)
    total_out = sum(r[1] for r in rows) & ((1 << 64) - 1)
    ends = [(r[3], r[4]) for r in rows if r[2] > 0]
    checks = {"fingerprint_in_eq_out": total_in == total_out, "count": sum(r[2] for r in rows) == N,
              "parts_sorted": all(r[5] for r in rows),
              "boundaries_ordered": all(ends[k][1] <= ends[k + 1][0] for k in range(len(ends) - 1)),
              "receive_bound": all(r[2] <= cap for r in rows), "max_part": max(r[2] for r in rows),
              "receive_bound_value": cap}
    dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        for i in range(args.steps):
            flush.zero_()
            dist.barrier()
            starts[i].record(stream)
            one_sort()
            ends_ev[i].record(stream)
        torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends_ev)]
    # exchange time (E8) from the library's phase events: NVLink GB/s
    gbs.profile_begin()
    for _ in range(3):
        dist.barrier()
        one_sort()
    torch.cuda.synchronize()
    ph = gbs.dist_profile_end()
    t = torch.tensor([statistics.mean(step_ms), ph.get("exchange_ms", 0.0), ph.get("exchange_bytes", 0.0)],
                     dtype=torch.float64, device=cdev)
    tmax = t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms = float(tmax[0].item())
    # e2e per rank: pinned host shard -> device -> multi-GPU sort -> the rank's part -> pinned host
    host = pristine.cpu().pin_memory()
    hout = torch.empty(out.numel(), dtype=torch.int32).pin_memory()
    e_ms, moved = [], 0
    for i in range(max(3, args.steps // 4) + 1):
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        keys.copy_(host, non_blocking=True)
        part = one_sort()
        hout[:part.numel()].copy_(part, non_blocking=True)
        b.record(stream)
        b.synchronize()
        if i:
            e_ms.append(a.elapsed_time(b))
        moved = part.numel()
    te = torch.tensor([statistics.mean(e_ms)], dtype=torch.float64, device=cdev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    em = float(te[0].item())
    comm.close()
    if rank != 0:
        return None
    ex_ms, ex_bytes = float(tmax[1].item()), float(t[2].item())
    res = {"value": N / (ms / 1e3), "unit": "keys/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
           "data": "synthetic", "verified": all(v for k, v in checks.items() if isinstance(v, bool)),
           "checks": checks, "clocks": clk.summary(),
           "e2e": {"value": N / (em / 1e3), "unit": "keys/s", "h2d_bytes_per_step": 4 * N,
                   "d2h_bytes_per_step": 4 * N, "ms_per_step": em},
           # our kernels per sort: the local sort's plan, plus (p > 1) samples, E4 sample sort,
           # fine cuts, push, merge and (peer-memory path) three barriers
           "gpu_launches": (gbs.plan(n)["kernels_per_sort"] + (0 if world == 1 else (8 if ph.get("path", "").startswith("peer") else 4))) * args.steps,
           "exchange": {"ms_max_over_ranks": ex_ms, "bytes_rank0": ex_bytes,
                        "nvlink_GBps_rank0": (ex_bytes / (ex_ms / 1e3) / 1e9) if ex_ms > 0 else None,
                        "nvlink_peak_GBps_per_direction": 900.0, "path": ph.get("path")},
           "phases_ms_rank0": {k: v for k, v in ph.items() if k.endswith("_ms")}}
    return res


if __name__ == "__main__":
    main()
