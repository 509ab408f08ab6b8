"""Time the CPU oracle (oracle/, single-threaded C) at the full SURVEY 8(d) configs on the
GPU box's host: C1, C2, C3 for every distribution and C4 once, pinned to one core, each
output checked against a library sort.  Writes one JSON object (stdout or argv[1]).

usage: python scripts/oracle_timing.py [out.json] [--skip-c4]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import gbs_inputs as gi  # noqa: E402
import oracle  # noqa: E402
from plans import TILE_KEYS, TILE_PAIRS, plan as plan_rule  # noqa: E402
sys.path.insert(0, ROOT)
from bench import cpu_info, pin_one_core  # noqa: E402


def run(n, dist, pairs=False):
    keys = gi.generate(dist, n, seed=0)
    vals = gi.pair_values(n) if pairs else None
    pl = plan_rule(n, TILE_PAIRS if pairs else TILE_KEYS)
    t0 = time.perf_counter()
    k, v, _ = oracle.gbs_sort(keys, vals, plan=pl)
    dt = time.perf_counter() - t0
    if pairs:
        order = np.argsort(keys, kind="stable")
        ok = bool(np.array_equal(k, keys[order]) and np.array_equal(v, vals[order]))
    else:
        ok = bool(np.array_equal(k, np.sort(keys)))
    return {"n": n, "dist": dist, "pairs": pairs, "plan": pl, "seconds": dt,
            "rate": n / dt, "unit": "pairs/s" if pairs else "keys/s", "equals_library_sort": ok}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else None
    core = pin_one_core()
    model, nproc = cpu_info()
    res = {"what": "oracle (plain single-threaded C, oracle/gbs_oracle.c) at the full configs", "pinned_core": core,
           "cpu_model": model, "nproc": nproc, "runs": []}
    res["runs"].append(run(1 << 16, "uniform"))
    res["runs"].append(run(1 << 25, "uniform"))
    for d in gi.DISTRIBUTIONS:
        res["runs"].append(run(1 << 26, d))
        print(json.dumps(res["runs"][-1]), file=sys.stderr, flush=True)
    avail = 0
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable"):
                avail = int(line.split()[1]) * 1024
    except OSError:
        pass
    res["host_mem_available_gb"] = avail / 2**30
    # C4 holds ~8 copies of 2^30 4-byte items on the host (inputs, oracle buffers, checks)
    if "--skip-c4" not in sys.argv and avail > 64 * 2**30:
        res["runs"].append(run(1 << 30, "uniform", pairs=True))
    js = json.dumps(res, indent=1)
    if out:
        open(out, "w").write(js)
    print(js)


if __name__ == "__main__":
    main()
