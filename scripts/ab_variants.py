"""A/B of libgbs build variants (-D switches) on the bench (GPU box): value and step split.

usage: python scripts/ab_variants.py name=DEF1,DEF2 name2= ... [-- bench args]"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1002_4464_b200 import _build
args = sys.argv[1:]
bench_args = []
if "--" in args:
    i = args.index("--")
    args, bench_args = args[:i], args[i + 1:]
for spec in args:
    name, _, defs = spec.partition("=")
    d = [x for x in defs.split(",") if x]
    lib = f"/tmp/libgbs_{name}.so"
    _build.build(out=lib, defines=d)
    for rep in range(2):
        r = subprocess.run([sys.executable, "bench.py", "--lib", lib, "--steps", "20", "--warmup", "3", "--no-cpu-baseline",
                            "--no-e2e", "--no-extras"] + bench_args,
                           capture_output=True, text=True, cwd=ROOT)
        try:
            j = json.loads(r.stdout.strip().splitlines()[-1])
            st = {}
            for lev, steps in (j.get("steps_breakdown") or {}).items():
                for k, v in steps.items():
                    st[f"{lev[-1]}:{k.split()[1]}"] = v["ms"]
            print(f"{name:14s} {j['value'] / 1e9:7.2f} G/s  {j['ms_per_step']:.4f} ms  {st}", flush=True)
        except Exception as e:  # noqa: BLE001
            print(name, "failed", e, r.stderr[-400:], flush=True)
