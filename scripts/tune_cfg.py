"""Tuning sweep (GPU box): build libgbs variants with different CTA-sort configs and
time a C2 sort with each (per-step events).  Not part of the product path."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1002_4464_b200 import _build
VARIANTS = {
    "k512x64c2_w512x32c2": ["GBS_KEYS_BLOCK=512", "GBS_KEYS_ITEMS=64", "GBS_KEYS_CHAINS=2", "GBS_WIDE_BLOCK=512", "GBS_WIDE_ITEMS=32", "GBS_WIDE_CHAINS=2"],
    "k1024x32c1_w1024x16c1": ["GBS_KEYS_BLOCK=1024", "GBS_KEYS_ITEMS=32", "GBS_KEYS_CHAINS=1", "GBS_WIDE_BLOCK=1024", "GBS_WIDE_ITEMS=16", "GBS_WIDE_CHAINS=1"],
    "k1024x32c2_w1024x16c2": ["GBS_KEYS_BLOCK=1024", "GBS_KEYS_ITEMS=32", "GBS_KEYS_CHAINS=2", "GBS_WIDE_BLOCK=1024", "GBS_WIDE_ITEMS=16", "GBS_WIDE_CHAINS=2"],
    "k512x64c1_w512x32c1": ["GBS_KEYS_BLOCK=512", "GBS_KEYS_ITEMS=64", "GBS_KEYS_CHAINS=1", "GBS_WIDE_BLOCK=512", "GBS_WIDE_ITEMS=32", "GBS_WIDE_CHAINS=1"],
}
names = sys.argv[1:] or list(VARIANTS)
for name in names:
    lib = f"/tmp/libgbs_{name}.so"
    _build.build(out=lib, defines=VARIANTS[name])
    env = dict(os.environ, GBS_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "10", "--warmup", "3",
                        "--no-cpu-baseline"], capture_output=True, text=True, env=env)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        br = {k.split()[0]: v["ms"] for k, v in d["steps_breakdown"].items()}
        print(name, f"{d['value']/1e9:.2f} Gkeys/s {d['ms_per_step']:.3f} ms", json.dumps(br), flush=True)
    except Exception as e:
        print(name, "FAILED", e, r.stdout[-500:], r.stderr[-2000:], flush=True)
