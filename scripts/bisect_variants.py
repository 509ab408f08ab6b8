"""Build libgbs variants with -D switches and run a pytest selection against each (GPU box)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1002_4464_b200 import _build
sel = sys.argv[1]
variants = {"default": [], "nopresort": ["GBS_PRESORTED=0"], "noadapt": ["GBS_ADAPT_DEPTH=0"],
            "neither": ["GBS_PRESORTED=0", "GBS_ADAPT_DEPTH=0"]}
for name, d in variants.items():
    lib = f"/tmp/libgbs_{name}.so"
    _build.build(out=lib, defines=d)
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-q", "-x", "-k", sel],
                       capture_output=True, text=True, env=dict(os.environ, GBS_LIB=lib), cwd=ROOT)
    print(name, r.stdout.strip().splitlines()[-1], flush=True)
