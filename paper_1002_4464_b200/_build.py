"""In-tree build of libgbs.so (nvcc, sm_100a) -- used by __graft_entry__.build()."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgbs.so")
SOURCES = ["gbs_api.cu", "gbs_dist.cu", "gbs_merge.cu"]
DEPS = SOURCES + ["gbs_kernels.cuh", "cta_sort.cuh", "gbs_internal.h", "../../include/gbs.h"]


def nccl_root() -> str:
    import nvidia.nccl  # torch's NCCL (same libnccl.so.2 the process loads with torch)
    return list(nvidia.nccl.__path__)[0]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(os.path.join(CSRC, d)) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile libgbs.so in-tree (or to `out` with extra -D `defines`, for tuning runs)."""
    if out is None and not force and not needs_build():
        return LIB
    target = out or LIB
    nccl = nccl_root()
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", f"-I{nccl}/include",
           *[os.path.join(CSRC, s) for s in SOURCES],
           f"-L{nccl}/lib", "-l:libnccl.so.2", "-Xlinker", "-rpath", "-Xlinker", f"{nccl}/lib",
           *[f"-D{d}" for d in defines],
           "-o", target + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build(force=True, verbose=True))
