"""In-tree build of libgbs.so (nvcc, sm_100a) -- used by __graft_entry__.build()."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgbs.so")
SOURCES = ["gbs_api.cu", "gbs_dist.cu"]
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
    """Compile libgbs.so in-tree (or to `out` with extra -D `defines`, for tuning runs).
    The translation units compile in parallel, then link."""
    if out is None and not force and not needs_build():
        return LIB
    target = out or LIB
    nccl = nccl_root()
    common = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", f"-I{nccl}/include", *[f"-D{d}" for d in defines]]
    if verbose:
        common.insert(1, "-Xptxas=-v")
    tag = f"{os.getpid()}_{abs(hash((target, tuple(defines)))) % 10**8}"
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join("/tmp", f"gbs_{tag}_{os.path.splitext(src)[0]}.o")
        objs.append(obj)
        procs.append((src, subprocess.Popen(common + ["-c", os.path.join(CSRC, src), "-o", obj])))
    failed = [src for src, pr in procs if pr.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, f"nvcc {failed}")
    subprocess.check_call([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs,
                           f"-L{nccl}/lib", "-l:libnccl.so.2", "-Xlinker", "-rpath", "-Xlinker", f"{nccl}/lib",
                           "-o", target + ".tmp"])
    for o in objs:
        try:
            os.remove(o)
        except OSError:
            pass
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build(force=True, verbose=True))
