"""Build libepsm.so in-tree with nvcc for sm_100a (no torch JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SOURCES = [os.path.join(CSRC, f) for f in ("epsm.cu", "epsm_sharded.cu", "epsm_multi.cu", "epsm_host.cu", "epsm_long.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("epsm_kernels.cuh", "epsm_multi.cuh", "epsm_ptx.cuh", "epsm_internal.h", "epsm_long.cuh", "epsm_mask.cuh", "epsm_code.cuh")] + \
    [os.path.join(ROOT, "include", "epsm.h")]
OUT = os.path.join(HERE, "libepsm.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_include() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            inc = os.path.join(loc, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include"
    raise RuntimeError("nccl.h not found")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    tmp = OUT + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, "-lineinfo", "-O3", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=default", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           "-I", nccl_include(), "-o", tmp, *SOURCES, "-ldl"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
