"""Builds the sm_100a engine library in-tree (paper_2510_24429_b200/libcclp_cuda.so)."""
from __future__ import annotations

import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libcclp_cuda.so")
# translation units: the engine (layouts, setup, iteration launches), the
# single-device C ABI and the sharded solve with its C ABI
SOURCES = ["csrc/engine.cu", "csrc/capi.cu", "csrc/sharded.cu"]
HEADERS = ["csrc/engine.cuh", "csrc/kernels.cuh", "csrc/iter_kernels.cuh", "csrc/setup_kernels.cuh",
           "csrc/sharded.cuh", "csrc/host_util.cuh", "csrc/context.cuh", "csrc/capi_util.cuh",
           "../include/cclp_cu.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(os.path.join(HERE, f)) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    # the translation units compile in parallel, then one shared link
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        cmd = [nvcc(), *NVCC_FLAGS, "-c", "-o", obj, os.path.join(HERE, src)]
        if verbose:
            print(" ".join(cmd))
        procs.append((src, subprocess.Popen(cmd, cwd=HERE)))
        objs.append(obj)
    failed = [src for src, p in procs if p.wait() != 0]
    if failed:
        raise RuntimeError(f"nvcc failed on {failed}")
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=HERE)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
