"""Build libpmg_b200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

``python -m paper_2205_09411_b200.build`` or ``__graft_entry__.build()``.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpmg_b200.so")

SOURCES = ["capi.cu", "ops.cu", "tree.cu"] + [f"ops_{d}_{n}.cu" for d in (2, 3) for n in (4, 8, 16, 32)]
HEADERS = ["ctx.h", "kernels.cuh", "cells.cuh", "pmg_dev.cuh", "stencil_build.cuh", "ops_impl.cuh", "tiles.cuh", "coarse.cuh", "tile_kernels.cuh", "coarse_cluster.cuh", "stream.cuh", "small.cuh", "fields.cuh", "brick.cuh", "dist.h", "coop.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # every per-cell result is bit-identical to the CPU reference only without
    # FMA contraction (the reference is built without -march)
    "--fmad=false",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr",
]


def _nvcc():
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if p and (os.path.exists(p) or p == "nvcc"):
            return p
    return "nvcc"


def stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    for f in SOURCES + HEADERS:
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    inc = os.path.join(HERE, "..", "include")
    for f in os.listdir(inc):
        p = os.path.join(inc, f)
        if os.path.isfile(p) and os.path.getmtime(p) > t:
            return True
    return False


def build(force=False, verbose=False, extra=None):
    if not force and not stale():
        return OUT
    objs, procs = [], []
    for s in SOURCES:  # translation units compile in parallel
        obj = os.path.join(CSRC, s.replace(".cu", ".o"))
        cmd = [_nvcc(), *NVCC_FLAGS, *(extra or []), "-c", os.path.join(CSRC, s), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(obj)
    for p, cmd in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, cmd)
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", OUT,
           "-lcudart"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    for o in objs:
        os.remove(o)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True,
          extra=["-Xptxas", "-v"] if "--ptxas" in sys.argv else None)
