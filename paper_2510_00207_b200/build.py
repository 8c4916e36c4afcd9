"""Build libflowmoe.so in-tree with nvcc for sm_100a (no GPU needed).

Every kernel is compiled with ``-gencode arch=compute_100a,code=sm_100a`` (plain
``-arch=sm_100a`` would emit compute_100 PTX, which rejects tcgen05.*).  NCCL
headers/libs come from the pip ``nvidia-nccl`` package that torch loads, so only
one NCCL (2.28) is ever loaded in-process.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(HERE, "libflowmoe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import nvidia.nccl  # the NCCL torch uses
    return list(nvidia.nccl.__path__)[0]


def _run(cmd):
    print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def build(force: bool = False, verbose_ptxas: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    nccl = nccl_dir()
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdrs = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "flowmoe.h"), os.path.join(ROOT, "include", "flowmoe_test.h")]
    hdr_mtime = max(os.path.getmtime(h) for h in hdrs)
    objs = []
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                    "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"),
                    "-I", os.path.join(nccl, "include")]
    if verbose_ptxas:
        flags += ["-Xptxas", "-v"]
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s) + ".o")
        objs.append(o)
        if not force and os.path.exists(o) and os.path.getmtime(o) > max(os.path.getmtime(s), hdr_mtime):
            continue
        _run([NVCC] + flags + ["-c", s, "-o", o])
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs +
             ["-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2",
              "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
