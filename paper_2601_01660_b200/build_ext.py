"""Build libdgsm.so (hand-written CUDA for sm_100a) in-tree with nvcc.

``python -m paper_2601_01660_b200.build_ext [--force] [--verbose]``

project.cu and slab.cu are compiled with ``-fmad=false`` (no FMA contraction: the binning
decisions follow DESIGN.md's fp64 "binning arithmetic contract"); every other
translation unit uses the default contraction.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libdgsm.so")
BUILD = os.path.join(HERE, "csrc", "build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
          "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
SOURCES = ["project.cu", "slab.cu", "scan.cu", "binning.cu", "onesweep.cu", "accumulate.cu", "query.cu", "transfer.cu", "dgsm_api.cu"]
PER_FILE = {"project.cu": ["-fmad=false"], "slab.cu": ["-fmad=false"]}
HEADERS = ["dgsm_internal.cuh"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def build(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdr_time = max(_mtime(os.path.join(CSRC, h)) for h in HEADERS)
    hdr_time = max(hdr_time, _mtime(os.path.join(ROOT, "include", "dgsm.h")))
    objs, rebuilt = [], False
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _mtime(o) < max(_mtime(s), hdr_time, _mtime(__file__)):
            cmd = [NVCC, *ARCH, *COMMON, *PER_FILE.get(src, []), *os.environ.get("DGSM_NVCC_EXTRA", "").split(),
                   "-c", s, "-o", o]
            if ptxas_verbose:
                cmd += ["-Xptxas", "-v"]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.check_call(cmd)
            rebuilt = True
    if rebuilt or force or _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv,
          ptxas_verbose="--ptxas" in sys.argv)
    print(LIB)
