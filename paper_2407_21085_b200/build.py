"""Build the CUDA library in-tree: paper_2407_21085_b200/libsrmdp_b200.so.

nvcc for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``), -lineinfo
for ncu source mapping; the host part is compiled with -ffp-contract=off
(docs/streams.md). NCCL is loaded at run time (dlopen), only its header is used.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsrmdp_b200.so")
SOURCES = [os.path.join(CSRC, f) for f in ("srmdp.cu",)]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] + \
    [os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    stale = force or not os.path.exists(LIB) or max(os.path.getmtime(p) for p in DEPS) > os.path.getmtime(LIB)
    if not stale:
        return LIB
    tmp = LIB + ".tmp%d" % os.getpid()
    cmd = [nvcc(), *NVCC_FLAGS, *(["-Xptxas", "-v"] if verbose else []), "-o", tmp, *SOURCES, "-ldl"]
    subprocess.check_call(cmd, cwd=CSRC)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
