"""Build the CUDA library in-tree: paper_2407_21085_b200/libsrmdp_b200.so.

nvcc for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``), -lineinfo
for ncu source mapping; the host part is compiled with -ffp-contract=off
(docs/streams.md). The per-(d,q) kernel instantiations live in separate
translation units (csrc/inst_*.cu) compiled in parallel, then linked with the
host orchestrator (csrc/srmdp.cu). NCCL is loaded at run time (dlopen), only
its header is used.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
import tempfile
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsrmdp_b200.so")


def sources():
    return [os.path.join(CSRC, "srmdp.cu")] + sorted(glob.glob(os.path.join(CSRC, "inst_*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))


NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def build(force: bool = False, verbose: bool = False, jobs: int | None = None, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile (if stale) into `out` (default: the in-tree LIB). `defines` are
    extra -D flags for A/B experiment builds."""
    lib = out or LIB
    dl = deps()
    stale = force or not os.path.exists(lib) or max(os.path.getmtime(p) for p in dl) > os.path.getmtime(lib)
    if not stale:
        return lib
    tmpdir = tempfile.mkdtemp(prefix="srmdp_build_")
    srcs = sources()
    objs = [os.path.join(tmpdir, os.path.basename(s) + ".o") for s in srcs]
    extra = ["-Xptxas", "-v"] if verbose else []

    def compile_one(pair):
        src, obj = pair
        r = subprocess.run([nvcc(), *NVCC_FLAGS, *extra, *["-D" + d for d in defines], "-c", "-o", obj, src], cwd=CSRC,
                           capture_output=True, text=True)
        return src, r

    jobs = jobs or min(len(srcs), os.cpu_count() or 4)
    with ThreadPoolExecutor(max_workers=jobs) as ex:
        results = list(ex.map(compile_one, zip(srcs, objs)))
    for src, r in results:
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError("nvcc failed on %s" % src)
    tmp = lib + ".tmp%d" % os.getpid()
    subprocess.check_call([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-ldl"])
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    os.rmdir(tmpdir)
    return lib


if __name__ == "__main__":
    # python build.py [--force] [-v] [--out PATH] [-DNAME=VALUE ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else None
    defs = tuple(a[2:] for a in args if a.startswith("-D"))
    print(build(force="--force" in args or bool(defs) or out is not None, verbose="-v" in args, out=out,
                defines=defs))
