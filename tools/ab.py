"""A/B timing of alternative library builds in one process, interleaved.

  python tools/ab.py [--config cfg4] [--rounds 4] [--M M] lib_a.so lib_b.so ...

Each build (`build.py --out PATH -DNAME=VALUE`, or an older commit's library)
is loaded with its own ctypes handle; per round every build runs one warm-up
and two timed solves of the same workload, and the device-timed step-kernel
sum (SRMDP_FLAG_TIME_KERNELS, `srmdp_stats.kernel_ms`) is recorded. Interleaving
the builds round by round spreads clock / thermal drift over all of them.
Prints path-steps/s per build (median and spread) as one JSON line.
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402
from paper_2407_21085_b200 import srmdp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--M", type=int, default=None)
    ap.add_argument("--N", type=int, default=None, help="override N (short sweeps weigh the per-path-start work)")
    a = ap.parse_args()
    w = workloads.CONFIGS[a.config](**({"M": a.M} if a.M else {}))
    if a.N:
        w = dict(w, N=a.N)
    libs = []
    for p in a.libs:
        L = ctypes.CDLL(os.path.abspath(p), mode=ctypes.RTLD_LOCAL)
        L.srmdp_create.argtypes = [ctypes.POINTER(srmdp.srmdp_config), ctypes.POINTER(ctypes.c_void_p)]
        L.srmdp_solve.argtypes = [ctypes.c_void_p]
        L.srmdp_stats.argtypes = [ctypes.c_void_p, ctypes.POINTER(srmdp.srmdp_stats_t)]
        L.srmdp_destroy.argtypes = [ctypes.c_void_p]
        L.srmdp_last_error.restype = ctypes.c_char_p
        L.srmdp_last_error.argtypes = [ctypes.c_void_p]
        cfg, keep = srmdp.config_from_workload(w, flags=srmdp.FLAG_TIME_KERNELS)
        h = ctypes.c_void_p()
        st = L.srmdp_create(ctypes.byref(cfg), ctypes.byref(h))
        if st != 0:
            raise SystemExit("%s: create failed %d %s" % (p, st, L.srmdp_last_error(None)))
        libs.append((p, L, h, keep))
    res = {p: [] for p, *_ in libs}
    steps = None
    rng = np.random.default_rng(0)
    for r in range(a.rounds):
        for idx in rng.permutation(len(libs)):       # build order shuffled per round (drift spreads evenly)
            p, L, h, _ = libs[idx]
            assert L.srmdp_solve(h) == 0
            for _ in range(2):
                assert L.srmdp_solve(h) == 0
                s = srmdp.srmdp_stats_t()
                L.srmdp_stats(h, ctypes.byref(s))
                steps = s.path_steps
                res[p].append(s.path_steps / (s.kernel_ms / 1e3))
    out = {"config": a.config, "M": w["M"], "rounds": a.rounds}
    base = None
    for p, *_ in libs:
        v = np.array(res[p])
        med = float(np.median(v))
        base = base or med
        out[os.path.basename(p)] = {"median": med, "min": float(v.min()), "max": float(v.max()),
                                    "rel": med / base}
    print(json.dumps(out))
    for p, L, h, _ in libs:
        L.srmdp_destroy(h)


if __name__ == "__main__":
    main()
