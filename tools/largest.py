"""The largest §5.1 benchmark that fits one B200 (SURVEY §8(d) cfg5 memory
note: the replicated table is N*K*B_pad*8 bytes; at N = 5, #C = 2 the largest
d that fits 180 GB is d = 22, 94 GB). d = 22 is outside the static kernel set,
so the NVRTC build runs. Times one solve (after a warm-up) and checks sampled
cells of slice N-1 against the oracle. Prints one JSON line.

  python tools/largest.py [d] [M]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the sampled check only)
import workloads  # noqa: E402
from paper_2407_21085_b200 import srmdp  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 22
M = int(sys.argv[2]) if len(sys.argv) > 2 else 3200
w = workloads.benchmark(d=d, N=5, C=2, M=M, seed=1, name="largest-d%d" % d)
t0 = time.perf_counter()
with srmdp.Solver(w, flags=srmdp.FLAG_TIME_KERNELS) as s:
    t_create = time.perf_counter() - t0
    s.solve()
    s.solve()
    st = s.stats()
    last = s.coeffs(w["N"] - 1)
    y0 = s.coeffs(0)
P = oracle.Problem(w)
try:   # the oracle's table is N*K*B doubles of virtual memory; pages appear only where it writes
    tab = P.new_table()
    cells = np.random.default_rng(0).choice(P.K, size=4, replace=False)
    P.step_cells(tab, w["N"] - 1, cells)
    err = max(float(np.max(np.abs(last[k] - tab[w["N"] - 1, k]) / np.maximum(np.abs(tab[w["N"] - 1, k]), 1e-3)))
              for k in cells)
except MemoryError:
    err = None
out = {"workload": w["name"], "d": d, "N": w["N"], "K": P.K, "M": M, "B_pad": st["B_pad"],
       "table_GB": w["N"] * P.K * st["B_pad"] * 8 / 1e9, "path_steps": st["path_steps"],
       "kernel_ms": st["kernel_ms"], "path_steps_per_s": st["path_steps"] / (st["kernel_ms"] / 1e3),
       "create_s_incl_nvrtc": t_create, "grid": st["grid"], "ctas_per_sm": st["ctas_per_sm"],
       "smem_bytes": st["smem_bytes"], "slice_N-1_sampled_max_rel_err_vs_oracle": err,
       "finite": bool(np.all(np.isfinite(y0)))}
print(json.dumps(out))
