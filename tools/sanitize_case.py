"""Small solves through the C ABI for compute-sanitizer runs (one tool per call):
cfg2-like GBM (d=2), benchmark d=4 with ragged M, d=19 (MMA Gram path), eval and
trace hooks, loopback sharding."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2407_21085_b200 import srmdp  # noqa: E402

cases = [workloads.cfg2(N=4, C=5, M=300), workloads.benchmark(d=4, N=3, C=3, M=300, seed=3),
         workloads.benchmark(d=19, N=2, C=1, M=600, seed=4)]
for w in cases:
    with srmdp.Solver(w) as s:
        s.solve()
        t = s.table()
        x = np.random.default_rng(0).normal(size=(100, w["d"]))
        s.eval(0, x)
        s.eval(w["N"], x, want_z=False)
        s.trace(0, 0, 0, 4)
        assert np.all(np.isfinite(t))
with srmdp.Solver(workloads.benchmark(d=3, N=3, C=3, M=100, seed=5), world=4, flags=srmdp.FLAG_LOOPBACK) as s:
    s.solve()
print("sanitize cases ok")
