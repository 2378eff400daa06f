"""Host-side breakdown of the e2e call sequence of bench.py (create, solve,
coeffs of every slice into pinned memory, destroy), wall clock with syncs."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_2407_21085_b200 import srmdp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
w = workloads.CONFIGS[name]()
torch.cuda.init()
stream = torch.cuda.Stream()
host = None
for rep in range(4):
    t = [time.perf_counter()]
    s = srmdp.Solver(w, stream=stream.cuda_stream)
    t.append(time.perf_counter())
    s.solve()
    t.append(time.perf_counter())
    st = s.stats()
    if host is None:
        host = torch.empty((w["N"], st["K"], st["B"]), dtype=torch.float64).pin_memory().numpy()
    for i in range(w["N"]):
        s.coeffs(i, 1, host[i])
    t.append(time.perf_counter())
    s.close()
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print("rep %d  create %.1f ms  solve %.1f ms  coeffs %.1f ms  destroy %.1f ms  total %.1f ms" % (rep, *d, t[-1] - t[0] and (t[-1] - t[0]) * 1e3))
