"""One cfg4 solve without the CUDA graph, for ncu captures of single step
kernels (`-k regex:step_kernel -s <launch> -c 1`). Launch n is time step
i = N-1-n (launch 14 = i = 15, the mean path length of cfg4)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2407_21085_b200 import srmdp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
w = workloads.CONFIGS[name]()
with srmdp.Solver(w, flags=srmdp.FLAG_NO_GRAPH) as s:
    s.solve()
    print(s.stats())
