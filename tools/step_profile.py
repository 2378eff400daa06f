"""Per-time-step kernel times of one solve (srmdp_step_ms) and the path-step
rate of every step: shows where per-cell overheads (start points, reduction,
Cholesky, epilogue) dominate (late steps, short paths)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2407_21085_b200 import srmdp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
w = workloads.CONFIGS[name]()
K = w["C"] ** w["d"]
with srmdp.Solver(w, flags=srmdp.FLAG_TIME_KERNELS) as s:
    s.solve()
    s.solve()
    ms = s.step_ms()
out = []
for i in range(w["N"]):
    steps = K * w["M"] * (w["N"] - i)
    out.append({"i": i, "ms": float(ms[i]), "path_steps": steps, "rate": steps / (ms[i] / 1e3)})
    print("i=%2d  %9.3f ms  %.3e path-steps/s" % (i, ms[i], steps / (ms[i] / 1e3)))
print(json.dumps({"config": name, "total_ms": float(ms.sum()), "steps": out}))
