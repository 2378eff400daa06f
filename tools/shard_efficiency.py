"""Per-rank kernel efficiency of the P-way sharding, measured on one GPU with
SRMDP_FLAG_LOOPBACK: the P shards of every step are launched one after
another, so (sum of shard kernel times) / (one-shard time) exposes the wave
quantisation a rank sees at P GPUs (cells per rank vs resident CTAs)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_2407_21085_b200 import srmdp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
w = workloads.CONFIGS[name]()
res = {}
for P in (1, 2, 4, 8):
    flags = srmdp.FLAG_TIME_KERNELS | (srmdp.FLAG_LOOPBACK if P > 1 else 0)
    with srmdp.Solver(w, world=P, flags=flags) as s:
        s.solve()
        s.solve()
        st = s.stats()
        res[P] = st["kernel_ms"]
    print("P=%d  kernel_ms(all shards)=%.1f  per-rank efficiency vs P=1: %.3f" % (P, res[P], res[1] / res[P]), flush=True)
print(json.dumps({"config": name, "kernel_ms": res}))
