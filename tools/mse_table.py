"""Reproduce the paper's MSE tables (tests/golden/paper_mse_all.txt) with the CUDA
solver: for every row within the path-step budget, R runs (R = 1000 as in the
paper when affordable), printed next to the paper's values (markdown)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402
from paper_2407_21085_b200.mse import mse_indicators  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 2e12     # total path-steps per row
rows = [l.split() for l in open(os.path.join(ROOT, "tests", "golden", "paper_mse_all.txt")) if l[0] != "#"]
print("| basis | d | N | #C | K | M | runs | ours Y,max / Y,av / Z,av | paper | P: | s |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    basis, d, N, C, K, M = r[0], int(r[1]), int(r[2]), int(r[3]), int(r[4]), int(r[5])
    paper = tuple(float(v) for v in r[6:9])
    steps = K * M * N * (N + 1) // 2
    runs = int(min(1000, max(20, budget // steps)))
    if steps * 20 > budget * 5 or (12 * N * K * ((d + 1) * 3 + 16) * 8 > 150e9):
        print("| %s | %d | %d | %d | %d | %d | skipped (%.2g path-steps/run) | | %.3f / %.3f / %.3f | %s | |"
              % (basis, d, N, C, K, M, steps, *paper, r[9]))
        continue
    w = workloads.benchmark(d=d, N=N, C=C, M=M, basis=basis)
    t0 = time.time()
    m = mse_indicators(w, runs)
    print("| %s | %d | %d | %d | %d | %d | %d | %.3f / %.3f / %.3f | %.3f / %.3f / %.3f | %s | %.0f |" % (
        basis, d, N, C, K, M, runs, m["MSE_Y_max"], m["MSE_Y_av"], m["MSE_Z_av"], *paper, r[9], time.time() - t0),
        flush=True)
