"""Paper-printed MSE indicators reproduced with the CUDA solver (GPU).

eq. mse over 10^3 runs, as the paper, on the §5.1
benchmark; rows from tests/golden/paper_mse_all.txt. The paper ran fp32; the
±0.3 band is SPEC's statistical acceptance band. All three
indicators are pinned on the Δt = 0.2 rows; on finer Δt only MSE_Z (our Y
errors are lower than the paper's there, DESIGN reading R24; the full
comparison is profiles/r01_mse_table.md).
"""
import os

import pytest

import workloads

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_mse_all.txt")


def rows():
    out = {}
    for line in open(GOLDEN):
        if line[0] == "#":
            continue
        r = line.split()
        out[r[9]] = r
    return out


CASES = [("P:1117", 3), ("P:1146", 3), ("P:1010", 3), ("P:1034", 3), ("P:1060", 3), ("P:1171", 3),
         ("P:1119", 1), ("P:982", 1)]


@pytest.mark.parametrize("line,n_pinned", CASES, ids=[c[0] for c in CASES])
def test_paper_mse_row(line, n_pinned):
    from paper_2407_21085_b200.mse import mse_indicators
    r = rows()[line]
    basis, d, N, C, K, M = r[0], int(r[1]), int(r[2]), int(r[3]), int(r[4]), int(r[5])
    assert C ** d == K
    paper = [float(v) for v in r[6:9]]
    m = mse_indicators(workloads.benchmark(d=d, N=N, C=C, M=M, basis=basis), runs=1000)
    ours = [m["MSE_Y_max"], m["MSE_Y_av"], m["MSE_Z_av"]]
    pinned = [2] if n_pinned == 1 else [0, 1, 2]
    for j in pinned:
        assert abs(ours[j] - paper[j]) < 0.3, (line, ours, paper)
