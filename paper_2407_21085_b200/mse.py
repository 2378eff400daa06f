"""MSE indicators of the paper's §5.1 experiments (eq. mse),
computed with the CUDA solver.

For R independent runs (Philox key = seed0 + r, `srmdp_reseed`), the solver's
truncated approximations y_i^(M), z_i^(M) are evaluated on the GPU
(`srmdp_eval`) at n points per time step drawn i.i.d. from the logistic law nu
(A_nu; independent of the simulations), against the benchmark's
explicit solution y_i = omega/(1+omega), z_{k,i} = omega/(1+omega)^2,
omega = exp(t_i + sum x):

  MSE_Y,max = ln( mean_runs  max_i  (1/n) sum_m |y_i - y_i^(M)|^2 )
  MSE_Y,av  = ln( mean_runs  (1/(nN)) sum_i sum_m |y_i - y_i^(M)|^2 )
  MSE_Z,av  = ln( mean_runs  (1/(nN)) sum_i sum_m |z_i - z_i^(M)|^2 )

(the paper's "average over 10^3 independent runs" read as the mean of the
inner quantity before the logarithm; n = 10^3 as in the paper).
"""
from __future__ import annotations

import math

import numpy as np

from .srmdp import Solver


def benchmark_solution(t: float, x: np.ndarray):
    """Explicit solution of the §5.1 BSDE at time t, points x (n x d)."""
    om = np.exp(t + x.sum(axis=1))
    y = om / (1.0 + om)
    z = om / (1.0 + om) ** 2
    return y, np.repeat(z[:, None], x.shape[1], axis=1)


def logistic_points(rng: np.random.Generator, n: int, d: int, mu: float = 1.0) -> np.ndarray:
    """n points i.i.d. from nu (product logistic with parameter mu), by inversion."""
    u = rng.uniform(size=(n, d))
    return np.log(u / (1.0 - u)) / mu


def mse_indicators(w: dict, runs: int, n_points: int = 1000, seed0: int = 1000, point_seed: int = 123,
                   **solver_kw) -> dict:
    """(MSE_Y,max, MSE_Y,av, MSE_Z,av) of the benchmark workload `w` over `runs` runs."""
    d, N, T = int(w["d"]), int(w["N"]), float(w["T"])
    rng = np.random.default_rng(point_seed)
    e_max, e_y, e_z = [], [], []
    with Solver(dict(w, seed=seed0), **solver_kw) as s:
        for r in range(runs):
            s.reseed(seed0 + r).solve()
            sy, sz = [], []
            for i in range(N):
                x = logistic_points(rng, n_points, d, float(w["mu"]))
                ty, tz = benchmark_solution(i * T / N, x)
                yh, zh = s.eval(i, x)
                sy.append(np.mean((ty - yh) ** 2))
                sz.append(np.mean(np.sum((tz - zh) ** 2, axis=1)))
            e_max.append(max(sy))
            e_y.append(np.mean(sy))
            e_z.append(np.mean(sz))
    return {"MSE_Y_max": math.log(np.mean(e_max)), "MSE_Y_av": math.log(np.mean(e_y)),
            "MSE_Z_av": math.log(np.mean(e_z)), "runs": runs, "n_points": n_points}
