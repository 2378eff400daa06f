"""Seeded synthetic workloads (INPUTS ONLY — no SRMDP arithmetic here).

Shared by tests/, bench.py and __graft_entry__.smoke(): the oracle and the
CUDA path each turn these plain dicts into their own problem objects.
Shapes follow BASELINE.json ``configs`` and SURVEY.md §8(d); the problem
families follow the paper's §5.1 benchmark and the
closed-form cases of DESIGN.md §Inputs.

Parameter layouts (docs/streams.md §7 and include/srmdp.h):
  dyn "bm": none; "gbm" and "gbm_exact": [mu_0..mu_{d-1}, s_0..s_{d-1}];
  "affine": [b0 (d), B1 (d*d row-major), S0 (d*q row-major)]
  f "zero": none; "linear": [a, c, theta_0..theta_{q-1}]  (f = a y + theta.z + c);
  "paper": none  ((sum z)(y - (2+q)/(2q)))
  g "affine": [a, w_0..w_{d-1}]; "paper": none (omega/(1+omega))
  "user" kinds: the problem is given as source (``user_src``, include/srmdp.h
  "User problems") with ``user_params``; the CUDA path compiles it with NVRTC,
  the oracle with gcc.
"""
from __future__ import annotations

import math


def paper_local_lipschitz(q: int) -> float:
    """Local L_f of the §5.1 driver on |y|<=1, |z_k|<=1 (reading R5)."""
    return max(q / 4.0, math.sqrt(q) * (0.5 + 1.0 / q))


def cfg1(seed: int = 1, M: int = 256) -> dict:
    """d=q=1, X=W, f=0, affine g, N=4, #C=10, M=256 (BASELINE configs[0])."""
    return dict(name="cfg1", d=1, q=1, N=4, T=1.0, dyn="bm", f="zero", g="affine",
                g_params=[0.5, 0.25], C=10, L=6.5, mu=1.0, M=M,
                C_y_override=math.inf, C_z_override=math.inf, seed=seed)


def cfg2(seed: int = 1, M: int = 1024, N: int = 10, C: int = 20) -> dict:
    """d=q=2 Black-Scholes-type linear driver, GBM, N=10, 20^2 cells, M=1024 (configs[1])."""
    mu, s, r = 0.05, 0.2, 0.03
    theta = (mu - r) / s
    return dict(name="cfg2", d=2, q=2, N=N, T=1.0, dyn="gbm",
                dyn_params=[mu, mu, s, s], f="linear", f_params=[-r, 0.0, -theta, -theta],
                g="affine", g_params=[1.0, 1.0, 1.0], C=C, L=6.5, mu=1.0, M=M,
                C_y_override=math.inf, C_z_override=math.inf, seed=seed,
                bs=dict(mu=mu, s=s, r=r, a=1.0, w=[1.0, 1.0]))


def cfg2_exact(seed: int = 1, M: int = 1024, N: int = 10, C: int = 20) -> dict:
    """cfg2 with the exact GBM transition (Alg. "SDE dynamics")."""
    return dict(cfg2(seed, M, N, C), name="cfg2x", dyn="gbm_exact")


def benchmark(d: int, N: int, C: int, M: int, seed: int = 1, name: str = "bench", basis: str = "lp1") -> dict:
    """§5.1 benchmark: X=W, d=q, T=1, mu=1, L=6.5, C_g=1, C_f=0.
    basis "lp1" (affine, the hot path) or "lp0" (piecewise constant)."""
    return dict(name=name, d=d, q=d, N=N, T=1.0, dyn="bm", f="paper", g="paper",
                C=C, L=6.5, mu=1.0, M=M, C_g=1.0, C_f=0.0, L_f=paper_local_lipschitz(d),
                seed=seed, basis=basis)


def cfg3(seed: int = 1, M: int = 2048) -> dict:
    """d=4 benchmark, N=20, 10^4 cells, M=2048 (configs[2])."""
    return benchmark(4, 20, 10, M, seed, "cfg3")


def cfg4(seed: int = 1, M: int = 4096) -> dict:
    """d=6 benchmark, N=30, 5^6 cells, M=4096 (configs[3]) — the bench workload."""
    return benchmark(6, 30, 5, M, seed, "cfg4")


def cfg5(seed: int = 1, M: int = 3200) -> dict:
    """d=19 benchmark, N=5, 2^19 cells, M=3200 (paper row P:1259; configs[4])."""
    return benchmark(19, 5, 2, M, seed, "cfg5")


def bookkeeping(d: int = 2, N: int = 5, C: int = 4, M: int = 64, seed: int = 7,
                beta=None, r: float = 0.1, a: float = 0.3, w=None) -> dict:
    """sigma=0, constant drift beta, f = r y, g = a + w.x (closed form)."""
    beta = list(beta) if beta is not None else [0.9 * (l + 1) for l in range(d)]
    w = list(w) if w is not None else [0.5 - 0.2 * l for l in range(d)]
    q = d
    dyn = beta + [0.0] * (d * d) + [0.0] * (d * q)
    return dict(name="bookkeeping", d=d, q=q, N=N, T=1.0, dyn="affine", dyn_params=dyn,
                f="linear", f_params=[r, 0.0] + [0.0] * q, g="affine", g_params=[a] + w,
                C=C, L=2.0, mu=1.0, M=M, C_y_override=math.inf, C_z_override=math.inf,
                seed=seed, bk=dict(beta=beta, r=r, a=a, w=w))


# ---------------------------------------------------------------------------
# User problems (include/srmdp.h "User problems"): b, sigma, f, g as source.
# The text is valid C and CUDA; SRMDP_D / SRMDP_Q / SRMDP_USER_FN come from the
# compiling side. Inputs only: each source *defines a problem*.
# ---------------------------------------------------------------------------
# cfg2's problem (GBM, linear driver, affine g) written as user code with the
# built-in families' operation order. p = [mu (d), s (d), a, c, theta (q), g0, w (d)].
USER_GBM_LINEAR_SRC = r"""
SRMDP_USER_FN void srmdp_user_b(const double* p, double t, const double* x, double* b) {
  for (int l = 0; l < SRMDP_D; ++l) b[l] = p[l] * x[l];
}
SRMDP_USER_FN void srmdp_user_sigma(const double* p, double t, const double* x, double* s) {
  for (int l = 0; l < SRMDP_D; ++l)
    for (int k = 0; k < SRMDP_Q; ++k) s[l * SRMDP_Q + k] = (l == k) ? p[SRMDP_D + l] * x[l] : 0.0;
}
SRMDP_USER_FN double srmdp_user_f(const double* p, double t, const double* x, double y, const double* z) {
  const double* th = p + 2 * SRMDP_D + 2;
  double v = p[2 * SRMDP_D] * y;
  for (int l = 0; l < SRMDP_Q; ++l) v = v + th[l] * z[l];
  return v + p[2 * SRMDP_D + 1];
}
SRMDP_USER_FN double srmdp_user_g(const double* p, const double* x) {
  const double* g = p + 2 * SRMDP_D + 2 + SRMDP_Q;
  double s = g[0];
  for (int l = 0; l < SRMDP_D; ++l) s = s + g[1 + l] * x[l];
  return s;
}
"""


def user_cfg2(seed: int = 1, M: int = 1024, N: int = 10, C: int = 20) -> dict:
    """cfg2 (GBM + linear driver + affine g) as a user problem: same problem,
    same operation order as the built-in families."""
    w = cfg2(seed, M, N, C)
    d = w["d"]
    mu, s = w["dyn_params"][:d], w["dyn_params"][d:]
    up = list(mu) + list(s) + list(w["f_params"]) + list(w["g_params"])
    return dict(w, name="user_cfg2", dyn="user", f="user", g="user", dyn_params=[], f_params=[], g_params=[],
                user_src=USER_GBM_LINEAR_SRC, user_params=up)


# The §5.1 benchmark as user code: X = W, f = (sum z)(y - (2+q)/(2q)),
# g = 1/(1 + exp(-(T + sum x))) (reading R22). p = [T].
USER_BENCH_SRC = r"""
SRMDP_USER_FN void srmdp_user_b(const double* p, double t, const double* x, double* b) {
  for (int l = 0; l < SRMDP_D; ++l) b[l] = 0.0;
}
SRMDP_USER_FN void srmdp_user_sigma(const double* p, double t, const double* x, double* s) {
  for (int l = 0; l < SRMDP_D; ++l)
    for (int k = 0; k < SRMDP_Q; ++k) s[l * SRMDP_Q + k] = (l == k) ? 1.0 : 0.0;
}
SRMDP_USER_FN double srmdp_user_f(const double* p, double t, const double* x, double y, const double* z) {
  double sz = 0.0;
  for (int l = 0; l < SRMDP_Q; ++l) sz = sz + z[l];
  return sz * (y - (2.0 + (double)SRMDP_Q) / (2.0 * (double)SRMDP_Q));
}
SRMDP_USER_FN double srmdp_user_g(const double* p, const double* x) {
  double s = p[0];
  for (int l = 0; l < SRMDP_D; ++l) s = s + x[l];
  return 1.0 / (1.0 + exp(-s));
}
"""


def user_benchmark(d: int, N: int, C: int, M: int, seed: int = 1) -> dict:
    """The §5.1 benchmark written as a user problem."""
    return dict(benchmark(d, N, C, M, seed, "user_bench"), dyn="user", f="user", g="user",
                user_src=USER_BENCH_SRC, user_params=[1.0])


# Time-dependent deterministic drift, driver reading t and x:
#   b_l(t, x) = beta_l (1 + t), sigma = 0, f(t, x, y, z) = r y + c t + e sum_l x_l,
#   g(x) = a + w.x.   p = [beta (d), r, c, e, a, w (d)].
# Closed form by the affine recursion Y_i(x) = Y_{i+1}(x + beta (1 + t_i) dt)
# + f(t_i, x, Y_{i+1}(...)) dt.
USER_TIME_SRC = r"""
SRMDP_USER_FN void srmdp_user_b(const double* p, double t, const double* x, double* b) {
  for (int l = 0; l < SRMDP_D; ++l) b[l] = p[l] * (1.0 + t);
}
SRMDP_USER_FN void srmdp_user_sigma(const double* p, double t, const double* x, double* s) {
  for (int l = 0; l < SRMDP_D * SRMDP_Q; ++l) s[l] = 0.0;
}
SRMDP_USER_FN double srmdp_user_f(const double* p, double t, const double* x, double y, const double* z) {
  double sx = 0.0;
  for (int l = 0; l < SRMDP_D; ++l) sx = sx + x[l];
  return (p[SRMDP_D] * y + p[SRMDP_D + 1] * t) + p[SRMDP_D + 2] * sx;
}
SRMDP_USER_FN double srmdp_user_g(const double* p, const double* x) {
  double s = p[SRMDP_D + 3];
  for (int l = 0; l < SRMDP_D; ++l) s = s + p[SRMDP_D + 4 + l] * x[l];
  return s;
}
"""


def user_time(d: int = 2, N: int = 5, C: int = 4, M: int = 40, seed: int = 7, beta=None, r: float = 0.1,
              c: float = 0.7, e: float = -0.3, a: float = 0.3, w=None) -> dict:
    """Deterministic user problem with t- and x-dependent drift / driver (closed form)."""
    beta = list(beta) if beta is not None else [0.6 * (l + 1) for l in range(d)]
    w = list(w) if w is not None else [0.5 - 0.2 * l for l in range(d)]
    return dict(name="user_time", d=d, q=d, N=N, T=1.0, dyn="user", f="user", g="user",
                user_src=USER_TIME_SRC, user_params=beta + [r, c, e, a] + w,
                C=C, L=2.0, mu=1.0, M=M, C_y_override=math.inf, C_z_override=math.inf, seed=seed,
                ut=dict(beta=beta, r=r, c=c, e=e, a=a, w=w))


# A nonlinear user problem: state-dependent (rational, bounded) diffusion with
# a cross term, mean-reverting drift with a time term, a driver reading t, x,
# y and every z_k (vendor sin), logistic terminal value (vendor exp).
# b and sigma use only + - * / so path states are reproducible bit for bit.
USER_NONLINEAR_SRC = r"""
SRMDP_USER_FN void srmdp_user_b(const double* p, double t, const double* x, double* b) {
  for (int l = 0; l < SRMDP_D; ++l) b[l] = p[0] * (x[(l + 1) % SRMDP_D] - x[l]) + p[1] * t;
}
SRMDP_USER_FN void srmdp_user_sigma(const double* p, double t, const double* x, double* s) {
  for (int l = 0; l < SRMDP_D; ++l)
    for (int k = 0; k < SRMDP_Q; ++k) {
      double v = 0.0;
      if (k == l % SRMDP_Q) v = p[2] * (1.0 + 0.5 * x[l] * x[l]) / (1.0 + x[l] * x[l]);
      else if (k == (l + 1) % SRMDP_Q) v = p[3];
      s[l * SRMDP_Q + k] = v;
    }
}
SRMDP_USER_FN double srmdp_user_f(const double* p, double t, const double* x, double y, const double* z) {
  double sz = 0.0;
  for (int k = 0; k < SRMDP_Q; ++k) sz = sz + z[k] * (1.0 + 0.1 * k);
  return -p[4] * y + p[5] * sin(sz) * (y - 0.5) + p[6] * t * x[0];
}
SRMDP_USER_FN double srmdp_user_g(const double* p, const double* x) {
  double s = 0.0;
  for (int l = 0; l < SRMDP_D; ++l) s = s + x[l];
  return 1.0 / (1.0 + exp(-s));
}
"""


def user_nonlinear(d: int = 3, q: int = 3, N: int = 5, C: int = 4, M: int = 300, seed: int = 5) -> dict:
    """Nonlinear user problem (parity case for the NVRTC path)."""
    return dict(name="user_nl", d=d, q=q, N=N, T=1.0, dyn="user", f="user", g="user",
                user_src=USER_NONLINEAR_SRC, user_params=[0.3, 0.2, 0.3, 0.05, 0.5, 0.2, 0.1],
                C=C, L=2.5, mu=1.0, M=M, C_y_override=math.inf, C_z_override=math.inf, seed=seed)


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}


def path_steps(w: dict) -> int:
    """K*M*N(N+1)/2 — the metric's unit."""
    K = w["C"] ** w["d"]
    return K * w["M"] * w["N"] * (w["N"] + 1) // 2


# ---------------------------------------------------------------------------
# Parameter schedules of the paper's experiments (captions of the MSE tables)
# and the §4.3 calibration. Inputs only.
# ---------------------------------------------------------------------------
def paper_schedule(table: str, N: int) -> tuple[int, int]:
    """(#C, M) of a table row from its caption formula.

    LP0 d=4 (table:LP0d4): #C = floor(4 sqrt N), M = N^2.
    LP0 d=6 (table:LP0d6_0 / _1): #C = floor(sqrt N) / floor(2 sqrt N), M = N^2.
    LP1 d=4 (table:LP1d4): #C = floor(3 sqrt(d sqrt N)) - 5, M = (d+1) N^2.
    LP1 d=6 (table:LP1d6_1): #C = floor(1.5 sqrt(d sqrt N)) - 3, M = (d+1) N^2.
    """
    if table == "table:LP0d4":
        return int(math.floor(4 * math.sqrt(N))), N * N
    if table == "table:LP0d6_0":
        return int(math.floor(math.sqrt(N))), N * N
    if table == "table:LP0d6_1":
        return int(math.floor(2 * math.sqrt(N))), N * N
    if table == "table:LP1d4":
        d = 4
        return int(math.floor(3 * math.sqrt(d * math.sqrt(N)))) - 5, (d + 1) * N * N
    if table == "table:LP1d6_1":
        d = 6
        return int(math.floor(1.5 * math.sqrt(d * math.sqrt(N)))) - 3, (d + 1) * N * N
    raise KeyError(table)


def complexity_domain_L(N: int, mu: float = 1.0) -> float:
    """L = log(N)/mu of the theoretical calibration: nu(R^d \\ [-L,L]^d) <= 2d e^{-mu L} = O(1/N)."""
    return math.log(N) / mu
