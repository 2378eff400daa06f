"""User problems (include/srmdp.h "User problems"): b, sigma,
f, g given as source. CPU side: the oracle's user path is pinned to the
built-in families (bit for bit) and to a closed form that exercises the t and x
arguments; the library's NVRTC build of the kernels is checked without a GPU.
"""
import numpy as np
import pytest

import workloads


@pytest.mark.parametrize("pair", [
    (workloads.cfg2(N=4, C=4, M=64), workloads.user_cfg2(N=4, C=4, M=64)),
    (workloads.benchmark(d=2, N=4, C=3, M=64), workloads.user_benchmark(d=2, N=4, C=3, M=64)),
    (workloads.benchmark(d=3, N=3, C=2, M=48, seed=4), workloads.user_benchmark(d=3, N=3, C=2, M=48, seed=4)),
], ids=["gbm-linear-affine", "bench-d2", "bench-d3"])
def test_oracle_user_equals_builtin_bitwise(orc, pair):
    """The same problem written as user code (same operation order) gives the
    built-in family's table bit for bit: pins the user Euler order
    (x + ((b dt) + sum_p s_lp dW_p)), the f / g plumbing and the parameters."""
    w0, w1 = pair
    t0, f0 = orc.Problem(w0).solve()
    t1, f1 = orc.Problem(w1).solve()
    assert f0 == f1 == 0
    assert np.array_equal(t0.view(np.uint64), t1.view(np.uint64))


def _time_truth(w):
    """Affine recursion of the deterministic user problem: Y_N = a + w.x and
    Y_i(x) = (1 + r dt) Y_{i+1}(x + beta (1 + t_i) dt) + (c t_i + e sum x) dt,
    i.e. f_i(x_i, y_{i+1}(x_{i+1}), .) with x_{i+1} = x_i + b(t_i, x_i) dt."""
    ut, N = w["ut"], w["N"]
    dt = w["T"] / N
    beta = np.array(ut["beta"])
    A, W = ut["a"], np.array(ut["w"], dtype=float)
    out = {N: (A, W)}
    for i in range(N - 1, -1, -1):
        ti = i * dt
        A1, W1 = out[i + 1]
        out[i] = ((1 + ut["r"] * dt) * (A1 + W1 @ beta * (1 + ti) * dt) + ut["c"] * ti * dt,
                  (1 + ut["r"] * dt) * W1 + ut["e"] * dt)
    return out


@pytest.mark.parametrize("d,N,C", [(1, 6, 5), (2, 5, 4), (3, 4, 3)])
def test_oracle_user_time_closed_form(orc, d, N, C):
    w = workloads.user_time(d=d, N=N, C=C, M=40)
    P = orc.Problem(w)
    tab, fb = P.solve()
    assert fb == 0
    truth = _time_truth(w)
    x = np.random.default_rng(0).uniform(-3, 3, (300, d))
    for i in range(N):
        y, _ = P.eval(tab, i, x)
        A, W = truth[i]
        ex = A + x @ W
        assert np.max(np.abs(y - ex) / np.maximum(np.abs(ex), 1.0)) < 1e-12, i


def test_time_closed_form_detects_time_shift():
    """Mutation check: reading b(t_{j+1}, .) or f(t_{j+1}, ...) changes the truth."""
    w = workloads.user_time(d=2, N=5, C=4)
    right = _time_truth(w)[0][0]
    shifted = dict(w, ut=dict(w["ut"]))
    dt = 1.0 / w["N"]
    # t_i -> t_{i+1} everywhere is the same as beta (1 + t + dt), c t -> c (t + dt)
    ut = shifted["ut"]
    ut["beta"] = [b * (1 + dt) for b in ut["beta"]]
    assert abs(_time_truth(shifted)[0][0] - right) > 1e-3


def test_user_params_reach_the_functions(orc):
    """Changing a user parameter changes the solution (the parameter array is
    passed through, not a stale copy)."""
    w = workloads.user_time(d=2, N=3, C=3)
    t0, _ = orc.Problem(w).solve()
    w2 = dict(w, user_params=list(w["user_params"]))
    w2["user_params"][2] = 0.2          # r
    t1, _ = orc.Problem(w2).solve()
    assert np.abs(t0 - t1).max() > 1e-3


# ------------------------------------------------------------------ NVRTC build, no GPU
@pytest.fixture(scope="module")
def lib():
    from paper_2407_21085_b200 import build, srmdp
    build.build()
    return srmdp


@pytest.mark.parametrize("w", [workloads.user_nonlinear(), workloads.user_cfg2(), workloads.user_time(d=3),
                               workloads.user_nonlinear(d=3, q=2)],
                         ids=["nonlinear", "gbm-linear", "time", "nonlinear-d3q2"])
def test_nvrtc_builds_user_problem(lib, w):
    ok, log = lib.srmdp_jit_check(w["d"], w["q"], w["dyn"], w["f"], w["g"], w["user_src"])
    assert ok, log
    assert "sm_100a CUBIN" in log


def test_nvrtc_builds_uncompiled_dq(lib):
    """(d, q) outside the static set (srmdp_build_info) come from NVRTC too."""
    assert "(9,9)" not in lib.srmdp_build_info()
    ok, log = lib.srmdp_jit_check(9, 9, "bm", "paper", "paper", None)
    assert ok, log
    ok, log = lib.srmdp_jit_check(10, 3, "affine", "linear", "affine", None)
    assert ok, log


def test_nvrtc_reports_user_errors(lib):
    ok, log = lib.srmdp_jit_check(2, 2, "user", "zero", "affine", "this is not C")
    assert not ok and "user_src(1)" in log
    # dynamics selected but srmdp_user_sigma missing
    src = "SRMDP_USER_FN void srmdp_user_b(const double* p, double t, const double* x, double* b) { b[0] = 0; }"
    ok, log = lib.srmdp_jit_check(2, 2, "user", "zero", "affine", src)
    assert not ok and "srmdp_user_sigma" in log
    with pytest.raises(lib.SrmdpError):
        lib.srmdp_jit_check(33, 1, "bm", "zero", "affine", None)
