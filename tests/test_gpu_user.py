"""GPU <-> oracle parity of the NVRTC path (include/srmdp.h "User problems";
SURVEY §8(f) row 4): user problems compiled at srmdp_create, (d, q) pairs
outside the static set, the equal-probability grid above d = 8, and the forced
NVRTC build of a compiled problem. Same bars as test_gpu_parity.py: path
states and cells bit-exact, coefficients within max(1e-9 |ref|, 1e-12).
"""
import numpy as np
import pytest

import workloads
from test_gpu_parity import assert_coeff_parity, gpu  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu

TRACE_CASES = [workloads.user_nonlinear(), workloads.user_nonlinear(d=3, q=2), workloads.user_cfg2(N=5, C=6, M=64),
               workloads.user_time(d=2), workloads.benchmark(d=9, N=3, C=2, M=40, seed=2)]


@pytest.mark.parametrize("w", TRACE_CASES, ids=lambda w: "%s-d%dq%d" % (w["name"], w["d"], w["q"]))
def test_user_path_states_bit_exact(gpu, orc, w):
    P = orc.Problem(w)
    rng = np.random.default_rng(11)
    with gpu.Solver(w) as s:
        for _ in range(5):
            i = int(rng.integers(0, w["N"]))
            k = int(rng.integers(0, P.K))
            m0 = int(rng.integers(0, 500))
            x, c, dw = s.trace(i, k, m0, 16)
            for t in range(16):
                ox, oc, ow = P.trace(i, k, m0 + t)
                assert np.array_equal(x[t].view(np.uint64), ox.view(np.uint64)), (i, k, m0 + t)
                assert np.array_equal(c[t], oc), (i, k, m0 + t)
                assert np.array_equal(dw[t].view(np.uint64), ow.view(np.uint64)), (i, k, m0 + t)


SOLVE_CASES = [
    workloads.user_nonlinear(),                                       # full-z driver, t, x; state-dependent sigma
    workloads.user_nonlinear(d=3, q=2, M=257),                        # q != d, ragged M
    workloads.user_nonlinear(d=2, q=2, N=4, C=5, M=600, seed=8),
    dict(workloads.user_nonlinear(d=3, q=3, N=4, C=4, M=200, seed=9), grid="equiprobable"),
    dict(workloads.user_nonlinear(d=2, q=2, N=4, C=4, M=200, seed=10), C_z_override=0.3, C_y_override=0.6),
    workloads.user_cfg2(N=5, C=6, M=128),
    workloads.user_nonlinear(d=5, q=5, N=4, C=3, M=300, seed=16),    # MMA Gram path (d >= 4) with a user driver
    dict(workloads.user_nonlinear(d=4, q=4, N=3, C=3, M=200, seed=18), C_z_override=0.2, C_y_override=0.55),
    workloads.user_nonlinear(d=6, q=2, N=3, C=2, M=257, seed=17),
    workloads.user_time(d=3, N=4, C=3, M=40),
    workloads.user_benchmark(d=4, N=4, C=3, M=200, seed=12),
    workloads.benchmark(d=9, N=3, C=2, M=120, seed=13),               # (9,9): not in the static set
    workloads.benchmark(d=10, N=2, C=2, M=64, seed=14),
    dict(workloads.cfg2(N=4, C=5, M=128), name="affine_d10q3", d=10, q=3, dyn="affine", C=2,
         dyn_params=[0.05] * 10 + [0.0] * 100 + [0.2, 0.0, 0.1] * 10, f_params=[-0.03, 0.01, 0.1, -0.2, 0.05],
         g_params=[1.0] + [0.5] * 10),
    dict(workloads.benchmark(d=11, N=2, C=2, M=64, seed=15), grid="equiprobable"),   # EQ above d = 8
    # maximum dimensions (d, q <= 32): one cell, affine dynamics
    dict(workloads.cfg2(N=2, C=1, M=80), name="affine_d32q1", d=32, q=1, dyn="affine", C=1,
         dyn_params=[0.05] * 32 + [0.0] * (32 * 32) + [0.3] * 32, f_params=[-0.03, 0.01, 0.2],
         g_params=[1.0] + [0.1] * 32),
    dict(workloads.cfg2(N=3, C=3, M=64), name="affine_d1q32", d=1, q=32, dyn="affine", C=3,
         dyn_params=[0.05, 0.1] + [0.02] * 32, f_params=[-0.03, 0.01] + [0.01] * 32, g_params=[1.0, 0.5]),
]


@pytest.mark.parametrize("w", SOLVE_CASES, ids=lambda w: "%s-d%dq%d-N%d-C%d-M%d%s" % (
    w["name"], w["d"], w["q"], w["N"], w["C"], w["M"], "-eq" if w.get("grid") else ""))
def test_user_solve_parity(gpu, orc, w):
    P = orc.Problem(w)
    ref, fb = P.solve()
    with gpu.Solver(w) as s:
        s.solve()
        assert s.stats()["lp0_fallbacks"] == fb
        assert_coeff_parity(s.table(), ref, "centered beta")
        x = np.random.default_rng(3).logistic(size=(400, w["d"]))
        for i in range(w["N"]):
            y, z = s.eval(i, x)
            oy, oz = P.eval(ref, i, x)
            assert_coeff_parity(y, oy, "eval y")
            assert_coeff_parity(z, oz, "eval z")
        y = s.eval(w["N"], x, want_z=False)
        assert_coeff_parity(y, P.eval(ref, w["N"], x, want_z=False), "eval g")


def test_user_time_closed_form_on_gpu(gpu):
    """The deterministic user problem reproduces its affine closed form."""
    from test_user_problem import _time_truth
    w = workloads.user_time(d=2, N=5, C=4, M=40)
    truth = _time_truth(w)
    x = np.random.default_rng(0).uniform(-3, 3, (300, 2))
    with gpu.Solver(w) as s:
        s.solve()
        for i in range(w["N"]):
            y, _ = s.eval(i, x)
            A, W = truth[i]
            ex = A + x @ W
            assert np.max(np.abs(y - ex) / np.maximum(np.abs(ex), 1.0)) < 1e-12


def test_forced_nvrtc_matches_static_build(gpu):
    """SRMDP_FLAG_JIT: the NVRTC build of a compiled (d, q) agrees with the
    static kernels within the coefficient bar (it differs only by --fmad=false
    in the non-path arithmetic), and both are deterministic."""
    w = workloads.benchmark(d=4, N=5, C=4, M=500, seed=21)
    with gpu.Solver(w) as a, gpu.Solver(w, flags=gpu.FLAG_JIT) as b:
        ta = a.solve().table()
        tb = b.solve().table()
        tb2 = b.solve().table()
    assert_coeff_parity(tb, ta, "jit vs static")
    assert np.array_equal(tb.view(np.uint64), tb2.view(np.uint64))


def test_user_and_builtin_agree_on_gpu(gpu):
    """cfg2 as user code vs the built-in GBM / linear / affine families."""
    w0, w1 = workloads.cfg2(N=5, C=6, M=256), workloads.user_cfg2(N=5, C=6, M=256)
    with gpu.Solver(w0) as a, gpu.Solver(w1) as b:
        assert_coeff_parity(b.solve().table(), a.solve().table(), "user vs builtin")


def test_module_cache_and_params(gpu):
    """Two handles with the same source share one module; different
    user_params give different tables (parameters are runtime data)."""
    import time
    w = workloads.user_time(d=2, N=3, C=3)
    with gpu.Solver(w) as a:
        ta = a.solve().table()
    t0 = time.perf_counter()
    w2 = dict(w, user_params=list(w["user_params"]))
    w2["user_params"][2] = 0.2
    with gpu.Solver(w2) as b:
        tb = b.solve().table()
    assert time.perf_counter() - t0 < 1.5          # no second NVRTC compile
    assert np.abs(ta - tb).max() > 1e-3
