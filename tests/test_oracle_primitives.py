"""Pins of the oracle's primitives against things other than itself.

Philox: published known-answer vectors. detmath: mpmath at high precision.
Sampler: closed forms of the logistic CDF and a KS test against the
analytic conditional law (Alg. stratify). Locate / Euler: closed
examples ((A_Strat.) P:188-197; Alg. Euler). Bounds: eq. prop:bound
 evaluated by hand.
"""
import math

import mpmath as mp
import numpy as np
import pytest
from scipy import stats

import workloads

mp.mp.prec = 120


def ulp_err(got, exact):
    exact = mp.mpf(exact)
    if exact == 0:
        return 0.0 if got == 0 else math.inf
    ulp = math.ulp(float(exact))
    return float(abs(mp.mpf(got) - exact) / ulp)


# ---------------------------------------------------------------- Philox
@pytest.mark.parametrize("ctr,key,out", [
    ([0, 0, 0, 0], [0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
    ([0xffffffff] * 4, [0xffffffff] * 2, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
    ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0],
     [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]),
])
def test_philox_known_answers(orc, ctr, key, out):
    assert orc.philox(ctr, key) == out


def test_u01_exact_extremes(orc):
    assert orc.u01(0) == 2.0 ** -53
    assert orc.u01(0xFFFFFFFFFFFFFFFF) == 1.0 - 2.0 ** -53
    assert orc.u01(1 << 63) == 0.5 + 2.0 ** -53
    # values are odd multiples of 2^-53: never 0 or 1
    rng = np.random.default_rng(3)
    for w in rng.integers(0, 2 ** 63, size=1000, dtype=np.uint64):
        u = orc.u01(int(w))
        assert 0.0 < u < 1.0 and (u * 2 ** 53) % 2 == 1


# ---------------------------------------------------------------- detmath
@pytest.mark.parametrize("fn", ["dm_log", "dm_log_series"])
def test_dm_log_ulp(orc, fn):
    f = getattr(orc, fn)
    rng = np.random.default_rng(11)
    xs = list(np.exp(rng.uniform(-745, 709, 3000))) + list(rng.uniform(0, 1, 3000)) + \
        list(1 + rng.uniform(-1e-3, 1e-3, 500)) + list(rng.uniform(0.99, 1.01, 500)) + \
        [2.0 ** -53, 1 - 2.0 ** -53, 0.5, 1.0, 2.0, math.sqrt(2), 1.4140625, 1.41405, 1.9921875,
         0.99609375, 5e-324, 2.2250738585072014e-308, 1e300]
    worst = max(ulp_err(f(float(x)), mp.log(mp.mpf(float(x)))) for x in xs if x > 0)
    assert worst <= 3.0, worst
    assert f(1.0) == 0.0
    assert f(0.0) == -math.inf and f(math.inf) == math.inf
    assert math.isnan(f(-1.0))


def test_dm_exp_ulp(orc):
    rng = np.random.default_rng(12)
    xs = list(rng.uniform(-700, 700, 3000)) + list(rng.uniform(-1, 1, 2000)) + [0.0, 1.0, -1.0, 709.7]
    worst = max(ulp_err(orc.dm_exp(float(x)), mp.exp(mp.mpf(float(x)))) for x in xs)
    assert worst <= 2.0, worst
    assert orc.dm_exp(0.0) == 1.0
    assert orc.dm_exp(800.0) == math.inf and orc.dm_exp(-800.0) == 0.0


@pytest.mark.parametrize("fn", ["dm_sincospi2", "dm_sincospi2_series"])
def test_dm_sincospi2(orc, fn):
    f = getattr(orc, fn)
    rng = np.random.default_rng(13)
    us = list(rng.uniform(0, 1, 4000)) + [2.0 ** -53, 0.125, 0.25, 0.5, 0.75, 1 - 2.0 ** -53] + \
        [j / 128 for j in range(128)] + [(j + 1) / 128 - 2.0 ** -53 for j in range(127)]
    ws, wc = 0.0, 0.0
    for u in us:
        s, c = f(float(u))
        a = 2 * mp.pi * mp.mpf(float(u))
        es, ec = mp.sin(a), mp.cos(a)
        # absolute error in units of 2^-53 (values near zero are not relatively accurate
        # because 2*pi*u itself is rounded when u is; the contract is bit-equality)
        ws = max(ws, float(abs(mp.mpf(s) - es) * 2 ** 53))
        wc = max(wc, float(abs(mp.mpf(c) - ec) * 2 ** 53))
    assert ws <= 3.0 and wc <= 3.0, (ws, wc)
    assert f(0.25)[0] == 1.0 and abs(f(0.25)[1]) < 1e-16
    assert f(0.5)[1] == -1.0


# ---------------------------------------------------------------- sampler
def test_logistic_cdf_closed_forms(orc):
    assert orc.F(1.0, 0.0) == 0.5
    assert abs(orc.F(1.0, math.log(3.0)) - 0.75) < 1e-15          # 1/(1+1/3)
    assert orc.F(2.0, math.inf) == 1.0 and orc.F(2.0, -math.inf) == 0.0
    for mu in (0.5, 1.0, 3.0):
        for x in (-4.0, -0.3, 0.0, 1.7, 6.5):
            assert abs(orc.F(mu, x) - 1.0 / (1.0 + math.exp(-mu * x))) < 2e-16


def test_inverse_conditional_cdf(orc):
    # median of the symmetric law and of symmetric cells is 0 (P:243 at U=1/2)
    assert orc.inv_cdf_cond(1.0, -math.inf, math.inf, 0.5) == 0.0
    for a in (0.3, 1.0, 6.5):
        assert abs(orc.inv_cdf_cond(1.0, -a, a, 0.5)) < 1e-15
    # F(x) = F(lo) + U (F(hi) - F(lo)) within 1e-12
    rng = np.random.default_rng(5)
    for _ in range(500):
        mu = rng.uniform(0.5, 3)
        lo, hi = np.sort(rng.uniform(-6, 6, 2))
        U = rng.uniform(0, 1)
        x = orc.inv_cdf_cond(mu, lo, hi, U)
        Fl, Fh = 1 / (1 + math.exp(-mu * lo)), 1 / (1 + math.exp(-mu * hi))
        assert abs(1 / (1 + math.exp(-mu * x)) - (Fl + U * (Fh - Fl))) < 1e-12
        assert lo - 1e-12 <= x <= hi + 1e-12


@pytest.mark.parametrize("cell", [0, 3, 9])
def test_start_points_ks_and_membership(orc, cell):
    w = workloads.cfg1(M=4000)
    P = orc.Problem(w)
    xs = np.array([P.start_point(2, cell, m)[0] for m in range(4000)])
    assert all(P.locate([x]) == cell for x in xs)
    C, L, mu = w["C"], w["L"], w["mu"]
    delta = 2 * L / C
    lo = -math.inf if cell == 0 else -L + cell * delta
    hi = math.inf if cell == C - 1 else -L + (cell + 1) * delta
    F = lambda x: 1 / (1 + np.exp(-mu * x))
    Fl = 0.0 if cell == 0 else F(lo)
    Fh = 1.0 if cell == C - 1 else F(hi)
    cdf = lambda x: (F(x) - Fl) / (Fh - Fl)
    D = stats.kstest(xs, cdf).statistic
    assert D < 1.63 / math.sqrt(len(xs))


def test_brownian_increments_are_normal(orc):
    w = workloads.benchmark(d=3, N=8, C=2, M=4000)
    P = orc.Problem(w)
    dt = 1.0 / 8
    z = np.array([P.brownian(1, 4, 5, m) for m in range(4000)]) / math.sqrt(dt)
    for l in range(3):
        assert stats.kstest(z[:, l], "norm").statistic < 1.63 / math.sqrt(4000)
    assert abs(np.corrcoef(z.T)[0, 1]) < 0.06   # independent components


def test_path_and_reference_functions_agree(orc):
    """The table-driven path functions and the series references compute the
    same functions (pins the tables: a wrong LT_j or SCT entry shifts a whole
    1/128 interval)."""
    rng = np.random.default_rng(14)
    for x in list(rng.uniform(0, 1, 2000)) + list(np.exp(rng.uniform(-40, 40, 2000))):
        a, b = orc.dm_log(float(x)), orc.dm_log_series(float(x))
        assert abs(a - b) <= 4 * math.ulp(max(abs(a), abs(b))), x
    for u in rng.uniform(0, 1, 2000):
        s1, c1 = orc.dm_sincospi2(float(u))
        s2, c2 = orc.dm_sincospi2_series(float(u))
        assert abs(s1 - s2) <= 5 * 2.0 ** -53 and abs(c1 - c2) <= 5 * 2.0 ** -53


def test_box_muller_special_case(orc):
    # u_a = e^{-1/2} gives rho = 1; the first increment is then sdt*cos(2 pi u_b)
    assert abs(math.sqrt(-2.0 * orc.dm_log(math.exp(-0.5))) - 1.0) < 1e-15


def test_locate_examples(orc):
    assert orc.locate1(-5.0, 2, 1.0) == 0
    assert orc.locate1(0.0, 2, 1.0) == 1                 # half-open [x-, x+)
    assert orc.locate1(1e300, 7, 6.5) == 6 and orc.locate1(-1e300, 7, 6.5) == 0
    assert orc.locate1(float("nan"), 7, 6.5) == 0
    w = dict(workloads.cfg1(), d=2, q=2, C=2, L=1.0, dyn="bm", g="affine", g_params=[0, 0, 0])
    P = orc.Problem(w)
    assert P.locate([0.5, -0.5]) == 1 * 2 + 0            # multi (1,0), row-major


def test_cell_centers(orc):
    w = dict(workloads.cfg1(), C=4, L=2.0)
    P = orc.Problem(w)
    assert [P.center(k)[0] for k in range(4)] == [-1.0, -0.5, 0.5, 1.0]
    P1 = orc.Problem(dict(workloads.cfg1(), C=1))
    assert P1.center(0)[0] == 0.0


def test_euler_examples(orc):
    w = dict(workloads.cfg1())
    P = orc.Problem(w)                                   # X = W
    x1 = P.euler(0.0, [0.0], [0.1])
    x2 = P.euler(0.25, x1, [-0.2])
    assert x1[0] == 0.1 and abs(x2[0] + 0.1) < 1e-16
    wa = workloads.bookkeeping(d=1, N=2, beta=[1.0])     # sigma = 0, b = 1, dt = 1/2
    Pa = orc.Problem(wa)
    y1 = Pa.euler(0.0, [0.0], [0.7])
    y2 = Pa.euler(0.5, y1, [-0.3])
    assert y1[0] == 0.5 and y2[0] == 1.0
    wg = workloads.cfg2()                                # GBM: x(1 + mu dt + s dW)
    Pg = orc.Problem(wg)
    xg = Pg.euler(0.0, [2.0, -1.0], [0.1, 0.2])
    dt = 0.1
    assert np.allclose(xg, [2.0 * (1 + 0.05 * dt + 0.2 * 0.1), -1.0 * (1 + 0.05 * dt + 0.2 * 0.2)],
                       rtol=1e-15)


def test_bounds(orc):
    cy, cz, cs, ok = orc.bounds(1.0, 0.0, 0.0, 1, 1.0, 4)
    assert abs(cy - math.exp(6.25)) < 1e-9 * cy and abs(cy - 518.0128) < 1e-4
    assert abs(cz * math.sqrt(0.25) - cy) < 1e-12 * cy
    assert cs == 1.0 and ok                              # L_f = C_f = 0 -> C_* = C_g
    cy2, _, _, ok2 = orc.bounds(1.0, 2.0, 3.0, 2, 1.0, 4)
    assert abs(cy2 - math.exp(0.25 + 6 * 2 * 9) * (1 + 2.0 / (2 * math.sqrt(2)))) < 1e-9 * cy2
    assert not ok2                                       # (T/N) L_f^2 = 2.25 > 1/24


def test_driver_and_terminal(orc):
    w = workloads.benchmark(d=3, N=4, C=2, M=8)
    P = orc.Problem(w)
    x = np.array([0.1, -0.2, 0.3])
    om = math.exp(1.0 + x.sum())
    assert abs(P.g(x) - om / (1 + om)) < 1e-15
    z = np.array([0.1, 0.2, -0.05])
    assert abs(P.f(0.0, x, 0.4, z) - z.sum() * (0.4 - 5 / 6)) < 1e-15


def test_equiprobable_grid(orc):
    """(A_Strat.) example ii: breakpoints at the logistic quantiles, so
    every stratum has nu-mass 1/C; samples stay in their cell (KS vs the
    conditional law) and locate agrees with the breakpoints."""
    C, mu = 5, 1.3
    w = dict(workloads.cfg1(M=3000), C=C, mu=mu, grid="equiprobable")
    P = orc.Problem(w)
    F = lambda x: 1 / (1 + np.exp(-mu * x))
    e = [-math.log(C / c - 1) / mu for c in range(1, C)]
    for c in range(1, C):
        assert abs(F(e[c - 1]) - c / C) < 1e-14
    edges = [-math.inf] + e + [math.inf]
    for cell in range(C):
        xs = np.array([P.start_point(0, cell, m)[0] for m in range(3000)])
        assert all(P.locate([x]) == cell for x in xs)
        assert np.all(xs >= edges[cell] - 1e-12) and np.all(xs <= edges[cell + 1] + 1e-12)
        Fl, Fh = F(edges[cell]) if cell else 0.0, F(edges[cell + 1]) if cell < C - 1 else 1.0
        assert stats.kstest(xs, lambda x: (F(x) - Fl) / (Fh - Fl)).statistic < 1.63 / math.sqrt(3000)
    for x in (-3.0, -0.2, 0.0, 0.7, 10.0):
        assert P.locate([x]) == sum(1 for b in e if b <= x)


def test_paper_schedules_reproduce_printed_rows():
    """The caption formulas (workloads.paper_schedule) give every printed #C and M,
    and K = #C^d on every row of tests/golden/paper_mse_all.txt."""
    import os
    rows = [l.split() for l in open(os.path.join(os.path.dirname(__file__), "golden", "paper_mse_all.txt"))
            if l[0] != "#"]
    checked = 0
    for r in rows:
        d, N, C, K, M, table = int(r[1]), int(r[2]), int(r[3]), int(r[4]), int(r[5]), r[10]
        assert C ** d == K, r
        try:
            c2, m2 = workloads.paper_schedule(table, N)
        except KeyError:
            continue                                # d >= 11 tables give #C and M explicitly
        assert (c2, m2) == (C, M), (r, c2, m2)
        checked += 1
    assert checked == 19
    assert abs(workloads.complexity_domain_L(50) - math.log(50)) < 1e-15
