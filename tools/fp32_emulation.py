"""Does single precision explain the paper's Y errors at dt < 0.2? (reading R24)

An independent, plain numpy re-implementation of the SRMDP sweep (Alg.
srmdp) in the paper's own GPU arithmetic: single
precision everywhere, the raw LP1 basis (1, x) of P:711 and a
Householder QR per hypercube (LAPACK sgeqrf through numpy), random
numbers from numpy (the paper used cuRAND). The same code in double
precision and with the centred basis (reading R13) is the control. For the
paper's LP1 d = 4 rows (table:LP1d4) it prints the MSE
indicators of eq. mse for each variant next to the printed ones.

Not the oracle and not the product: an experiment with its own arithmetic.

  python tools/fp32_emulation.py [N] [runs]      (N in 5, 10, 20)
"""
import json
import math
import sys

import numpy as np

ROWS = {5: (3, 125, (-4.021, -4.132, -0.900), "P:1117"), 10: (5, 500, (-4.291, -4.696, -1.551), "P:1119"),
        20: (7, 2000, (-4.541, -5.022, -2.281), "P:1121")}


def solve(d, N, C, M, dtype, centred, rng, L=6.5, T=1.0):
    """One SRMDP sweep; returns the coefficient table [N, K, q+1, d+1] in `dtype`
    (raw basis (1, x), or centred (1, x - r_k) when `centred`) and the centres."""
    f = dtype
    q = d
    K = C ** d
    dt = f(T / N)
    sdt = f(math.sqrt(T / N))
    delta = 2.0 * L / C
    edges = np.array([-np.inf] + [-L + c * delta for c in range(1, C)] + [np.inf])
    F = 1.0 / (1.0 + np.exp(-edges))
    cen1 = np.array([0.0] if C == 1 else [(-L + delta) if c == 0 else (-L + (C - 1) * delta) if c == C - 1
                                          else (-L + (c + 0.5) * delta) for c in range(C)])
    cc = np.array(np.unravel_index(np.arange(K), (C,) * d)).T          # [K, d], row-major, last dim fastest
    r = cen1[cc].astype(f)                                             # cell centres [K, d]
    Fa, Fb = F[cc].astype(f), F[cc + 1].astype(f)
    lo, hi = edges[cc].astype(f), edges[cc + 1].astype(f)
    cq = f((2.0 + q) / (2.0 * q))
    tab = np.zeros((N, K, q + 1, d + 1), dtype=f)

    def locate(x):
        c = np.clip(np.floor((x + f(L)) / f(delta)), 0, C - 1).astype(np.int64)
        return np.ravel_multi_index(tuple(c[..., l] for l in range(d)), (C,) * d)

    def evaluate(j, x):                          # y_j, z_j at x [..., d] from slice j (raw or centred)
        kn = locate(x)
        a = x - r[kn] if centred else x
        blk = tab[j, kn]                         # [..., q+1, d+1]
        v = blk[..., 0] + np.einsum("...ol,...l->...o", blk[..., 1:], a)
        return v[..., 0], v[..., 1:]

    def g(x):
        return (f(1.0) / (f(1.0) + np.exp(-(f(T) + x.sum(-1))))).astype(f)

    def fdrv(y, z):
        return (z.sum(-1) * (y - cq)).astype(f)

    for i in range(N - 1, -1, -1):
        U = rng.random((K, M, d), dtype=f)
        p = Fa[:, None, :] + U * (Fb - Fa)[:, None, :]
        p = np.clip(p, np.finfo(f).tiny, np.nextafter(f(1.0), f(0.0)))   # as the contract: p in (0, 1)
        x0 = np.clip(-np.log(f(1.0) / p - f(1.0)), lo[:, None, :], np.nextafter(hi, -np.inf)[:, None, :]).astype(f)
        X = x0.copy()
        dW0 = (sdt * rng.standard_normal((K, M, q), dtype=f)).astype(f)
        X = (X + dW0).astype(f)
        if i + 1 < N:
            Y1, zc = evaluate(i + 1, X)
        else:
            Y1, zc = g(X), None
        acc = np.zeros((K, M), dtype=f)
        yv = Y1
        for j in range(i + 1, N):
            dWj = (sdt * rng.standard_normal((K, M, q), dtype=f)).astype(f)
            X = (X + dWj).astype(f)
            if j + 1 < N:
                yv, zn = evaluate(j + 1, X)
            else:
                yv, zn = g(X), None
            acc = (acc + fdrv(yv, zc) * dt).astype(f)                  # f_j(x_j, y_{j+1}(x_{j+1}), z_j(x_j))
            zc = zn
        B = (yv + acc).astype(f) if i + 1 < N else Y1                  # S_{Y,i+1} = g(x_N) + sum
        A = np.concatenate([np.ones((K, M, 1), dtype=f), (x0 - r[:, None, :]) if centred else x0], axis=-1)
        Qm, R = np.linalg.qr(A)                                        # Householder QR per cell
        tz = (B[..., None] * dW0 / dt).astype(f)                       # Z responses
        bz = np.linalg.solve(R, np.einsum("kmp,kml->kpl", Qm, tz))     # [K, d+1, q]
        zi = np.einsum("kmp,kpl->kml", A, bz).astype(f)
        ty = (B + fdrv(Y1, zi) * dt).astype(f)                         # Y responses with the fresh z_i
        by = np.linalg.solve(R, np.einsum("kmp,km->kp", Qm, ty)[..., None])[..., 0]
        tab[i, :, 0, :] = by
        tab[i, :, 1:, :] = np.transpose(bz, (0, 2, 1))
    return tab, r, locate


def mse(d, N, C, M, dtype, centred, runs, seed=0, npts=1000):
    rng = np.random.default_rng(seed)
    prng = np.random.default_rng(seed + 7)
    emax, ey, ez = [], [], []
    for _ in range(runs):
        tab, r, locate = solve(d, N, C, M, dtype, centred, rng)
        sy, sz = [], []
        for i in range(N):
            u = prng.random((npts, d))
            x = np.log(u / (1 - u))
            om = np.exp(i / N + x.sum(1))
            ty, tz = om / (1 + om), om / (1 + om) ** 2
            kn = locate(x.astype(dtype))
            a = (x - r[kn]) if centred else x
            blk = tab[i, kn].astype(np.float64)
            v = blk[..., 0] + np.einsum("nol,nl->no", blk[..., 1:], a)
            sy.append(np.mean((ty - v[:, 0]) ** 2))
            sz.append(np.mean(np.sum((tz[:, None] - v[:, 1:]) ** 2, axis=1)))
        emax.append(max(sy))
        ey.append(np.mean(sy))
        ez.append(np.mean(sz))
    return [round(math.log(np.mean(v)), 3) for v in (emax, ey, ez)]


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    runs = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    which = sys.argv[3].split(",") if len(sys.argv) > 3 else ["fp32_raw", "fp64_raw", "fp64_centred"]
    C, M, paper, line = ROWS[N]
    out = {"row": "table:LP1d4 d=4 N=%d #C=%d M=%d (%s)" % (N, C, M, line), "runs": runs,
           "paper_fp32_printed": list(paper),
           "indicators": "MSE_Y,max / MSE_Y,av / MSE_Z,av (ln, eq. mse P:926-935)"}
    variants = {"fp32_raw": (np.float32, False), "fp32_centred": (np.float32, True), "fp64_raw": (np.float64, False),
                "fp64_centred": (np.float64, True)}
    for v in which:
        out[v + "_basis_QR"] = mse(4, N, C, M, variants[v][0], variants[v][1], runs)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
