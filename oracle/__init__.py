"""CPU ORACLE of the SRMDP hot path — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around ``oracle/srmdp_oracle.c`` (plain C, fp64, Householder QR;
Alg. SRMDP of arXiv 2407.21085). Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline / ``--impl
reference``) may import this package. It never imports the CUDA product
(``paper_2407_21085_b200``) and the product never imports it.

The problem description it accepts is the plain dict produced by
``workloads.py`` (inputs only; no method arithmetic there).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "srmdp_oracle.c")
_HDR = os.path.join(_HERE, "srmdp_oracle.h")
_LIB = os.path.join(_HERE, "liboracle_srmdp.so")

DYN = {"bm": 0, "gbm": 1, "affine": 2, "gbm_exact": 3, "user": 4}
FKIND = {"zero": 0, "linear": 1, "paper": 2, "user": 3}
GKIND = {"affine": 0, "paper": 1, "user": 2}

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=gnu11", "-pthread"]


def build(force: bool = False) -> str:
    """Compile the oracle shared library (gcc, -ffp-contract=off)."""
    stale = force or not os.path.exists(_LIB) or max(
        os.path.getmtime(_SRC), os.path.getmtime(_HDR)) > os.path.getmtime(_LIB)
    if stale:
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_PDc = ctypes.POINTER(ctypes.c_double)
_USER_VEC = ctypes.CFUNCTYPE(None, _PDc, ctypes.c_double, _PDc, _PDc)
_USER_F = ctypes.CFUNCTYPE(ctypes.c_double, _PDc, ctypes.c_double, _PDc, ctypes.c_double, _PDc)
_USER_G = ctypes.CFUNCTYPE(ctypes.c_double, _PDc, _PDc)


def build_user(src: str, d: int, q: int) -> str:
    """Compile a user problem's source (include/srmdp.h "User problems") as
    plain C with the oracle's flags (gcc, -ffp-contract=off: each written
    operation one rounding). The source is an input of the problem, like a
    parameter array; it is cached by content hash under the temp directory."""
    import hashlib
    import tempfile
    text = "#include <math.h>\n#define SRMDP_D %d\n#define SRMDP_Q %d\n#define SRMDP_USER_FN\n%s\n" % (d, q, src)
    h = hashlib.sha1((" ".join(CFLAGS) + text).encode()).hexdigest()[:16]
    out = os.path.join(tempfile.gettempdir(), "srmdp_oracle_user_%s.so" % h)
    if not os.path.exists(out):
        c = out[:-3] + ".%d.c" % os.getpid()
        with open(c, "w") as f:
            f.write(text)
        tmp = out + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, c, "-lm"])
        os.replace(tmp, out)
        os.remove(c)
    return out


class _Problem(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int), ("q", ctypes.c_int), ("N", ctypes.c_int),
        ("T", ctypes.c_double),
        ("dyn_kind", ctypes.c_int), ("dyn_params", ctypes.POINTER(ctypes.c_double)),
        ("f_kind", ctypes.c_int), ("f_params", ctypes.POINTER(ctypes.c_double)),
        ("g_kind", ctypes.c_int), ("g_params", ctypes.POINTER(ctypes.c_double)),
        ("C", ctypes.c_int), ("L", ctypes.c_double), ("mu", ctypes.c_double),
        ("M", ctypes.c_int64),
        ("C_y", ctypes.c_double), ("C_z", ctypes.c_double),
        ("seed", ctypes.c_uint64),
        ("lp0", ctypes.c_int),
        ("grid", ctypes.c_int),
        ("user_b", _USER_VEC), ("user_sigma", _USER_VEC), ("user_f", _USER_F), ("user_g", _USER_G),
        ("user_params", ctypes.POINTER(ctypes.c_double)),
    ]


_lib = None
_D = ctypes.c_double
_PD = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.POINTER(_Problem)
        sig = {
            "or_philox4x32_10": (None, [ctypes.POINTER(ctypes.c_uint32)] * 3),
            "or_u01": (_D, [ctypes.c_uint64]),
            "or_dm_log": (_D, [_D]),
            "or_dm_exp": (_D, [_D]),
            "or_dm_sincospi2": (None, [_D, _PD, _PD]),
            "or_dm_log_series": (_D, [_D]),
            "or_dm_sincospi2_series": (None, [_D, _PD, _PD]),
            "or_F": (_D, [_D, _D]),
            "or_inv_cdf_cond": (_D, [_D, _D, _D, _D]),
            "or_locate1": (ctypes.c_int, [_D, ctypes.c_int, _D]),
            "or_locate": (_I64, [P, _PD]),
            "or_cell_center": (None, [P, _I64, _PD]),
            "or_num_cells": (_I64, [P]),
            "or_g": (_D, [P, _PD]),
            "or_f": (_D, [P, _D, _PD, _D, _PD]),
            "or_euler": (None, [P, _D, _PD, _PD, _PD]),
            "or_bounds": (ctypes.c_int, [_D, _D, _D, ctypes.c_int, _D, ctypes.c_int, _PD, _PD, _PD]),
            "or_start_point": (None, [P, ctypes.c_int, _I64, _I64, _PD]),
            "or_brownian": (None, [P, ctypes.c_int, ctypes.c_int, _I64, _I64, _PD]),
            "or_trace_path": (None, [P, ctypes.c_int, _I64, _I64, _PD, ctypes.POINTER(_I64), _PD]),
            "or_ols_qr": (ctypes.c_int, [_PD, _I64, ctypes.c_int, _PD, ctypes.c_int, _PD]),
            "or_step": (_I64, [P, _PD, ctypes.c_int, _I64, _I64, _I64]),
            "or_solve": (_I64, [P, _PD]),
            "or_step_cells": (_I64, [P, _PD, ctypes.c_int, ctypes.POINTER(_I64), _I64]),
            "or_eval": (None, [P, _PD, ctypes.c_int, _I64, _PD, _PD, _PD]),
            "or_num_threads": (ctypes.c_int, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _dptr(a):
    return a.ctypes.data_as(_PD) if a is not None else None


def bounds(C_g, C_f, L_f, q, T, N):
    """Prop. bound: returns (C_y, C_z, C_star, smallness_ok)."""
    cy, cz, cs = _D(), _D(), _D()
    ok = lib().or_bounds(C_g, C_f, L_f, q, T, N, ctypes.byref(cy), ctypes.byref(cz), ctypes.byref(cs))
    return cy.value, cz.value, cs.value, bool(ok)


class Problem:
    """Oracle-side problem built from a ``workloads`` dict."""

    def __init__(self, w: dict):
        self.w = dict(w)
        self.d, self.q, self.N = int(w["d"]), int(w["q"]), int(w["N"])
        self.T = float(w["T"])
        self.C = int(w["C"])
        self.M = int(w["M"])
        self._dyn = np.ascontiguousarray(np.asarray(w.get("dyn_params", []), dtype=np.float64).ravel())
        self._f = np.ascontiguousarray(np.asarray(w.get("f_params", []), dtype=np.float64).ravel())
        self._g = np.ascontiguousarray(np.asarray(w.get("g_params", []), dtype=np.float64).ravel())
        cy, cz = truncation_constants(w)
        self.C_y, self.C_z = cy, cz
        self.s = _Problem(
            self.d, self.q, self.N, self.T,
            DYN[w["dyn"]], _dptr(self._dyn) if self._dyn.size else None,
            FKIND[w["f"]], _dptr(self._f) if self._f.size else None,
            GKIND[w["g"]], _dptr(self._g) if self._g.size else None,
            self.C, float(w["L"]), float(w["mu"]), self.M, cy, cz,
            int(w["seed"]) & 0xFFFFFFFFFFFFFFFF, 1 if w.get("basis", "lp1") == "lp0" else 0,
            1 if w.get("grid", "uniform") == "equiprobable" else 0)
        if w.get("user_src") is not None:      # user problem: the same source, compiled as C
            self._user = ctypes.CDLL(build_user(w["user_src"], self.d, self.q))
            self._up = np.ascontiguousarray(np.asarray(w.get("user_params", [0.0]), dtype=np.float64).ravel())
            if w["dyn"] == "user":
                self.s.user_b = _USER_VEC(("srmdp_user_b", self._user))
                self.s.user_sigma = _USER_VEC(("srmdp_user_sigma", self._user))
            if w["f"] == "user":
                self.s.user_f = _USER_F(("srmdp_user_f", self._user))
            if w["g"] == "user":
                self.s.user_g = _USER_G(("srmdp_user_g", self._user))
            self.s.user_params = _dptr(self._up) if self._up.size else None
        self.K = int(lib().or_num_cells(ctypes.byref(self.s)))
        self.B = (self.q + 1) * (self.d + 1)

    @property
    def ref(self):
        return ctypes.byref(self.s)

    def new_table(self):
        return np.zeros((self.N, self.K, self.B), dtype=np.float64)

    def solve(self):
        t = self.new_table()
        fb = lib().or_solve(self.ref, _dptr(t))
        return t, int(fb)

    def step(self, table, i, k_begin=0, k_end=None, k_stride=1):
        if k_end is None:
            k_end = self.K
        return int(lib().or_step(self.ref, _dptr(table), i, k_begin, k_end, k_stride))

    def step_cells(self, table, i, cells):
        c = np.ascontiguousarray(np.asarray(cells, dtype=np.int64))
        return int(lib().or_step_cells(self.ref, _dptr(table), i, c.ctypes.data_as(ctypes.POINTER(_I64)), c.size))

    def eval(self, table, i, x, want_z=True):
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, self.d)
        n = x.shape[0]
        y = np.zeros(n)
        z = np.zeros((n, self.q)) if want_z else None
        lib().or_eval(self.ref, _dptr(table), i, n, _dptr(x), _dptr(y), _dptr(z) if want_z else None)
        return (y, z) if want_z else y

    def start_point(self, i, k, m):
        x = np.zeros(self.d)
        lib().or_start_point(self.ref, i, k, m, _dptr(x))
        return x

    def brownian(self, i, j, k, m):
        w = np.zeros(self.q)
        lib().or_brownian(self.ref, i, j, k, m, _dptr(w))
        return w

    def trace(self, i, k, m):
        n = self.N - i
        x = np.zeros((n + 1, self.d))
        c = np.zeros(n + 1, dtype=np.int64)
        w = np.zeros((n, self.q))
        lib().or_trace_path(self.ref, i, k, m, _dptr(x), c.ctypes.data_as(ctypes.POINTER(_I64)), _dptr(w))
        return x, c, w

    def locate(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return int(lib().or_locate(self.ref, _dptr(x)))

    def center(self, k):
        r = np.zeros(self.d)
        lib().or_cell_center(self.ref, k, _dptr(r))
        return r

    def g(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return lib().or_g(self.ref, _dptr(x))

    def f(self, t, x, y, z):
        x = np.ascontiguousarray(x, dtype=np.float64)
        z = np.ascontiguousarray(z, dtype=np.float64)
        return lib().or_f(self.ref, t, _dptr(x), y, _dptr(z))

    def euler(self, t, x, dW):
        x = np.ascontiguousarray(x, dtype=np.float64)
        dW = np.ascontiguousarray(dW, dtype=np.float64)
        xn = np.zeros(self.d)
        lib().or_euler(self.ref, t, _dptr(x), _dptr(dW), _dptr(xn))
        return xn

    def raw_alpha(self, table):
        """Convert centered beta to the paper's raw basis alpha (docs/layout.md)."""
        out = table.copy()
        n = self.d + 1
        for k in range(self.K):
            r = self.center(k)
            for blk in range(self.q + 1):
                b = table[:, k, blk * n:(blk + 1) * n]
                out[:, k, blk * n] = b[:, 0] - b[:, 1:] @ r
        return out


def truncation_constants(w: dict):
    """C_y, C_z from overrides or Prop. bound, reading R5."""
    cy = w.get("C_y_override")
    cz = w.get("C_z_override")
    if cy is None or cz is None:
        by, bz, _, _ = bounds(w.get("C_g", 0.0), w.get("C_f", 0.0), w.get("L_f", 0.0),
                              int(w["q"]), float(w["T"]), int(w["N"]))
        cy = by if cy is None else cy
        cz = bz if cz is None else cz
    return float(cy), float(cz)


# primitive wrappers ------------------------------------------------------

def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return [int(v) for v in o]


def u01(w):
    return lib().or_u01(int(w) & 0xFFFFFFFFFFFFFFFF)


def dm_log(x):
    return lib().or_dm_log(float(x))


def dm_log_series(x):
    return lib().or_dm_log_series(float(x))


def dm_sincospi2_series(u):
    s, c = _D(), _D()
    lib().or_dm_sincospi2_series(float(u), ctypes.byref(s), ctypes.byref(c))
    return s.value, c.value


def dm_exp(x):
    return lib().or_dm_exp(float(x))


def dm_sincospi2(u):
    s, c = _D(), _D()
    lib().or_dm_sincospi2(float(u), ctypes.byref(s), ctypes.byref(c))
    return s.value, c.value


def F(mu, x):
    return lib().or_F(float(mu), float(x))


def inv_cdf_cond(mu, lo, hi, U):
    return lib().or_inv_cdf_cond(float(mu), float(lo), float(hi), float(U))


def locate1(x, C, L):
    return int(lib().or_locate1(float(x), int(C), float(L)))


def ols_qr(A, S):
    """OLS by Householder QR. Returns (beta, full_rank)."""
    A = np.ascontiguousarray(A, dtype=np.float64).copy()
    S = np.ascontiguousarray(S, dtype=np.float64)
    if S.ndim == 1:
        S = S[:, None]
    S = S.copy()
    M, n = A.shape
    beta = np.zeros((n, S.shape[1]))
    ok = lib().or_ols_qr(_dptr(A), M, n, _dptr(S), S.shape[1], _dptr(beta))
    return beta, bool(ok)


def num_threads():
    return int(lib().or_num_threads())
