"""ctypes binding of include/srmdp.h (+ include/srmdp_debug.h).

Argument marshalling only: every step of the SRMDP sweep runs in the CUDA
kernels of ``libsrmdp_b200.so``. Function names mirror the C ABI. Loading
fails loudly (``SrmdpError``) when the library is missing — there is no CPU
or PyTorch fallback.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SRMDP_LIB") or os.path.join(_HERE, "libsrmdp_b200.so")   # override: A/B builds

DYN = {"bm": 0, "gbm": 1, "affine": 2, "gbm_exact": 3, "user": 4}
FKIND = {"zero": 0, "linear": 1, "paper": 2, "user": 3}
GKIND = {"affine": 0, "paper": 1, "user": 2}
FLAG_NO_GRAPH = 1
FLAG_TIME_KERNELS = 2
FLAG_FORCE_NCCL = 4
FLAG_LOOPBACK = 8
FLAG_JIT = 16
FLAG_P2P_EXCHANGE = 32
FLAG_P2P_SELF_PEER = 64
FLAG_NVLS_EXCHANGE = 128
FLAG_INKERNEL_FLAGS = 256

STATUS = {0: "SRMDP_OK", -1: "SRMDP_E_ARG", -2: "SRMDP_E_PRECOND", -3: "SRMDP_E_STATE", -4: "SRMDP_E_CUDA",
          -5: "SRMDP_E_NCCL", -6: "SRMDP_E_NOMEM", -7: "SRMDP_E_UNSUPPORTED", -8: "SRMDP_E_JIT"}


class SrmdpError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


class srmdp_fn(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("n_params", ctypes.c_int), ("params", ctypes.POINTER(ctypes.c_double))]


class srmdp_config(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int), ("q", ctypes.c_int), ("N", ctypes.c_int), ("T", ctypes.c_double),
        ("dyn", srmdp_fn), ("driver", srmdp_fn), ("terminal", srmdp_fn),
        ("cells_per_dim", ctypes.c_int), ("L", ctypes.c_double), ("mu", ctypes.c_double),
        ("M", ctypes.c_int64),
        ("C_g", ctypes.c_double), ("C_f", ctypes.c_double), ("L_f", ctypes.c_double),
        ("C_y_override", ctypes.c_double), ("C_z_override", ctypes.c_double),
        ("seed", ctypes.c_uint64),
        ("rank", ctypes.c_int), ("world", ctypes.c_int), ("nccl_unique_id", ctypes.c_void_p),
        ("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("flags", ctypes.c_int),
        ("lp0", ctypes.c_int),
        ("grid", ctypes.c_int),
        ("user_src", ctypes.c_char_p), ("user_params", ctypes.POINTER(ctypes.c_double)),
        ("n_user_params", ctypes.c_int),
    ]


class srmdp_stats_t(ctypes.Structure):
    _fields_ = [
        ("solve_ms", ctypes.c_double), ("kernel_ms", ctypes.c_double), ("kernel_launches", ctypes.c_int),
        ("path_steps", ctypes.c_uint64), ("rank_path_steps", ctypes.c_uint64), ("lp0_fallbacks", ctypes.c_uint64),
        ("smallness_violated", ctypes.c_int), ("C_y", ctypes.c_double), ("C_z", ctypes.c_double),
        ("K", ctypes.c_int64), ("K_pad", ctypes.c_int64), ("chunk", ctypes.c_int64),
        ("k_begin", ctypes.c_int64), ("k_end", ctypes.c_int64), ("B", ctypes.c_int), ("B_pad", ctypes.c_int),
        ("grid", ctypes.c_int), ("block", ctypes.c_int), ("smem_bytes", ctypes.c_int), ("ctas_per_sm", ctypes.c_int),
        ("exact_z_evals", ctypes.c_uint64), ("exact_z_i", ctypes.c_uint64), ("gather_ms", ctypes.c_double),
    ]


class srmdp_plan_t(ctypes.Structure):
    _fields_ = [("L", ctypes.c_double), ("delta", ctypes.c_double), ("cells_per_dim", ctypes.c_int),
                ("K", ctypes.c_int64), ("M", ctypes.c_int64), ("B", ctypes.c_int), ("B_pad", ctypes.c_int),
                ("table_bytes", ctypes.c_double), ("path_steps", ctypes.c_double), ("path_starts", ctypes.c_double),
                ("fits", ctypes.c_int)]


_lib = None
_PD = ctypes.POINTER(ctypes.c_double)
_P64 = ctypes.POINTER(ctypes.c_int64)
_PU32 = ctypes.POINTER(ctypes.c_uint32)
_H = ctypes.c_void_p

# name -> (restype, argtypes): exactly the declarations of include/srmdp.h and srmdp_debug.h
SIGNATURES = {
    "srmdp_create": (ctypes.c_int, [ctypes.POINTER(srmdp_config), ctypes.POINTER(_H)]),
    "srmdp_solve": (ctypes.c_int, [_H]),
    "srmdp_solve_async": (ctypes.c_int, [_H]),
    "srmdp_wait": (ctypes.c_int, [_H]),
    "srmdp_coeffs": (ctypes.c_int, [_H, ctypes.c_int, ctypes.c_int, _PD, ctypes.c_size_t]),
    "srmdp_eval": (ctypes.c_int, [_H, ctypes.c_int, ctypes.c_size_t, _PD, _PD, _PD]),
    "srmdp_destroy": (None, [_H]),
    "srmdp_reseed": (ctypes.c_int, [_H, ctypes.c_uint64]),
    "srmdp_solve_steps": (ctypes.c_int, [_H, ctypes.c_int, ctypes.c_int]),
    "srmdp_table_save": (ctypes.c_int, [_H, ctypes.c_char_p]),
    "srmdp_table_load": (ctypes.c_int, [_H, ctypes.c_char_p]),
    "srmdp_step_ms": (ctypes.c_int, [_H, _PD, ctypes.c_int]),
    "srmdp_exchange_ms": (ctypes.c_int, [_H, _PD, ctypes.c_int]),
    "srmdp_last_error": (ctypes.c_char_p, [_H]),
    "srmdp_nccl_unique_id": (ctypes.c_int, [ctypes.c_void_p]),
    "srmdp_stats": (ctypes.c_int, [_H, ctypes.POINTER(srmdp_stats_t)]),
    "srmdp_shard_plan": (ctypes.c_int, [ctypes.c_int64, ctypes.c_int, ctypes.c_int, _P64]),
    "srmdp_build_info": (ctypes.c_char_p, []),
    "srmdp_plan": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                  ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.POINTER(srmdp_plan_t)]),
    "srmdp_jit_check": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t]),
    "srmdp_debug_trace": (ctypes.c_int, [_H, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _PD, _P64, _PD]),
    "srmdp_debug_step_dump": (ctypes.c_int, [_H, ctypes.c_int, ctypes.c_int, _PU32, _PD]),
    "srmdp_debug_detmath": (ctypes.c_int, [ctypes.c_int, ctypes.c_size_t, _PD, _PD, _PD]),
    "srmdp_debug_philox": (ctypes.c_int, [ctypes.c_size_t, _PU32, _PU32, _PU32]),
}


def library():
    """Load libsrmdp_b200.so (raises SrmdpError if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SrmdpError(-4, "CUDA library %s is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                             % LIB_PATH)
        L = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(st, h=None):
    if st != 0:
        msg = library().srmdp_last_error(h)
        raise SrmdpError(st, msg.decode() if msg else "")


def _dp(a):
    return a.ctypes.data_as(_PD)


def srmdp_build_info() -> str:
    return library().srmdp_build_info().decode()


def srmdp_last_error(h=None) -> str:
    return library().srmdp_last_error(h).decode()


def srmdp_jit_check(d: int, q: int, dyn: str, f: str, g: str, user_src: str | None = None):
    """NVRTC-compile the kernels of a user problem without a GPU. Returns
    (ok, log); see srmdp.h."""
    buf = ctypes.create_string_buffer(1 << 16)
    st = library().srmdp_jit_check(d, q, DYN[dyn], FKIND[f], GKIND[g],
                                   user_src.encode() if user_src is not None else None, buf, len(buf))
    if st == -1:
        raise SrmdpError(st, "d, q must be in 1..32")
    return st == 0, buf.value.decode()


def srmdp_plan(d: int, q: int, N: int, mu: float = 1.0, lp0: bool = False, c_delta: float = 0.0, c_M: float = 0.0,
               mem_bytes: float = 0.0) -> dict:
    """The paper's §4.3 parameter calibration (include/srmdp.h srmdp_plan); pure host arithmetic."""
    out = srmdp_plan_t()
    _check(library().srmdp_plan(d, q, N, mu, 1 if lp0 else 0, c_delta, c_M, mem_bytes, ctypes.byref(out)))
    return {name: getattr(out, name) for name, _ in srmdp_plan_t._fields_}


def srmdp_shard_plan(K: int, world: int, rank: int):
    out = (ctypes.c_int64 * 4)()
    _check(library().srmdp_shard_plan(K, world, rank, out))
    return tuple(int(v) for v in out)


def srmdp_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(library().srmdp_nccl_unique_id(buf))
    return buf.raw


def config_from_workload(w: dict, rank: int = 0, world: int = 1, device: int = 0, stream=None, flags: int = 0,
                         nccl_id: bytes | None = None):
    """Build an srmdp_config from a ``workloads`` dict. Returns (config, keepalive)."""
    keep = []

    def fn(kind, params):
        arr = np.ascontiguousarray(np.asarray(params if params is not None else [], dtype=np.float64).ravel())
        keep.append(arr)
        return srmdp_fn(kind, arr.size, _dp(arr) if arr.size else None)

    nan = float("nan")
    cfg = srmdp_config()
    cfg.d, cfg.q, cfg.N, cfg.T = int(w["d"]), int(w["q"]), int(w["N"]), float(w["T"])
    cfg.dyn = fn(DYN[w["dyn"]], w.get("dyn_params"))
    cfg.driver = fn(FKIND[w["f"]], w.get("f_params"))
    cfg.terminal = fn(GKIND[w["g"]], w.get("g_params"))
    cfg.cells_per_dim, cfg.L, cfg.mu = int(w["C"]), float(w["L"]), float(w["mu"])
    cfg.M = int(w["M"])
    cfg.C_g, cfg.C_f, cfg.L_f = float(w.get("C_g", 0.0)), float(w.get("C_f", 0.0)), float(w.get("L_f", 0.0))
    cy, cz = w.get("C_y_override"), w.get("C_z_override")
    cfg.C_y_override = nan if cy is None else float(cy)
    cfg.C_z_override = nan if cz is None else float(cz)
    cfg.seed = int(w["seed"]) & 0xFFFFFFFFFFFFFFFF
    cfg.rank, cfg.world, cfg.device, cfg.flags = rank, world, device, flags
    cfg.lp0 = 1 if w.get("basis", "lp1") == "lp0" else 0
    cfg.grid = 1 if w.get("grid", "uniform") == "equiprobable" else 0
    if w.get("user_src") is not None:          # user problem (srmdp.h, SRMDP_*_USER)
        src = ctypes.create_string_buffer(w["user_src"].encode())
        keep.append(src)
        cfg.user_src = ctypes.cast(src, ctypes.c_char_p)
    up = np.ascontiguousarray(np.asarray(w.get("user_params", []), dtype=np.float64).ravel())
    keep.append(up)
    cfg.n_user_params = int(up.size)
    cfg.user_params = _dp(up) if up.size else None
    if nccl_id is not None:
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
        keep.append(idbuf)
        cfg.nccl_unique_id = ctypes.cast(idbuf, ctypes.c_void_p)
    cfg.stream = stream
    return cfg, keep


def srmdp_create(cfg: srmdp_config):
    h = _H()
    st = library().srmdp_create(ctypes.byref(cfg), ctypes.byref(h))
    if st != 0:
        raise SrmdpError(st, srmdp_last_error(None))
    return h


def srmdp_solve(h):
    _check(library().srmdp_solve(h), h)


def srmdp_solve_async(h):
    _check(library().srmdp_solve_async(h), h)


def srmdp_wait(h):
    _check(library().srmdp_wait(h), h)


def srmdp_stats(h) -> dict:
    s = srmdp_stats_t()
    _check(library().srmdp_stats(h, ctypes.byref(s)), h)
    return {name: getattr(s, name) for name, _ in srmdp_stats_t._fields_}


def srmdp_coeffs(h, i: int, basis: int = 1, out: np.ndarray | None = None) -> np.ndarray:
    st = srmdp_stats(h)
    K, B = st["K"], st["B"]
    if out is None:
        out = np.empty((K, B), dtype=np.float64)
    assert out.dtype == np.float64 and out.flags.c_contiguous and out.size == K * B
    _check(library().srmdp_coeffs(h, i, basis, _dp(out), out.size), h)
    return out


def srmdp_eval(h, i: int, x: np.ndarray, d: int, q: int, want_z: bool = True):
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, d)
    n = x.shape[0]
    y = np.empty(n)
    z = np.empty((n, q)) if want_z else None
    _check(library().srmdp_eval(h, i, n, _dp(x), _dp(y), _dp(z) if want_z else None), h)
    return (y, z) if want_z else y


def srmdp_reseed(h, seed: int):
    _check(library().srmdp_reseed(h, int(seed) & 0xFFFFFFFFFFFFFFFF), h)


def srmdp_solve_steps(h, i_hi: int, i_lo: int):
    _check(library().srmdp_solve_steps(h, i_hi, i_lo), h)


def srmdp_table_save(h, path: str):
    _check(library().srmdp_table_save(h, os.fsencode(path)), h)


def srmdp_table_load(h, path: str):
    _check(library().srmdp_table_load(h, os.fsencode(path)), h)


def srmdp_step_ms(h, N: int) -> np.ndarray:
    out = np.zeros(N)
    _check(library().srmdp_step_ms(h, _dp(out), N), h)
    return out


def srmdp_exchange_ms(h, N: int) -> np.ndarray:
    out = np.zeros(N)
    _check(library().srmdp_exchange_ms(h, _dp(out), N), h)
    return out


def srmdp_destroy(h):
    if h:
        library().srmdp_destroy(h)


class Solver:
    """Convenience owner of one handle (create on construction, destroy on close)."""

    def __init__(self, w: dict, **kw):
        self.w = dict(w)
        self.cfg, self._keep = config_from_workload(w, **kw)
        self.h = srmdp_create(self.cfg)
        self.d, self.q, self.N = int(w["d"]), int(w["q"]), int(w["N"])

    def solve(self):
        srmdp_solve(self.h)
        return self

    def solve_async(self):
        srmdp_solve_async(self.h)
        return self

    def wait(self):
        srmdp_wait(self.h)
        return self

    def reseed(self, seed):
        srmdp_reseed(self.h, seed)
        return self

    def solve_steps(self, i_hi, i_lo):
        srmdp_solve_steps(self.h, i_hi, i_lo)
        return self

    def save(self, path):
        srmdp_table_save(self.h, path)

    def load(self, path):
        srmdp_table_load(self.h, path)
        return self

    def step_ms(self):
        return srmdp_step_ms(self.h, self.N)

    def exchange_ms(self):
        return srmdp_exchange_ms(self.h, self.N)

    def stats(self):
        return srmdp_stats(self.h)

    def coeffs(self, i, basis=1, out=None):
        return srmdp_coeffs(self.h, i, basis, out)

    def table(self, basis=1):
        return np.stack([self.coeffs(i, basis) for i in range(self.N)])

    def eval(self, i, x, want_z=True):
        return srmdp_eval(self.h, i, x, self.d, self.q, want_z and i < self.N)

    def trace(self, i, k, m0, n):
        steps = self.N - i
        x = np.empty((n, steps + 1, self.d))
        c = np.empty((n, steps + 1), dtype=np.int64)
        w = np.empty((n, steps, self.q))
        _check(library().srmdp_debug_trace(self.h, i, k, m0, n, _dp(x), c.ctypes.data_as(_P64), _dp(w)), self.h)
        return x, c, w

    def step_dump(self, i, dump_m):
        """srmdp_debug_step_dump: cells[kl][m][N-i-1], x[kl][m][N-i][d] as the step kernel located them."""
        st = srmdp_stats(self.h)
        nk, steps = st["k_end"] - st["k_begin"], self.N - i
        c = np.zeros((nk, dump_m, steps - 1), dtype=np.uint32)
        x = np.empty((nk, dump_m, steps, self.d))
        _check(library().srmdp_debug_step_dump(self.h, i, dump_m, c.ctypes.data_as(_PU32), _dp(x)), self.h)
        return c, x

    def close(self):
        srmdp_destroy(self.h)
        self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            if self.h:
                self.close()
        except Exception:
            pass


def debug_detmath(op: int, x: np.ndarray):
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    o0 = np.empty_like(x)
    o1 = np.empty_like(x)
    _check(library().srmdp_debug_detmath(op, x.size, _dp(x), _dp(o0), _dp(o1)))
    return (o0, o1) if op == 1 else o0


def debug_philox(ctr: np.ndarray, key):
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32).ravel())
    out = np.empty_like(ctr)
    _check(library().srmdp_debug_philox(ctr.shape[0], ctr.ctypes.data_as(_PU32), k.ctypes.data_as(_PU32),
                                        out.ctypes.data_as(_PU32)))
    return out


def inf_or(x):
    return math.inf if x is None else x
