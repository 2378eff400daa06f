"""C-ABI checks that need no GPU: the library builds for sm_100a, loads, and
exports every symbol include/*.h declares; the pure-host shard planner
(docs/layout.md) tiles the cell range."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for f in os.listdir(os.path.join(ROOT, "include")):
        src = open(os.path.join(ROOT, "include", f)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(srmdp_\w+)\s*\(", src))
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_2407_21085_b200 import build
    build.build()
    from paper_2407_21085_b200 import srmdp
    return srmdp


def test_header_declares_the_boundary():
    names = declared_symbols()
    for n in ("srmdp_create", "srmdp_solve", "srmdp_coeffs", "srmdp_eval", "srmdp_destroy",
              "srmdp_stats", "srmdp_nccl_unique_id", "srmdp_shard_plan", "srmdp_debug_trace"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    so = lib.library()
    for n in declared_symbols():
        assert hasattr(so, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(srmdp_\w+)$", out, flags=re.M))
    assert declared_symbols() <= exported
    # the binding declares exactly the header's functions
    assert set(lib.SIGNATURES) == declared_symbols()


def test_built_for_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_100a" in lib.srmdp_build_info()


@pytest.mark.parametrize("K,world", [(1, 1), (10, 1), (10, 3), (15625, 8), (7, 8), (524288, 8)])
def test_shard_plan_tiles_cells(lib, K, world):
    ranges = [lib.srmdp_shard_plan(K, world, r) for r in range(world)]
    chunk, K_pad = ranges[0][2], ranges[0][3]
    assert K_pad == chunk * world and K_pad >= K and K_pad - K < world
    pos = 0
    for r, (b, e, c, kp) in enumerate(ranges):
        assert (c, kp) == (chunk, K_pad)
        assert b == min(r * chunk, K) and e == min((r + 1) * chunk, K)
        assert b == pos or (b == K and e == K)
        pos = e
    assert pos == K


def test_shard_plan_rejects_bad_args(lib):
    with pytest.raises(lib.SrmdpError):
        lib.srmdp_shard_plan(0, 1, 0)
    with pytest.raises(lib.SrmdpError):
        lib.srmdp_shard_plan(10, 2, 2)


def test_product_does_not_import_oracle():
    """The product package never references the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2407_21085_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "srmdp_oracle" not in src and "or_solve" not in src, f


def test_create_validation_needs_no_gpu(lib):
    """srmdp_create validates the configuration before touching CUDA, so every
    rejection is testable on the CPU: status codes and messages (srmdp.h)."""
    import workloads
    base = workloads.benchmark(d=2, N=3, C=3, M=10)
    cases = [
        (dict(base, d=0, q=0), -1, "d and q"),
        (dict(base, N=0), -1, "N must"),
        (dict(base, T=0.0), -1, "T must"),
        (dict(base, C=0), -1, "cells_per_dim"),
        (dict(base, L=-1.0), -1, "L must"),
        (dict(base, mu=0.0), -1, "mu must"),
        (dict(base, M=2), -2, "M < d+1"),
        (dict(base, C=3000), -7, "cells_per_dim > 2048"),
        (dict(base, N=1 << 24), -7, "N >= 2^24"),
        (dict(base, d=33, q=33, C=1, M=40), -7, "d, q <= 32"),
        (dict(base, d=8, q=8, C=16, M=20), -7, "K = C^d"),
        (dict(base, dyn="gbm", dyn_params=[0.1, 0.1, 0.2, 0.2], q=3), -1, "q == d"),
        (dict(base, dyn="affine", dyn_params=[0.0]), -1, "parameter count"),
        (dict(base, dyn="user"), -1, "user_src"),
    ]
    for w, status, msg in cases:
        with pytest.raises(lib.SrmdpError) as e:
            lib.Solver(w)
        assert e.value.status == status, (w, e.value)
        assert msg in str(e.value), (msg, str(e.value))
    with pytest.raises(lib.SrmdpError) as e:           # world > 1 needs the NCCL id
        lib.Solver(base, world=2, rank=0)
    assert e.value.status == -1 and "nccl_unique_id" in str(e.value)
    with pytest.raises(lib.SrmdpError) as e:
        lib.Solver(base, world=2, rank=2, nccl_id=b"x" * 128)
    assert e.value.status == -1
    with pytest.raises(lib.SrmdpError) as e:           # P2P exchange excludes loopback
        lib.Solver(base, world=2, flags=lib.FLAG_LOOPBACK | lib.FLAG_P2P_EXCHANGE)
    assert e.value.status == -1


def test_exchange_flag_validation_needs_no_gpu(lib):
    """The fused-exchange modes reject inconsistent flag sets before any CUDA
    call (include/srmdp.h: P2P_SELF_PEER is a world == 1 test mode of
    P2P_EXCHANGE; NVLS_EXCHANGE excludes LOOPBACK and P2P_EXCHANGE)."""
    import workloads
    base = workloads.benchmark(d=2, N=3, C=3, M=10)
    for flags, world, msg in ((lib.FLAG_P2P_SELF_PEER, 1, "P2P_SELF_PEER"),
                              (lib.FLAG_P2P_EXCHANGE | lib.FLAG_P2P_SELF_PEER, 2, "P2P_SELF_PEER"),
                              (lib.FLAG_NVLS_EXCHANGE | lib.FLAG_P2P_EXCHANGE, 1, "NVLS_EXCHANGE"),
                              (lib.FLAG_NVLS_EXCHANGE | lib.FLAG_LOOPBACK, 2, "NVLS_EXCHANGE")):
        with pytest.raises(lib.SrmdpError) as e:
            lib.Solver(base, world=world, rank=0, flags=flags, nccl_id=b"x" * 128 if world > 1 else None)
        assert e.value.status == -1 and msg in str(e.value), (flags, str(e.value))


def test_plan_follows_the_papers_calibration(lib):
    """srmdp_plan (§4.3) is host arithmetic: L = log(N)/mu,
    delta = N^{-1/4} (LP1) / N^{-1/2} (LP0), #C = ceil(2L/delta),
    M = (d+1) N^2 (LP1) / N^2 (LP0); the cost exponents of P:836-847
    (K M N^2 ~ N^{4 + d/4} for LP1) follow from them."""
    import math
    p = lib.srmdp_plan(4, 4, 20, 1.0)
    assert abs(p["L"] - math.log(20)) < 1e-15
    assert abs(p["delta"] - 20 ** -0.25) < 1e-15
    assert p["cells_per_dim"] == math.ceil(2 * math.log(20) / 20 ** -0.25)
    assert p["K"] == p["cells_per_dim"] ** 4 and p["M"] == 5 * 400
    assert p["B"] == 25 and p["B_pad"] == 48
    assert p["path_steps"] == p["K"] * p["M"] * 20 * 21 / 2 and p["fits"] == 1
    q = lib.srmdp_plan(4, 4, 20, 2.0, lp0=True, c_delta=0.5, c_M=2.0, mem_bytes=1e3)
    assert abs(q["L"] - math.log(20) / 2) < 1e-15 and abs(q["delta"] - 0.5 / math.sqrt(20)) < 1e-15
    assert q["M"] == 800 and q["fits"] == 0
    # LP1 cost exponent: K M N(N+1)/2 grows like N^{4 + d/4} (up to the log terms of L and ceil)
    for d in (2, 4, 8):
        a, b = lib.srmdp_plan(d, d, 400, 1.0), lib.srmdp_plan(d, d, 6400, 1.0)
        slope = math.log(b["path_steps"] / a["path_steps"]) / math.log(16)
        logs = d * math.log(math.log(6400) / math.log(400)) / math.log(16)   # the (log N)^d of K
        assert abs(slope - logs - (4 + d / 4)) < 0.1 * d / 4 + 0.05, (d, slope)
    with pytest.raises(lib.SrmdpError):
        lib.srmdp_plan(0, 1, 10, 1.0)
