"""bench.py's roofline accounting (host arithmetic, no GPU): the SURVEY §8(d)
per-unit flop model, the units per solve, and the measured evidence files it
reads (executed FP64 flops, ncu traffic) -- so the JSON line's `achieved`,
`executed_tflops` and `hbm` fields are what DESIGN.md §5 / §10 state."""
import json
import os

import pytest

import bench
import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_flop_model_of_the_bench_workloads():
    w4, w5 = workloads.cfg4(), workloads.cfg5()
    # F_step = 33 q + F_euler + 3 d + 2 (q+1)(d+1) + F_f + 2, F_euler = d (BM), F_f = q + 4
    assert bench.flops_per_path_step(w4) == 33 * 6 + 6 + 18 + 2 * 7 * 7 + 10 + 2 == 332
    assert bench.flops_per_path_step(w5) == 33 * 19 + 19 + 57 + 2 * 20 * 20 + 23 + 2 == 1528
    # per path start: 31 d + (d+1)(d+2) + 4 q (d+1) + 2 (d+1) + 3 q + (d+3)
    assert bench.flops_per_path_start(w4) == 186 + 56 + 168 + 14 + 18 + 9 == 451
    steps = 15625 * 4096 * 30 * 31 // 2
    assert workloads.path_steps(w4) == steps == 29760000000
    assert bench.algorithmic_flops(w4) == 332 * steps + 451 * 15625 * 4096 * 30
    assert abs(bench.algorithmic_flops(w4) - 1.075e13) / 1.075e13 < 1e-3


def test_fp64_peak_is_the_derived_one():
    peak, src, measured = bench.fp64_peak()
    assert abs(peak - 148 * 64 * 2 * 1.965e9 / 1e12) < 1e-9 and "derived" in src
    assert measured is None or 30 < measured < peak


@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_executed_flops_evidence(name):
    """profiles/executed_flops.json: ncu counts over every launch of one solve,
    fewer than the model credits (the certified contraction skips the
    q-component z evaluation) and at least the DMMA Gram."""
    e = bench.executed_flops(name)
    assert e is not None and e["launches"] == workloads.CONFIGS[name]()["N"]
    flop = 2 * e["dfma"] + e["dmul"] + e["dadd"] + 512 * e["dmma_warp_inst"]
    assert abs(flop - e["flop_per_solve"]) < 1e-6 * flop
    model = bench.algorithmic_flops(workloads.CONFIGS[name]())
    assert 0.5 * model < e["flop_per_solve"] < model


@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_traffic_evidence(name):
    t = bench.ncu_traffic(name)
    assert t is not None and t["launch"].startswith(name + ",")
    assert t["dram_bytes_per_launch"] == pytest.approx(t["dram_bytes_read"] + t["dram_bytes_write"])
    assert os.path.exists(os.path.join(ROOT, t["source"].split()[0]))
