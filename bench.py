"""bench.py — SRMDP backward-sweep throughput on B200 (one JSON line on rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl srmdp|reference] [--config cfg4]

A "step" is one full SRMDP solve (Alg. srmdp: all N time
points, every hypercube, every path) of the synthetic workload (default cfg4 =
BASELINE.json configs[3]: §5.1 benchmark d=q=6, N=30, #C=5 -> K=15625, M=4096).
metric = simulated path-steps/s = K*M*N(N+1)/2 per solve / seconds.

Timing: W warm-up solves, then K solves each bracketed by CUDA events on the
library's stream, L2 flushed (256 MB write) before every timed solve outside
the events; barrier + synchronize on both sides; max over ranks. For N>1 the
driver launches this under torchrun; the library shards cells over ranks and
all-gathers every step's coefficients with NCCL (strong scaling of a fixed
problem). `--impl reference` times the CPU oracle (test infrastructure) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads  # noqa: E402


# ----------------------------------------------------------------------------
# algorithmic FP64 work per unit: the per-unit model of SURVEY.md §8(d)
# (DESIGN.md §5): per path-step q normals at F_norm = 33 flop, the Euler step,
# locate + centering (3d), the evaluation of y and the q components of z
# (2(q+1)(d+1)) and the driver; per path-start the inverse CDFs (31 d), Gram,
# Z / Y right-hand sides, the pass-2 z_i and g. It is the method's work, not
# the kernel's executed instruction count (the kernel evaluates sum_l w_l z_l
# through a certified contraction and fewer flops; ncu FP64-pipe utilisation
# is reported separately in profiles/).
# ----------------------------------------------------------------------------
F_NORM = 33


def flops_per_path_step(w):
    d, q = w["d"], w["q"]
    euler = {"bm": d, "gbm": 4 * d, "gbm_exact": 30 * d, "affine": d * (2 * d + 2 * q + 2)}[w["dyn"]]
    f_f = {"zero": 0, "linear": q + 3, "paper": q + 4}[w["f"]]
    return q * F_NORM + euler + 3 * d + 2 * (q + 1) * (d + 1) + f_f + 2


def flops_per_path_start(w):
    d, q = w["d"], w["q"]
    f_g = d + 3
    return 31 * d + (d + 1) * (d + 2) + 4 * q * (d + 1) + 2 * (d + 1) + 3 * q + f_g


def algorithmic_flops(w):
    K = w["C"] ** w["d"]
    steps = K * w["M"] * w["N"] * (w["N"] + 1) // 2
    starts = K * w["M"] * w["N"]
    return flops_per_path_step(w) * steps + flops_per_path_start(w) * starts


def fp64_peak():
    """Roofline denominator of the ALU-bound step kernel: MEASURED_PEAKS.json
    if it ever carries an FP64 entry, else the peak derived from unit counts and
    the max clock (148 SM x 64 FP64 FMA/clk x 2 flop x 1.965 GHz
    = 37.2 TFLOP/s). Returns (peak, source, measured DFMA microbenchmark or None)."""
    measured = None
    try:
        m = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))
        measured = float(m["fp64_tflops_sustained"])
    except Exception:
        pass
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        for k in ("fp64_tflops_sustained", "fp64_tflops"):
            if k in mp:
                return float(mp[k]), "MEASURED_PEAKS.json:" + k, measured
    except Exception:
        pass
    return (148 * 64 * 2 * 1.965e9 / 1e12, "derived (DESIGN.md §5): 148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz",
            measured)


def gather_block(w, path_steps_per_s):
    """Secondary roofline: the per-lane coefficient gather through L1/L2. Bytes
    per path-step = the hot part [beta^Y | W | S] read with 256-bit loads
    (2(d+1)+1 doubles rounded up to 32 B); ceilings from tools/gather_bw.cu
    (profiles/gather_bw.json: random lanes and warp-local lanes, same
    occupancy). Context for the ALU roofline, not the headline."""
    nhot = 2 * (w["d"] + 1) + 1
    bps = ((nhot * 8 + 31) // 32) * 32
    out = {"bytes_per_path_step": bps, "achieved_GBps": path_steps_per_s * bps / 1e9}
    try:
        g = json.load(open(os.path.join(ROOT, "profiles", "gather_bw.json")))
        out["ceiling_random_lanes_GBps"] = g["random_ldg256"]["GB_per_s"]
        out["ceiling_warp_local_GBps"] = g["local_ldg256"]["GB_per_s"]
        out["source"] = "profiles/gather_bw.json (tools/gather_bw.cu)"
    except Exception:
        pass
    return out


def ncu_traffic(name="cfg4"):
    """ncu DRAM / L2 bytes of one captured step-kernel launch of workload
    `name` (profiles/step_kernel_traffic*.json, from `ncu --set full`)."""
    fn = "step_kernel_traffic.json" if name == "cfg4" else "step_kernel_traffic_%s.json" % name
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", fn)))
        return t if t.get("launch", "").startswith(name + ",") else None
    except Exception:
        return None


def executed_flops(name):
    """FP64 flops the step kernels EXECUTE per solve, counted by ncu over every
    launch of one solve (profiles/executed_flops.json: DFMA x 2 + DMUL + DADD
    thread instructions + DMMA m8n8k4 x 512 per warp instruction), next to the
    method's algorithmic count -- the certified contraction evaluates fewer
    flops than the model credits."""
    try:
        e = json.load(open(os.path.join(ROOT, "profiles", "executed_flops.json")))
        return e.get(name)
    except Exception:
        return None


# ----------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap", "power.draw"]

    def __init__(self, device_index):
        self.dev = device_index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for s in self.samples for j in range(4) if s[2 + j].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------
def cpu_baseline(w, target_path_steps=2.0e8):
    """The oracle (as it stands) on a bounded sample of the same workload:
    every time step i = N-1..0 on the cells k = 0, s, 2s, ... (s chosen so
    the sample has ~target path-steps), all host cores (OpenMP)."""
    import oracle
    P = oracle.Problem(w)
    total = workloads.path_steps(w)
    stride = max(1, int(math.ceil(total / target_path_steps)))
    ncell = (P.K + stride - 1) // stride
    tab = P.new_table()
    t0 = time.perf_counter()
    for i in range(w["N"] - 1, -1, -1):
        P.step(tab, i, 0, P.K, stride)
    dt = time.perf_counter() - t0
    sample_steps = ncell * w["M"] * w["N"] * (w["N"] + 1) // 2
    return {"value": sample_steps / dt, "unit": "path-steps/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": "%s: all %d time steps on %d of %d cells (stride %d), M=%d: %.3g path-steps in %.1f s" % (
                w["name"], w["N"], ncell, P.K, stride, w["M"], sample_steps, dt)}


def run_reference(args, w, rank):
    if rank != 0:
        return 0
    K, W = args.steps, args.warmup
    vals = []
    base = None
    for s in range(W + K):
        r = cpu_baseline(w, target_path_steps=args.ref_path_steps)
        if s >= W:
            vals.append(r["value"])
            base = r
    v = float(np.median(vals))
    base["value"] = v
    line = {"impl": "reference", "metric": "simulated path-steps/sec per SRMDP solve", "value": v,
            "unit": "path-steps/s", "n_gpus": args.gpus, "steps": K, "warmup": W,
            "ms_per_step": workloads.path_steps(w) / v * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(w, args), "cpu_baseline": base,
            "e2e": {"value": v, "unit": "path-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)
    return 0


def run_secondary(w, args, rank, world, local, dev, stream, fresh_nccl_id, barrier, flush, xflag, steps):
    """BASELINE configs[4] (cfg5: §5.1 benchmark d = q = 19, N = 5, 2^19 cells,
    M = 3200 -- the paper's largest row), measured in the same
    run with the same timing rules: 1 warm-up, `steps` timed solves with L2
    flushed, CUDA events on the library's stream, clocks sampled, max over
    ranks. Its roofline: FP64 (credited and executed flops) and HBM (ncu DRAM
    bytes of a captured launch; the 1.68 GB slices exceed L2)."""
    import torch
    import torch.distributed as dist
    from paper_2407_21085_b200 import srmdp
    solver = srmdp.Solver(w, rank=rank, world=world, device=local, stream=stream.cuda_stream,
                          flags=srmdp.FLAG_TIME_KERNELS | xflag, nccl_id=fresh_nccl_id())
    solver.solve()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    kms = []
    with ClockSampler(local) as clk:
        barrier()
        for s in range(steps):
            flush.fill_(float(s))
            ev[s][0].record(stream)
            solver.solve_async()
            ev[s][1].record(stream)
            solver.wait()
            kms.append(solver.stats()["kernel_ms"])
        barrier()
    tot = float(sum(a.elapsed_time(b) for a, b in ev))
    kern = float(sum(kms))
    if world > 1:
        t = torch.tensor([tot, kern], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot, kern = float(t[0]), float(t[1])
    st = solver.stats()
    solver.close()
    value = st["path_steps"] * steps / (tot / 1e3)
    peak, _, peak_meas = fp64_peak()
    achieved = algorithmic_flops(w) / world * steps / (kern / 1e3) / 1e12
    ex = executed_flops(w["name"])
    ex_tf = (ex["flop_per_solve"] / world * steps / (kern / 1e3) / 1e12) if ex else None
    tr = ncu_traffic(w["name"])
    hbm = None
    if tr:
        gbps = tr["dram_bytes_per_launch"] / (tr["duration_ms_ncu"] / 1e3) / 1e9
        hbm_peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
            if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6545.6
        hbm = {"dram_GBps_ncu_launch": gbps, "peak_GBps": hbm_peak, "frac": gbps / hbm_peak,
               "lts_GBps_ncu_launch": tr.get("lts_bytes_per_launch", 0) / (tr["duration_ms_ncu"] / 1e3) / 1e9
               if tr.get("lts_bytes_per_launch") else None,
               "launch": tr["launch"], "source": tr.get("source")}
    return {"workload": w["name"], "d": w["d"], "q": w["q"], "N": w["N"], "K": w["C"] ** w["d"], "M": w["M"],
            "path_steps_per_solve": st["path_steps"], "value": value, "unit": "path-steps/s", "steps": steps,
            "warmup": 1, "ms_per_step": tot / steps, "kernel_share_of_step": kern / tot,
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "frac_of_measured_dfma": (achieved / peak_meas) if peak_meas else None,
                         "executed_tflops": ex_tf, "executed_frac": (ex_tf / peak) if ex_tf else None,
                         "flops_per_path_step": flops_per_path_step(w), "flops_per_path_start": flops_per_path_start(w)},
            "hbm": hbm, "gather": gather_block(w, value), "clocks": clk.summary(),
            # the same workload in the paper (table:LP1d15_19: d = 19, N = 5, #C = 2, M = 3200):
            # 4370.31 s on a GTX TITAN Black in fp32 -> 5.76e6 path-steps/s (context,
            # other hardware and precision)
            "paper_context": {"line": "PAPER.md:1259", "gpu": "GeForce GTX TITAN Black (Kepler), fp32",
                              "seconds": 4370.31, "path_steps_per_s": 5.76e6,
                              "ratio": value / 5.76e6 if (w["d"], w["N"], w["C"], w["M"]) == (19, 5, 2, 3200) else None},
            "lp0_fallbacks": st["lp0_fallbacks"],
            "launch": {"grid": st["grid"], "block": st["block"], "smem_bytes": st["smem_bytes"],
                       "ctas_per_sm": st["ctas_per_sm"]}}


def config_block(w, args):
    return {"workload": w["name"], "d": w["d"], "q": w["q"], "N": w["N"], "cells_per_dim": w["C"],
            "K": w["C"] ** w["d"], "M": w["M"], "problem": "PAPER.md §5.1 benchmark (X=W, mu=1, T=1, L=6.5)"
            if w["f"] == "paper" else w["name"], "path_steps_per_solve": workloads.path_steps(w),
            "parallelism": "cells sharded over %d GPU(s), %s per time step" % (
                args.gpus, {"p2p": "fused NVLink-store exchange", "nvls": "NVLS multicast-store exchange"}.get(
                    getattr(args, "exchange", "nccl"), "ncclAllGather")),
            "l2": "flushed (256 MB write) before every timed solve"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="srmdp", choices=["srmdp", "reference"])
    ap.add_argument("--config", default="cfg4", choices=sorted(workloads.CONFIGS))
    ap.add_argument("--M", type=int, default=None)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p", "nvls"],
                    help="per-step slice exchange for N > 1: in-place ncclAllGather (default), the fused "
                         "NVLink store epilogue (SRMDP_FLAG_P2P_EXCHANGE) or the NVLS multicast store epilogue "
                         "(SRMDP_FLAG_NVLS_EXCHANGE)")
    ap.add_argument("--ref-path-steps", type=float, default=2.0e8)
    ap.add_argument("--no-cfg5", action="store_true", help="skip the secondary cfg5 (d = 19) block")
    ap.add_argument("--cfg5-steps", type=int, default=2)
    ap.add_argument("--e2e-mode", default="auto", choices=["auto", "create", "reseed"],
                    help="e2e step: a fresh handle (create) or srmdp_reseed on one handle (reseed); "
                         "auto = create at N = 1, reseed at N > 1")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    kw = {"seed": args.seed}
    if args.M:
        kw["M"] = args.M
    w = workloads.CONFIGS[args.config](**kw)
    if args.impl == "reference":
        return run_reference(args, w, rank)

    import torch
    import torch.distributed as dist
    from paper_2407_21085_b200 import srmdp

    torch.cuda.set_device(local)
    if world > 1 and "NCCL_DEBUG" not in os.environ:
        # NCCL's init log (ranks, NVLink / NVLS transport) on stderr, readable next to the JSON line
        os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT", NCCL_DEBUG_FILE="/dev/stderr")
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    # a dedicated (non-default) stream: the library, the L2 flush and the timing
    # events all run on it, so the events bracket exactly the solve's kernels
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    srmdp.library()

    def fresh_nccl_id():
        """A new ncclUniqueId per communicator (rank 0 creates, torch.distributed broadcasts)."""
        if world == 1:
            return None
        obj = [srmdp.srmdp_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    nccl_id = fresh_nccl_id()

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()

    xflag = {"nccl": 0, "p2p": srmdp.FLAG_P2P_EXCHANGE, "nvls": srmdp.FLAG_NVLS_EXCHANGE}[args.exchange]
    solver = srmdp.Solver(w, rank=rank, world=world, device=local, stream=stream.cuda_stream,
                          flags=srmdp.FLAG_TIME_KERNELS | xflag, nccl_id=nccl_id)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    for _ in range(args.warmup):
        solver.solve()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kernel_ms = []
    with ClockSampler(local) as clk:
        barrier()
        for s in range(args.steps):
            flush.fill_(float(s))                     # on `stream` (current stream)
            ev[s][0].record(stream)
            solver.solve_async()          # one graph launch on `stream`, no host gap inside the events
            ev[s][1].record(stream)
            solver.wait()
            kernel_ms.append(solver.stats()["kernel_ms"])
        barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(step_ms))
    kern_ms = float(sum(kernel_ms))
    if world > 1:
        t = torch.tensor([total_ms, kern_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, kern_ms = float(t[0]), float(t[1])
    st = solver.stats()
    path_steps = st["path_steps"]
    value = path_steps * args.steps / (total_ms / 1e3)

    # dominant kernel roofline: the fused step kernel (N launches per solve)
    peak, peak_src, peak_meas = fp64_peak()
    flops = algorithmic_flops(w) / world         # per rank per solve
    launches_per_solve = st["kernel_launches"]
    achieved = flops * args.steps / (kern_ms / 1e3) / 1e12
    traffic = ncu_traffic(w["name"])
    ex = executed_flops(w["name"])
    ex_tf = (ex["flop_per_solve"] / world * args.steps / (kern_ms / 1e3) / 1e12) if ex else None
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            # ncu DRAM bytes per launch of this workload's captured launch (profiles/), else null
            "traffic": (traffic or {}).get("dram_bytes_per_launch"),
            "executed_tflops": ex_tf, "executed_frac": (ex_tf / peak) if ex_tf else None,
            "executed_source": ex.get("source") if ex else None,
            "kernel": "srk::step_kernel<%d,%d>" % (w["d"], w["q"]),
            "peak_source": peak_src,
            "peak_measured_dfma": peak_meas, "frac_of_measured_dfma": (achieved / peak_meas) if peak_meas else None,
            "flops_per_path_step": flops_per_path_step(w),
            "flops_per_path_start": flops_per_path_start(w),
            "kernel_share_of_step": kern_ms / total_ms, "avg_launch_ms": kern_ms / (args.steps * max(1, launches_per_solve))}
    gather_ms = float(st["gather_ms"]) if world > 1 or args.exchange != "nccl" else 0.0   # the last timed solve's exchange (srmdp_stats: per solve)
    solver.close()

    secondary = None
    if args.config == "cfg4" and not args.no_cfg5:
        secondary = run_secondary(workloads.cfg5(seed=args.seed), args, rank, world, local, dev, stream,
                                  fresh_nccl_id, barrier, flush, xflag, steps=args.cfg5_steps)

    # e2e: the user's call sequence through the C ABI with host buffers:
    # create (uploads parameters) -> solve -> coeffs of every slice to pinned host memory -> destroy
    host = torch.empty((w["N"], st["K"], st["B"]), dtype=torch.float64).pin_memory()
    hnp = host.numpy()
    # N = 1: every step is a fresh handle (create uploads the problem, destroy
    # frees). N > 1: one handle (its NCCL communicator is set up once, as a
    # serving process would), every step a new seed -- srmdp_reseed -- then
    # solve and the coefficient download.
    e2e_times = []
    persistent = None
    reseed_mode = args.e2e_mode == "reseed" or (args.e2e_mode == "auto" and world > 1)
    if reseed_mode:
        persistent = srmdp.Solver(w, rank=rank, world=world, device=local, stream=stream.cuda_stream,
                                  flags=xflag, nccl_id=fresh_nccl_id())
    for s in range(1 + args.steps):
        barrier()
        t0 = time.perf_counter()
        if persistent is None:
            sv = srmdp.Solver(w, rank=rank, world=world, device=local, stream=stream.cuda_stream,
                              flags=xflag, nccl_id=None)
        else:
            sv = persistent.reseed(args.seed + 1000 + s)
        sv.solve()
        for i in range(w["N"]):
            sv.coeffs(i, 1, hnp[i])
        if persistent is None:
            sv.close()
        barrier()
        if s > 0:
            e2e_times.append(time.perf_counter() - t0)
    if persistent is not None:
        persistent.close()
    e2e_s = float(sum(e2e_times))
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t[0])
    n_par = len(w.get("dyn_params", [])) + len(w.get("f_params", [])) + len(w.get("g_params", []))
    h2d = 8 * (n_par + 3 * w["C"] + 2) if not reseed_mode else 8     # problem upload, or the new seed
    d2h = 8 * w["N"] * st["K"] * st["B"]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w)

    if rank == 0:
        line = {
            "metric": "simulated path-steps/sec per SRMDP solve", "value": value, "unit": "path-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Philox clouds of the §5.1 benchmark; no dataset)",
            "config": config_block(w, args),
            "roofline": roof,
            "gather": gather_block(w, path_steps * args.steps / (total_ms / 1e3)),
            "cpu_baseline": cpu,
            "e2e": {"value": path_steps * args.steps / e2e_s, "unit": "path-steps/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "calls": "srmdp_create+srmdp_solve+srmdp_coeffs(all i, pinned host)+srmdp_destroy"
                    if not reseed_mode else "srmdp_reseed+srmdp_solve+srmdp_coeffs(all i, pinned host) on one handle per rank"},
            # step kernels + (fused exchange) the epoch / entry-barrier kernels and a signal + wait per slice
            "gpu_launches": (launches_per_solve + ((3 + 2 * w["N"]) if args.exchange in ("p2p", "nvls") else 0)) * args.steps,
            "clocks": clk.summary(),
            "lp0_fallbacks": st["lp0_fallbacks"],
            "exchange_ms_per_solve": gather_ms,
            "cfg5": secondary,
            "launch": {"grid": st["grid"], "block": st["block"], "smem_bytes": st["smem_bytes"],
                       "ctas_per_sm": st["ctas_per_sm"]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
