"""World-size-2 exchange protocol on CPU (gloo), no GPU.

Each rank takes its cell range from the PRODUCT's shard planner
(srmdp_shard_plan, docs/layout.md), computes those cells of every time step
with the oracle, and all-gathers the slice after every step exactly as the
library does with ncclAllGather (fixed-size padded chunks, rank order). The
reassembled table must be bit-identical to a single-process sweep: the
per-cell arithmetic and the exchange do not depend on the partition
(SURVEY §8(e) determinism), and a wrong offset / chunk / padding breaks it.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, wl, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import oracle
    from paper_2407_21085_b200 import srmdp

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P = oracle.Problem(wl)
        kb, ke, chunk, K_pad = srmdp.srmdp_shard_plan(P.K, world, rank)
        # table with the library's padded slice layout [N][K_pad][B]
        tab = np.zeros((wl["N"], K_pad, P.B))
        for i in range(wl["N"] - 1, -1, -1):
            work = tab[:, :P.K, :].copy()            # oracle indexes cells 0..K-1
            if ke > kb:
                P.step(work, i, kb, ke)
            tab[:, :P.K, :] = work
            mine = torch.from_numpy(np.ascontiguousarray(tab[i, rank * chunk:(rank + 1) * chunk]))
            parts = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(parts, mine)
            tab[i] = torch.cat(parts).numpy()
        # max-over-ranks reduction as bench.py does for times
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == world
        if rank == 0:
            np.save(out, tab[:, :P.K, :])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("wl", [workloads.cfg2(N=4, C=5, M=48), workloads.benchmark(d=3, N=3, C=3, M=40, seed=4)],
                         ids=["cfg2-K25", "bench-d3-K27"])
def test_two_rank_exchange_matches_single_process(orc, tmp_path, wl):
    from paper_2407_21085_b200 import build
    build.build()
    out = str(tmp_path / "t.npy")
    mp.start_processes(_worker, args=(2, _free_port(), wl, out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    ref, _ = orc.Problem(wl).solve()
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))
