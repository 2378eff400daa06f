"""Schedule check of the fused exchange's flag protocol (SRMDP_FLAG_P2P_EXCHANGE,
csrc/exchange_kernels.cuh, srmdp.cu enqueue_sweep) under random interleavings
of P ranks. Each rank runs exactly the stream-ordered sequence enqueue_sweep
enqueues:

  epoch++ ; signal(slot N) ; wait(slot N) ;
  for i = N-1 .. 0:  step i (reads slices > i of its own table, stores its
                     blocks of slice i into every rank's table) ;
                     signal(slot i) ; wait(slot i)

between solves the host may read its own table (srmdp_coeffs). signal stores
the epoch into every rank's flags[slot][me]; wait spins until all
flags[slot][*] >= epoch. Checked: a step never reads a slice some rank has not
finished writing in this solve, the host never reads a slice that a peer is
rewriting for the next solve, and every schedule terminates. (This checks the
protocol the CUDA code implements; the one-GPU parity test runs the kernels.)
"""
import random

import pytest


def run(P, N, solves, seed):
    rnd = random.Random(seed)
    flags = [[[0] * P for _ in range(N + 1)] for _ in range(P)]   # flags[owner][slot][writer]
    table = [[(0, -1)] * N for _ in range(P)]                      # table[owner][slice] = (epoch, writers bitmask)
    progs = []
    for r in range(P):
        ops = []
        for e in range(1, solves + 1):
            ops += [("host_read", e - 1), ("signal", N, e), ("wait", N, e)]
            for i in range(N - 1, -1, -1):
                ops += [("step", i, e), ("signal", i, e), ("wait", i, e)]
        ops.append(("host_read", solves))
        progs.append(ops)
    pc = [0] * P
    partial = {}                    # (owner, slice, epoch) -> set of writers done
    steps = 0
    while any(pc[r] < len(progs[r]) for r in range(P)):
        ready = []
        for r in range(P):
            if pc[r] >= len(progs[r]):
                continue
            op = progs[r][pc[r]]
            if op[0] == "wait" and not all(flags[r][op[1]][w] >= op[2] for w in range(P)):
                continue
            ready.append(r)
        assert ready, "deadlock"
        r = rnd.choice(ready)
        op = progs[r][pc[r]]
        if op[0] == "signal":
            _, slot, e = op
            for o in range(P):
                flags[o][slot][r] = e
        elif op[0] == "step":
            _, i, e = op
            for s in range(i + 1, N):   # reads slices > i: complete for this epoch
                assert partial.get((r, s, e), set()) == set(range(P)), ("stale read", r, s, e)
            for o in range(P):          # stores its blocks of slice i everywhere
                assert partial.get((o, i, e - 1), set(range(P))) == set(range(P)) or e == 1
                partial.setdefault((o, i, e), set()).add(r)
        elif op[0] == "host_read" and op[1] > 0:
            e = op[1]
            for s in range(N):          # the host's table is the epoch-e table, not being rewritten
                assert partial.get((r, s, e), set()) == set(range(P)), ("incomplete", r, s, e)
                assert not any((r, s, e + 1) in partial and partial[(r, s, e + 1)] for _ in [0]), \
                    ("overwritten before the owner entered the next solve", r, s, e)
        pc[r] += 1
        steps += 1
    return steps


@pytest.mark.parametrize("P,N", [(2, 3), (3, 4), (8, 2), (4, 5)])
def test_flag_protocol_random_schedules(P, N):
    for seed in range(60):
        run(P, N, solves=3, seed=seed)


def test_protocol_without_entry_barrier_fails():
    """Mutation: dropping the entry barrier lets a fast rank overwrite a slow
    rank's table while its host still reads the previous solve."""
    import test_p2p_protocol as m

    def run_no_entry(P, N, solves, seed):
        rnd = random.Random(seed)
        flags = [[[0] * P for _ in range(N + 1)] for _ in range(P)]
        partial = {}
        progs = []
        for r in range(P):
            ops = []
            for e in range(1, solves + 1):
                ops += [("host_read", e - 1)]
                for i in range(N - 1, -1, -1):
                    ops += [("step", i, e), ("signal", i, e), ("wait", i, e)]
            progs.append(ops)
        pc = [0] * P
        while any(pc[r] < len(progs[r]) for r in range(P)):
            ready = [r for r in range(P) if pc[r] < len(progs[r]) and not (
                progs[r][pc[r]][0] == "wait" and
                not all(flags[r][progs[r][pc[r]][1]][w] >= progs[r][pc[r]][2] for w in range(P)))]
            r = rnd.choice(ready)
            op = progs[r][pc[r]]
            if op[0] == "signal":
                for o in range(P):
                    flags[o][op[1]][r] = op[2]
            elif op[0] == "step":
                for o in range(P):
                    partial.setdefault((o, op[1], op[2]), set()).add(r)
            elif op[0] == "host_read" and op[1] > 0:
                for s in range(N):
                    if partial.get((r, s, op[1] + 1)):
                        return True          # hazard observed
            pc[r] += 1
        return False

    assert any(run_no_entry(3, 3, 3, s) for s in range(200))
    assert m.run(3, 3, 3, 0) > 0
