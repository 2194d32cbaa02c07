"""Multi-rank pivot sharding on CPU (gloo, world sizes 2 and 3).

The GPU box offers one device, so the N>1 plumbing -- interleaved pivot
shards, the (objective, pivot) all-gather, the owner's broadcast of v -- is
exercised here with gloo and the oracle as the per-shard solver.  The
combined result must equal the single-process fit bit for bit
(pkg/tests/test_acceptance.py:228-257 asks the same of worker counts).
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2402_16712_b200.engine import PivotWinner


def _oracle_solver(X, lams, p_begin, p_stride, npiv):
    pivs = [p_begin + k * p_stride for k in range(npiv)]
    out = []
    for li, lam in enumerate(lams):
        best = None
        for p in pivs:  # ascending pivot order, strict '<'
            line = oracle.fit_for_pivot(X, p, lam)
            if best is None or line.objective < best.objective:
                best = PivotWinner(p, float(lam), line.v, line.error, line.penalty_norm, line.objective)
        out.append(best)
    return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, X, lams, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2402_16712_b200.distributed import fit_lines_distributed
        lines = fit_lines_distributed(X, lams, solver=_oracle_solver)
        q.put((rank, [(l.preserved, l.v.tobytes(), l.objective, l.error, l.penalty_norm, l.lam)
                      for l in lines]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fit_matches_single_process(world):
    rng = np.random.default_rng(world)
    X = rng.uniform(-10, 10, size=(30, 7))
    X[:, 2] = 0.0                      # a degenerate pivot lands on some shard
    X[:, 5] = X[:, 1]                  # objective tie across shards -> smallest pivot
    lams = [0.0, 0.7, 5.0, 60.0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, lams, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = oracle.fit_line_multi(X, lams)
    for r in range(world):
        for k, w in enumerate(want):
            piv, vb, z, e, pn, lam = res[r][k]
            assert piv == w.preserved and vb == w.v.tobytes()
            assert z == w.objective and e == w.error and pn == w.penalty_norm and lam == lams[k]


def _exchange_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2402_16712_b200.distributed import _shard_solve, ub_exchange
        ex = ub_exchange()
        tops = [5.0 + rank, float("inf") if rank == 1 else 2.0 - rank, 1e300 * (rank + 1)]
        got = [ex(t) for t in tops]
        # a rank that owns no pivots still joins the exchanges the others make:
        # one vector for an all-finite sweep, one scalar per penalty otherwise
        if rank == world - 1:
            none = _shard_solve(None, [0.0, 1.0, 1.0], 0, 1, 0, True)
            assert none == [None, None, None]
            none = _shard_solve(None, [0.0, float("inf")], 0, 1, 0, True)
            assert none == [None, None]
        else:
            got += [float(x) for x in ex(np.array([float(rank), -float(rank)]))]
            got += [ex(float(rank)), ex(-float(rank))]
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_ub_exchange_is_global_min(world):
    """The pruning threshold exchange (all-reduce MIN), including ranks without pivots."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [5.0, min(2.0 - r for r in range(world) if r != 1), 1e300]
    for r in range(world):
        assert res[r][:3] == want
        if r != world - 1:
            assert res[r][3:] == [0.0, -float(world - 2), 0.0, -float(world - 2)]


def test_exchange_calls_follow_the_shard_paths():
    from paper_2402_16712_b200.distributed import exchange_calls
    assert exchange_calls([1.0], True) == [0]
    assert exchange_calls([0.0, 1.0, 1.0, 3.0], True) == [3]       # one vector over distinct penalties
    assert exchange_calls([0.0, float("inf")], True) == [0, 0]     # per-penalty loop
    assert exchange_calls([2.0, 2.0], True) == [0, 0]
    assert exchange_calls([0.0, 1.0], False) == []


def _combine_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2402_16712_b200.distributed import combine_winners
        m = 5
        v = np.array([1.0, -0.0, 0.0, -2.5, 3.0]) * (rank + 1)
        v[0] = 1.0
        # penalty 0: rank 1 wins outright; penalty 1: tie on the objective -> the smaller pivot
        # (rank 0); penalty 2: rank 0 owns no candidate
        local = [PivotWinner(rank, 0.0, v, 1.0, 2.0, 10.0 - rank),
                 PivotWinner(10 + rank, 1.0, v, 1.0, 2.0, 7.0),
                 None if rank == 0 else PivotWinner(20 + rank, 2.0, v, 1.0, 2.0, 3.0 + rank)]
        out = combine_winners(local, m)
        q.put((rank, [(w.pivot, w.v.tobytes(), w.objective) for w in out]))
    finally:
        dist.destroy_process_group()


def test_combine_winners_two_collectives_keep_signed_zeros():
    """One all_gather of the records plus one integer all_reduce of the winners'
    bit patterns carries every winning direction byte for byte (-0.0 too)."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_combine_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0

    def vb(r):
        v = np.array([1.0, -0.0, 0.0, -2.5, 3.0]) * (r + 1)
        v[0] = 1.0
        return v.tobytes()
    want = [(world - 1, vb(world - 1), 10.0 - (world - 1)), (10, vb(0), 7.0), (21, vb(1), 4.0)]
    for r in range(world):
        assert res[r] == want
