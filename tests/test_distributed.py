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
        # a rank that owns no pivots still joins one exchange per lambda
        if rank == world - 1:
            none = _shard_solve(None, [0.0, 1.0], 0, 1, 0, True)
            assert none == [None, None]
        else:
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
            assert res[r][3:] == [0.0, -float(world - 2)]
