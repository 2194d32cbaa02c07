"""Pivot-sharded fit over several GPUs (one process per GPU).

SURVEY.md 8(e): the m pivots are independent units (fit.py:97), so rank r
fits pivots p = r, r + W, r + 2W, ... (interleaved, so zero-heavy column
ranges stay balanced) on its own replica of X, and only the per-shard
winner crosses the interconnect:

1. every rank reports (exact objective, pivot) of its shard winner
   (``torch.distributed.all_gather`` of 16 bytes per rank, NCCL over
   NVLink on the GPU box, gloo in the CPU tests);
2. all ranks take the lexicographic minimum of (objective, pivot) -- the
   strict '<' in ascending pivot order of fit.py:98-102;
3. the owning rank broadcasts the winning direction (8*m bytes).

With pivot pruning (engine.DeviceFit.shard_winners) one more exchange sits
between the bound pass and the exact fits: an all-reduce(MIN) of the
shards' best upper bounds (8 bytes per lambda), so every shard prunes
against the global best pivot and fits only what can still win overall.

Each pivot is solved on exactly one rank with exactly the single-GPU
kernels and re-scored with NumPy's summation order, so the result is
byte-identical for any world size.  There is no data-path collective.
"""

from __future__ import annotations

from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

from .core import FittedLine
from .engine import DeviceFit, PivotWinner, shard

__all__ = ["shard", "combine_winners", "ub_exchange", "fit_lines_distributed", "fit_line_distributed",
           "fit_subspace_distributed"]


def _comm_device(group=None) -> torch.device:
    backend = dist.get_backend(group)
    if backend == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def combine_winners(local: list[PivotWinner | None], m: int, group=None) -> list[PivotWinner]:
    """Global winner per lambda from every rank's shard winner: two collectives
    for any number of penalties.

    1. one ``all_gather`` of every rank's [L][5] (objective, pivot, error,
       penalty norm, lambda) records; every rank takes the lexicographic
       minimum of (objective, pivot) per lambda -- the strict '<' in
       ascending pivot order of fit.py:98-102 (``local[l]`` is None when the
       rank owns no pivot that can win);
    2. one ``all_reduce(SUM)`` of an [L][m] int64 tensor holding, in each
       lambda's row, the bit pattern of the winning direction on its owning
       rank and zeros elsewhere: integer sums with one nonzero term are exact,
       so every rank receives the owners' bytes (-0.0 included).
    """
    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    dev = _comm_device(group)
    L = len(local)
    rec = torch.full((L, 5), float("inf"), dtype=torch.float64)
    for l, w in enumerate(local):
        if w is not None:
            rec[l] = torch.tensor([w.objective, float(w.pivot), w.error, w.penalty_norm, w.lam],
                                  dtype=torch.float64)
    rec = rec.to(dev)
    gathered = [torch.empty_like(rec) for _ in range(world)]
    dist.all_gather(gathered, rec, group=group)
    allr = torch.stack(gathered).cpu().numpy()  # [world][L][5]
    owner = []
    for l in range(L):
        best_r = -1
        for r in range(world):
            z, p = allr[r, l, 0], allr[r, l, 1]
            if np.isinf(p):
                continue
            if best_r < 0:
                best_r = r
                continue
            bz, bp = allr[best_r, l, 0], allr[best_r, l, 1]
            if z < bz or (z == bz and p < bp):
                best_r = r
        if best_r < 0:
            raise ValueError("no rank owns any pivot")
        owner.append(best_r)
    bits = np.zeros((L, m), dtype=np.int64)
    for l in range(L):
        if owner[l] == me:
            bits[l] = np.ascontiguousarray(local[l].v, dtype=np.float64).view(np.int64)
    vb = torch.from_numpy(bits).to(dev)
    dist.all_reduce(vb, op=dist.ReduceOp.SUM, group=group)
    V = vb.cpu().numpy().view(np.float64)
    out = []
    for l in range(L):
        z, p, e, pn, lam = allr[owner[l], l]
        out.append(PivotWinner(int(p), float(lam), V[l].copy(), float(e), float(pn), float(z)))
    return out


def ub_exchange(group=None) -> Callable:
    """all-reduce(MIN) of the shards' best upper bounds: one value (a single
    penalty) or a vector (every penalty of a sweep) per call, one collective."""
    dev = _comm_device(group)

    def exchange(top):
        arr = np.atleast_1d(np.asarray(top, dtype=np.float64))
        t = torch.from_numpy(arr.copy()).to(dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        out = t.cpu().numpy()
        return float(out[0]) if np.ndim(top) == 0 else out
    return exchange


def exchange_calls(lams, prune: bool) -> list[int]:
    """The ub_exchange calls a pruning shard makes for ``lams``, as vector
    lengths (engine.DeviceFit.shard_winners' paths): one scalar for a single
    penalty, one vector over the distinct finite penalties of an all-finite
    sweep, else one scalar per penalty.  A rank without pivots makes the same
    calls with +inf so the collectives stay matched."""
    lam = np.atleast_1d(np.asarray(lams, dtype=np.float64))
    if not prune:
        return []
    if lam.size == 1:
        return [0]
    uniq = np.unique(lam[np.isfinite(lam)])
    if uniq.size > 1 and np.all(np.isfinite(lam)):
        return [int(uniq.size)]
    return [0] * int(lam.size)


def _shard_solve(eng: DeviceFit | None, lams, p_begin, p_stride, npiv, prune: bool, group=None):
    """One shard's winners; a rank without pivots still joins the exchanges."""
    ex = ub_exchange(group) if prune else None
    if npiv == 0:
        for size in exchange_calls(lams, prune):
            ex(float("inf") if size == 0 else np.full(size, np.inf))
        return [None] * len(lams)
    return eng.shard_winners(lams, p_begin, p_stride, npiv, prune=prune, ub_exchange=ex)


def _device_solver(X, lams, p_begin, p_stride, npiv, group=None):
    eng = DeviceFit(X, max_pivots=max(1, npiv))
    return _shard_solve(eng, lams, p_begin, p_stride, npiv, eng.auto_prune(), group)


def fit_lines_distributed(X, lams, group=None,
                          solver: Callable | None = None) -> list[FittedLine]:
    """fit_line for every lambda with the pivots sharded over the process group.

    ``solver(X, lams, p_begin, p_stride, npiv) -> list[PivotWinner]`` runs one
    shard; it defaults to the device engine (tests substitute the CPU oracle
    to exercise the multi-rank plumbing with gloo).
    """
    X = np.ascontiguousarray(getattr(X, "values", X), dtype=np.float64)
    lams = [float(x) for x in np.atleast_1d(lams)]
    m = X.shape[1]
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    p_begin, p_stride, npiv = shard(m, rank, world)
    if solver is None:
        local = _device_solver(X, lams, p_begin, p_stride, npiv, group)
    else:
        local = solver(X, lams, p_begin, p_stride, npiv) if npiv > 0 else [None] * len(lams)
    wins = combine_winners(local, m, group)
    return [FittedLine(v=w.v, preserved=w.pivot, lam=w.lam, error=w.error, penalty_norm=w.penalty_norm,
                       objective=w.objective) for w in wins]


def fit_line_distributed(X, lam: float, group=None, solver: Callable | None = None) -> FittedLine:
    return fit_lines_distributed(X, [lam], group, solver)[0]


def fit_subspace_distributed(data, lam: float, k: int, group=None):
    """fit_subspace (subspace.py:54-76) with every component's pivots sharded.

    Each rank keeps its own device replica of X; after the winner of a
    component is combined, every rank deflates its replica with the same v
    (subspace.py:22-36), so the replicas stay bit-identical with no traffic
    beyond the winner exchange.
    """
    import math

    from .core import SubspaceFit

    X = np.ascontiguousarray(getattr(data, "values", data), dtype=np.float64)
    n, m = X.shape
    if not 1 <= k < m:
        raise ValueError(f"component count {k} must be in [1, {m - 1}]")
    if lam < 0.0 or not math.isfinite(lam):
        raise ValueError("penalty weight must be finite and nonnegative")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    p_begin, p_stride, npiv = shard(m, rank, world)
    eng = DeviceFit(X, max_pivots=max(1, npiv))
    scale = max(1.0, eng.absmax())
    comps = []
    for t in range(k):
        if eng.absmax() <= 1e-10 * scale:
            return SubspaceFit(tuple(comps), degenerate=True)
        eng.set_steer(0 if t == 0 else -1)  # api.fit_subspace's steering policy
        local = _shard_solve(eng, [float(lam)], p_begin, p_stride, npiv, eng.auto_prune(), group)
        w = combine_winners(local, m, group)[0]
        comps.append(FittedLine(v=w.v, preserved=w.pivot, lam=w.lam, error=w.error,
                                penalty_norm=w.penalty_norm, objective=w.objective))
        if not np.any(w.v):  # subspace.py:75 / 32-33: the reference's deflate rejects v = 0
            raise ValueError("cannot deflate along the zero vector")
        if t + 1 < k:
            eng.deflate(w.v)
    return SubspaceFit(tuple(comps), degenerate=False)
