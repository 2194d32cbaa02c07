"""Algorithm 2 on the B200: per-pivot breakpoints of the regularisation path.

Mirror of the reference's ``l1line.path`` front half ("next"
row 1), same names, fields and semantics:

* ``PivotBreakpoints`` / ``pivot_breakpoints(data, pivot)``  <- path.py:38-102
* ``PivotSolutions`` / ``major_breakpoints(data, threads)``   <- path.py:105-154

For every column of a pivot, sorted position k of the tableau holds the
optimum for the half-open run of penalties starting at
``start_k = sgn(r_k) (T - P_k - P_{k-1}) - w_k`` of width ``2 w_k``; runs whose
right end is not positive are dropped, starts clamp at 0, and the largest
right end is the column's death weight.  The device
(``l1b_pivot_breakpoints``, ``csrc/path.cuh``) computes the exact ratios,
the stable sort of every column and the sequential prefix sums -- the
reference's 84 % -- bit for bit; this module keeps the
live runs and builds the same entry tuples.  The envelope merge
(Algorithm 3, ``merge_path``, path.py:166-277) runs natively too
(``l1b_merge_path``, ``csrc/merge.inc``): the same operations in the same
order in C++, so the path's breakpoints, lines and objectives are
bit-identical to the reference's.
"""

from __future__ import annotations

from bisect import bisect_right
from dataclasses import dataclass

import numpy as np

from .api import _as_data, _engine, resolve_threads
from .core import DataMatrix, EmptyPivotError, FittedLine, PathSegment, SolutionPath
from .engine import DeviceFit

__all__ = ["PivotBreakpoints", "PivotSolutions", "pivot_breakpoints", "major_breakpoints", "merge_path",
           "solution_path", "DEDUP_TOL"]

DEDUP_TOL = 1e-9  # path.py:34: breakpoints closer than this (absolute) are one


@dataclass(frozen=True)
class PivotBreakpoints:
    """Piecewise-constant snap values of every column of one pivot (path.py:38-73).

    ``entries[target]``: ascending (weight, value) pairs, the column takes
    ``value`` from that weight on; the last pair is (lambda_max[target], 0.0).
    """

    pivot: int
    entries: dict[int, tuple[tuple[float, float], ...]]
    lambda_max: dict[int, float]

    def column_value(self, target: int, lam: float) -> float:
        if lam < 0.0:
            raise ValueError("penalty weight must be nonnegative")
        entries = self.entries[target]
        return entries[bisect_right([bp for bp, _ in entries], lam) - 1][1]

    def breakpoint_set(self) -> set[float]:
        out: set[float] = set()
        for target, entries in self.entries.items():
            out.add(self.lambda_max[target])
            out.update(bp for bp, _ in entries[:-1] if bp > 0.0)
        return out


def _maps(pivot: int, m: int, rs: np.ndarray, st: np.ndarray, rt: np.ndarray,
          weights: list | None = None) -> PivotBreakpoints:
    entries: dict[int, tuple[tuple[float, float], ...]] = {}
    lambda_max: dict[int, float] = {}
    targets = [j for j in range(m) if j != pivot]
    for c, target in enumerate(targets):
        right = rt[c]
        live = right > 0.0
        # (max(0, start), r) for the live runs in sorted order, then (death, 0.0),
        # stably ordered by weight (path.py:92-97); max(0.0, x) == (x if x > 0.0 else 0.0)
        s_live = st[c][live]
        w = np.append(np.where(s_live > 0.0, s_live, 0.0), max(0.0, float(right.max())))
        val = np.append(rs[c][live], 0.0)
        order = np.argsort(w, kind="stable")
        entries[target] = tuple(zip(w[order].tolist(), val[order].tolist()))
        lambda_max[target] = float(w[-1])
        if weights is not None:
            weights.append(w)
    return PivotBreakpoints(pivot=pivot, entries=entries, lambda_max=lambda_max)


def _pivot_maps(eng: DeviceFit, pivot: int, weights: list | None = None) -> PivotBreakpoints:
    rs, st, rt = eng.pivot_runs(pivot)
    if rs is None:
        raise EmptyPivotError(f"column {pivot} is identically zero")
    return _maps(pivot, eng.m, rs, st, rt, weights)


def _dedup(vals: np.ndarray) -> np.ndarray:
    """path.py:146-152 on an array: keep v when v - (last kept) > DEDUP_TOL, ascending.

    Exact duplicates never survive, so np.unique first changes nothing; an
    element more than DEDUP_TOL above its predecessor is always kept (the last
    kept value is at most the predecessor), so only runs of closer neighbours
    need the sequential rule."""
    u = np.unique(vals)
    keep = np.ones(u.size, dtype=bool)
    close = np.nonzero(np.diff(u) <= DEDUP_TOL)[0] + 1
    if close.size:
        starts = close[np.concatenate(([True], np.diff(close) > 1))]
        ends = close[np.concatenate((np.diff(close) > 1, [True]))]
        for a, b in zip(starts.tolist(), ends.tolist()):
            last = float(u[a - 1])
            for i in range(a, b + 1):
                x = float(u[i])
                if x - last > DEDUP_TOL:
                    last = x
                else:
                    keep[i] = False
    return u[keep]


def pivot_breakpoints(data, pivot: int) -> PivotBreakpoints:
    """Closed-form breakpoints of one pivot's snap values (path.py:76-102)."""
    d = _as_data(data)
    if not 0 <= pivot < d.m:
        raise IndexError(f"pivot column {pivot} out of range")
    return _pivot_maps(_engine(data, d), int(pivot))


@dataclass(frozen=True)
class PivotSolutions:
    """Breakpoint maps of every usable pivot plus the degenerate ones (path.py:105-125)."""

    data: DataMatrix
    pivots: dict[int, PivotBreakpoints]
    degenerate: tuple[int, ...]

    def solution_at(self, pivot: int, lam: float) -> np.ndarray:
        v = np.zeros(self.data.m)
        if pivot in self.pivots:
            v[pivot] = 1.0
            for target, entries in self.pivots[pivot].entries.items():
                v[target] = entries[bisect_right([bp for bp, _ in entries], lam) - 1][1]
        elif pivot not in self.degenerate:
            raise IndexError(f"unknown pivot {pivot}")
        return v


def major_breakpoints(data, threads: int | None = None) -> tuple[np.ndarray, PivotSolutions]:
    """Every weight where some pivot's own solution changes (path.py:127-154):
    the ascending deduplicated grid (starting at 0) and the per-pivot maps."""
    resolve_threads(threads)
    d = _as_data(data)
    eng = _engine(data, d)  # K0 once; one device pass per pivot
    pivots: dict[int, PivotBreakpoints] = {}
    degenerate = []
    weights = [np.zeros(1)]  # the grid always starts at 0
    for p in range(d.m):
        try:
            pivots[p] = _pivot_maps(eng, p, weights)
        except EmptyPivotError:
            degenerate.append(p)
    return _dedup(np.concatenate(weights)), PivotSolutions(d, pivots, tuple(degenerate))


def _snap_indices(lambdas: np.ndarray, bps: np.ndarray) -> np.ndarray:
    """path.py:157-163 for an array of breakpoints."""
    idx = np.searchsorted(lambdas, bps)
    K = lambdas.size
    ic = np.minimum(idx, K - 1)
    here = (idx < K) & (np.abs(lambdas[ic] - bps) <= DEDUP_TOL)
    im = np.maximum(idx - 1, 0)
    left = (idx > 0) & (np.abs(lambdas[im] - bps) <= DEDUP_TOL)
    if not np.all(here | left):
        raise AssertionError("a breakpoint is missing from the weight grid")
    return np.where(here, idx, idx - 1)


def _events(solutions: PivotSolutions):
    """(pivot, target, value, breakpoint) of every entry in the reference's
    insertion order: pivot, target, entry (path.py:193-196)."""
    ep, et, ev, eb = [], [], [], []
    for p in sorted(solutions.pivots):
        for t, entries in solutions.pivots[p].entries.items():
            for bp, val in entries:
                ep.append(p)
                et.append(t)
                ev.append(val)
                eb.append(bp)
    return (np.asarray(ep, dtype=np.int64), np.asarray(et, dtype=np.int64), np.asarray(ev, dtype=np.float64),
            np.asarray(eb, dtype=np.float64))


def merge_path(lambdas, solutions: PivotSolutions, data) -> SolutionPath:
    """Lower envelope of the per-pivot objectives across the weight grid
    (path.py:166-277) on the device (``l1b_merge_path_device``)."""
    d = _as_data(data)
    return _merge(_engine(data, d), d, np.asarray(lambdas, dtype=np.float64),
                  np.asarray(sorted(solutions.pivots), dtype=np.int64),
                  np.asarray(sorted(solutions.degenerate), dtype=np.int64), *_events(solutions))


def _merge(eng: DeviceFit, d: DataMatrix, lambdas, piv, deg, ep, et, ev, eb) -> SolutionPath:
    import ctypes

    import torch

    from . import _lib
    lam = np.ascontiguousarray(lambdas, dtype=np.float64)
    lib = _lib.load()
    # events grouped by snapped grid index, insertion order kept (path.py:157-163, 193-196)
    eb = np.ascontiguousarray(eb, dtype=np.float64)
    order = np.empty(eb.size, dtype=np.int64)
    off = np.empty(lam.size + 1, dtype=np.int64)
    rc = lib.l1b_snap_events(lam.ctypes.data, lam.size, eb.ctypes.data, eb.size, DEDUP_TOL, order.ctypes.data,
                             off.ctypes.data)
    if rc == _lib.L1B_EINTERNAL:
        raise AssertionError("a breakpoint is missing from the weight grid")
    _lib.check(rc, "l1b_snap_events")
    ep = np.ascontiguousarray(np.asarray(ep, dtype=np.int64)[order])
    et = np.ascontiguousarray(np.asarray(et, dtype=np.int64)[order])
    ev = np.ascontiguousarray(np.asarray(ev, dtype=np.float64)[order])
    p64 = ctypes.POINTER(ctypes.c_int64)
    pd = ctypes.POINTER(ctypes.c_double)
    buf = ctypes.c_void_p()
    cnt = ctypes.c_int64()
    with torch.cuda.device(eng.device):
        rc = lib.l1b_merge_path_device(
            eng.X.data_ptr(), d.n, d.m, lam.ctypes.data_as(pd), lam.size, piv.ctypes.data_as(p64), piv.size,
            deg.ctypes.data_as(p64), deg.size, off.ctypes.data_as(p64), ep.ctypes.data_as(p64),
            et.ctypes.data_as(p64), ev.ctypes.data_as(pd), ctypes.byref(buf), ctypes.byref(cnt), eng.ws.data_ptr(),
            eng.ws.numel(), eng._s)
    _lib.check(rc, "l1b_merge_path_device")
    S, rec = int(cnt.value), 8 + d.m
    try:
        raw = np.ctypeslib.as_array(ctypes.cast(buf, pd), shape=(max(1, S) * rec,))[:S * rec].reshape(S, rec).copy()
    finally:
        lib.l1b_csv_free(buf)
    segs = []
    for r in raw:
        line = FittedLine(v=r[8:].copy(), preserved=int(r[2]), lam=float(r[0]), error=float(r[3]),
                          penalty_norm=float(r[4]), objective=float(r[5]))
        segs.append(PathSegment(lambda_lo=float(r[0]), lambda_hi=float(r[1]), line=line, z_lo=float(r[6]),
                                z_hi=float(r[7])))
    return SolutionPath(tuple(segs))


def _pivot_events(eng: DeviceFit, pivot: int):
    """Pivot p's breakpoint entries as arrays, without building tuples:
    (targets, weights, values) in the order of _maps (target ascending, then
    the entries stably sorted by weight, the death entry last among equals),
    or None for a zero pivot column."""
    rs, st, rt = eng.pivot_runs(pivot)
    if rs is None:
        return None
    m1, k = rs.shape
    live = rt > 0.0
    w = np.full((m1, k + 1), np.inf)
    w[:, :k] = np.where(live, np.where(st > 0.0, st, 0.0), np.inf)
    w[:, k] = np.maximum(0.0, rt.max(axis=1))
    val = np.zeros((m1, k + 1))
    val[:, :k] = rs
    order = np.argsort(w, axis=1, kind="stable")
    ws = np.take_along_axis(w, order, axis=1)
    vs = np.take_along_axis(val, order, axis=1)
    keep = np.isfinite(ws)  # the dropped (dead) runs sort last as +inf
    targets = np.array([j for j in range(eng.m) if j != pivot], dtype=np.int64)
    return np.broadcast_to(targets[:, None], ws.shape)[keep], ws[keep], vs[keep]


def solution_path(data, threads: int | None = None) -> SolutionPath:
    """Breakpoint grid plus envelope merge in one call (path.py:280-283):
    the runs come off the device as arrays and feed the device merge
    directly (the same entries, grid and events as major_breakpoints +
    merge_path)."""
    resolve_threads(threads)
    d = _as_data(data)
    eng = _engine(data, d)
    piv, deg, ep, et, ev = [], [], [], [], []
    for p in range(d.m):
        r = _pivot_events(eng, p)
        if r is None:
            deg.append(p)
            continue
        piv.append(p)
        ep.append(np.full(r[0].size, p, dtype=np.int64))
        et.append(r[0])
        ev.append((r[1], r[2]))
    eb = np.concatenate([w for w, _ in ev]) if ev else np.zeros(0)
    vals = np.concatenate([v for _, v in ev]) if ev else np.zeros(0)
    lambdas = _dedup(np.concatenate((np.zeros(1), eb)))
    return _merge(eng, d, lambdas, np.asarray(piv, dtype=np.int64), np.asarray(deg, dtype=np.int64),
                  np.concatenate(ep) if ep else np.zeros(0, dtype=np.int64),
                  np.concatenate(et) if et else np.zeros(0, dtype=np.int64), vals, eb)
