"""Device-resident fit engine: one matrix, one workspace, one CUDA stream.

``DeviceFit`` owns the device copy of X (row-major f64 exactly as
``DataMatrix.values`` lays it out, core.py:49) and the workspace the C ABI
needs, and runs Algorithm 1 for a pivot shard and a batch of penalty
weights.  PyTorch is only the allocator/stream provider here; every
computation is a kernel in ``csrc/l1b200.cu`` called through ``_lib``.

Winner selection reproduces fit.py:98-102 exactly: the kernels rank pivots
by objectives summed in a fixed device order, then every pivot whose
objective is within ``RESCORE_RTOL`` of the minimum is re-scored with the
reference's own rounding (``l1b_residual_exact`` = residual_error's NumPy
pairwise order, core.py:93; ``np.abs(v).sum()`` for the penalty,
core.py:131) and the first pivot with the smallest exact objective wins.
The device sums differ from NumPy's by far less than RESCORE_RTOL, so the
chosen pivot, error, penalty and objective are those the reference would
report for the same directions.
"""

from __future__ import annotations

import ctypes
import math
import os
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

RESCORE_RTOL = 1e-8
# absolute part of the re-score window, times n*m*max|x|: device and NumPy
# residual terms differ by a few ulps of |x_ij| + |v_j x_ip|, so a near-zero
# objective (an exact fit) needs an absolute floor, not only a relative one
RESCORE_ATOL = 1e-13
# pruning keeps every pivot whose lower bound is within this of the best
# upper bound (the bounds already carry their float-error margins; this
# covers the reference's own rounding of the objective)
PRUNE_RTOL = 1e-9
# refine (one more bounding pass per level on the survivors) while more than
# REFINE_MIN pivots survive, at most REFINE_PASSES levels; each level costs
# one pass per surviving pivot and shrinks the bound gaps ~1000x
REFINE_MIN = 2
REFINE_PASSES = 3


def _stream_handle(stream: torch.cuda.Stream | None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


@dataclass
class PivotWinner:
    """Exact-rescored winner of one pivot shard at one penalty weight."""

    pivot: int
    lam: float
    v: np.ndarray
    error: float
    penalty_norm: float
    objective: float


def shard(m: int, rank: int, world: int) -> tuple[int, int, int]:
    """Interleaved pivot shard p = rank, rank + world, ...."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    npiv = max(0, (m - rank + world - 1) // world)
    return rank, world, npiv


_STAGING: dict = {}
_STAGE_DOUBLES = 1 << 19  # 4 MB pinned chunks
_STAGE_THREADS = 8


def _upload(Xh: np.ndarray, device: torch.device) -> torch.Tensor:
    """Host numpy -> device through two reused pinned chunks (l1b_upload): the
    CPU copy of chunk i+1 into pinned memory overlaps the DMA of chunk i
    (instead of pinning the whole matrix, then copying it).  The CPU copy is
    l1b_host_copy: a few pool threads with streaming stores, so the copy
    engine reads the chunk from DRAM at full link speed (hostcopy.inc)."""
    key = (device.type, device.index)
    if key not in _STAGING:
        with torch.cuda.device(device):
            _STAGING[key] = [torch.empty(_STAGE_DOUBLES, dtype=torch.float64).pin_memory() for _ in range(2)]
    stage = _STAGING[key]
    lib = _lib.load()
    with torch.cuda.device(device):
        dst = torch.empty(Xh.shape, dtype=torch.float64, device=device)
        stream = torch.cuda.current_stream(device)
        _lib.check(lib.l1b_upload(dst.data_ptr(), Xh.ctypes.data, Xh.nbytes, stage[0].data_ptr(), stage[1].data_ptr(),
                                  8 * _STAGE_DOUBLES, _STAGE_THREADS, stream.cuda_stream), "l1b_upload")
        # the stages are reused by the next upload: its first wait is on these transfers'
        # events inside l1b_upload, so nothing else is needed here
    return dst


class DeviceFit:
    """A data matrix resident on one GPU plus everything a fit needs."""

    def __init__(self, X, device: torch.device | str | None = None,
                 stream: torch.cuda.Stream | None = None, max_pivots: int | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2402_16712_b200 needs a CUDA device (there is no CPU fallback)")
        self.lib = _lib.load()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.stream = stream
        if isinstance(X, torch.Tensor):
            Xd = X.to(device=self.device, dtype=torch.float64).contiguous()
        else:
            Xh = np.ascontiguousarray(X, dtype=np.float64)
            if Xh.size >= (1 << 16):
                Xd = _upload(Xh, self.device)
            else:
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore", UserWarning)
                    Xd = torch.from_numpy(Xh).to(self.device)
        if Xd.dim() != 2:
            raise ValueError(f"expected a 2-d array, got shape {tuple(Xd.shape)}")
        self.X = Xd
        self.n, self.m = int(Xd.shape[0]), int(Xd.shape[1])
        self.max_pivots = self.m if max_pivots is None else int(max_pivots)
        self.last_candidates = None
        nbytes = self.lib.l1b_workspace_bytes(self.n, self.m, 1, max(1, self.max_pivots))
        if nbytes == 0:
            raise ValueError(f"bad matrix shape {(self.n, self.m)}")
        with torch.cuda.device(self.device):
            self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            self.tmp = torch.empty(self.n + 2, dtype=torch.float64, device=self.device)
            self.scalar = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.prepare()

    # ------------------------------------------------------------- kernels --
    @property
    def _s(self) -> int:
        return _stream_handle(self.stream)

    def prepare(self) -> None:
        """K0 (l1b_prepare); rerun whenever X changes."""
        self._scale = None
        with torch.cuda.device(self.device):
            _lib.check(self.lib.l1b_prepare(self.X.data_ptr(), self.n, self.m, self.ws.data_ptr(),
                                            self.ws.numel(), self._s), "l1b_prepare")

    def fit_pivots(self, lams, p_begin: int = 0, p_stride: int = 1, npiv: int | None = None,
                   want_v: bool = True):
        """K1+K2 for a pivot shard: device tensors V [L][np][m], err/pen/obj [L][np]."""
        lam = np.ascontiguousarray(np.atleast_1d(np.asarray(lams, dtype=np.float64)))
        if npiv is None:
            npiv = shard(self.m - p_begin, 0, p_stride)[2] if p_stride > 1 else self.m - p_begin
        if npiv > self.max_pivots:
            raise ValueError(f"shard of {npiv} pivots exceeds workspace for {self.max_pivots}")
        L = lam.size
        with torch.cuda.device(self.device):
            V = torch.empty((L, npiv, self.m), dtype=torch.float64, device=self.device) if want_v else None
            err = torch.empty((L, npiv), dtype=torch.float64, device=self.device)
            pen = torch.empty_like(err)
            obj = torch.empty_like(err)
            rc = self.lib.l1b_fit_pivots(
                self.X.data_ptr(), self.n, self.m, lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                L, p_begin, p_stride, npiv, V.data_ptr() if want_v else None, err.data_ptr(),
                pen.data_ptr(), obj.data_ptr(), self.ws.data_ptr(), self.ws.numel(), self._s)
        _lib.check(rc, "l1b_fit_pivots")
        return V, err, pen, obj

    def straggler_counts(self, npiv: int | None = None) -> tuple[int, int]:
        """Problems the last fit_pivots sent to the exact straggler solver."""
        out = (ctypes.c_uint64 * 2)()
        with torch.cuda.device(self.device):
            _lib.check(self.lib.l1b_fit_stats(self.n, self.m, npiv or self.max_pivots, self.ws.data_ptr(),
                                              self.ws.numel(), ctypes.addressof(out), self._s), "l1b_fit_stats")
        return int(out[0]), int(out[1])

    def residual_exact(self, v_dev: torch.Tensor, pivot: int) -> float:
        """residual_error (core.py:79-93) with NumPy's exact summation order."""
        with torch.cuda.device(self.device):
            _lib.check(self.lib.l1b_residual_exact(self.X.data_ptr(), self.n, self.m, v_dev.data_ptr(),
                                                   int(pivot), self.scalar.data_ptr(), self.ws.data_ptr(),
                                                   self.ws.numel(), self._s), "l1b_residual_exact")
            return float(self.scalar.item())

    def deflate(self, v) -> None:
        """subspace.py:22-36 in place on the device copy, then re-prepare."""
        with torch.cuda.device(self.device):
            v_dev = torch.tensor(np.asarray(v, dtype=np.float64), device=self.device)  # a copy: v may be read-only
            _lib.check(self.lib.l1b_deflate(self.X.data_ptr(), self.n, self.m, v_dev.data_ptr(),
                                            self.tmp.data_ptr(), self._s), "l1b_deflate")
        self.prepare()

    def set_steer(self, mode: int) -> None:
        """Steering of the first bound pass (l1b_set_steer): -1 automatic, 0 off, s > 1 stride."""
        _lib.check(self.lib.l1b_set_steer(self.ws.data_ptr(), int(mode)), "l1b_set_steer")

    def absmax(self) -> float:
        """max |x| of the prepared X (K0 computes it; no pass over X here)."""
        with torch.cuda.device(self.device):
            _lib.check(self.lib.l1b_prepared_absmax(self.ws.data_ptr(), self.n, self.m, self.ws.numel(),
                                                    self.scalar.data_ptr(), self._s), "l1b_prepared_absmax")
            return float(self.scalar.item())

    # ------------------------------------------------------------- winners --
    def fit_pivot_list(self, lams, pivots, want_v: bool = True):
        """K1+K2 for an explicit pivot list: V [L][k][m], err/pen/obj [L][k] in list order."""
        lam = np.ascontiguousarray(np.atleast_1d(np.asarray(lams, dtype=np.float64)))
        piv = np.ascontiguousarray(np.asarray(pivots, dtype=np.int64))
        k = piv.size
        if k > self.max_pivots:
            raise ValueError(f"{k} pivots exceed the workspace for {self.max_pivots}")
        L = lam.size
        with torch.cuda.device(self.device):
            V = torch.empty((L, k, self.m), dtype=torch.float64, device=self.device) if want_v else None
            err = torch.empty((L, k), dtype=torch.float64, device=self.device)
            pen = torch.empty_like(err)
            obj = torch.empty_like(err)
            rc = self.lib.l1b_fit_pivot_list(
                self.X.data_ptr(), self.n, self.m, lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), L,
                piv.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), k, V.data_ptr() if want_v else None,
                err.data_ptr(), pen.data_ptr(), obj.data_ptr(), self.ws.data_ptr(), self.ws.numel(), self._s)
        _lib.check(rc, "l1b_fit_pivot_list")
        return V, err, pen, obj

    def fit_pivot_list_seeded(self, lam: float, pivots, seed, seed_npiv: int):
        """fit_pivot_list for one lambda, seeded by the last bound call (l1b_fit_pivot_list_seeded):
        pivot k was entry seed[k] of that call's list of seed_npiv pivots."""
        piv = np.ascontiguousarray(np.asarray(pivots, dtype=np.int64))
        sd = np.ascontiguousarray(np.asarray(seed, dtype=np.int64))
        k = piv.size
        with torch.cuda.device(self.device):
            V = torch.empty((1, k, self.m), dtype=torch.float64, device=self.device)
            err = torch.empty((1, k), dtype=torch.float64, device=self.device)
            pen = torch.empty_like(err)
            obj = torch.empty_like(err)
            rc = self.lib.l1b_fit_pivot_list_seeded(
                self.X.data_ptr(), self.n, self.m, float(lam), piv.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                k, sd.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(seed_npiv), V.data_ptr(), err.data_ptr(),
                pen.data_ptr(), obj.data_ptr(), self.ws.data_ptr(), self.ws.numel(), self._s)
        _lib.check(rc, "l1b_fit_pivot_list_seeded")
        return V, err, pen, obj

    def bound_pivot_sums(self, lam: float, p_begin: int = 0, p_stride: int = 1, npiv: int | None = None,
                         steer: int = 0):
        """The same bounds from fit_line's lean first pass (l1b_bound_pivot_sums): per-pivot
        sums only, no per-column bounds left behind."""
        if npiv is None:
            npiv = shard(self.m - p_begin, 0, p_stride)[2] if p_stride > 1 else self.m - p_begin
        with torch.cuda.device(self.device):
            b = torch.empty((2, npiv), dtype=torch.float64, device=self.device)
            rc = self.lib.l1b_bound_pivot_sums(self.X.data_ptr(), self.n, self.m, float(lam), p_begin, p_stride,
                                               npiv, int(steer), b[0].data_ptr(), b[1].data_ptr(), self.ws.data_ptr(),
                                               self.ws.numel(), self._s)
            _lib.check(rc, "l1b_bound_pivot_sums")
            bh = b.cpu().numpy()
        return bh[0], bh[1]

    def bound_pivots(self, lam: float, p_begin: int = 0, p_stride: int = 1, npiv: int | None = None):
        """Rigorous bounds lb <= z_p <= ub of every shard pivot's objective (host arrays)."""
        if npiv is None:
            npiv = shard(self.m - p_begin, 0, p_stride)[2] if p_stride > 1 else self.m - p_begin
        with torch.cuda.device(self.device):
            b = torch.empty((2, npiv), dtype=torch.float64, device=self.device)
            rc = self.lib.l1b_bound_pivots(self.X.data_ptr(), self.n, self.m, float(lam), p_begin, p_stride, npiv,
                                           b[0].data_ptr(), b[1].data_ptr(), self.ws.data_ptr(), self.ws.numel(),
                                           self._s)
            _lib.check(rc, "l1b_bound_pivots")
            bh = b.cpu().numpy()
        return bh[0], bh[1]

    def pivot_runs(self, pivot: int):
        """Sorted tableau runs of one pivot (l1b_pivot_breakpoints): ratios, starts and
        right ends [m-1][n_p] in sorted order per target column, or (None, None, None)
        for a zero pivot column."""
        nr = ctypes.c_int64()
        with torch.cuda.device(self.device):
            _lib.check(self.lib.l1b_pivot_breakpoints(self.X.data_ptr(), self.n, self.m, int(pivot),
                                                      ctypes.byref(nr), None, None, None, 0, self.ws.data_ptr(),
                                                      self.ws.numel(), self._s), "l1b_pivot_breakpoints")
            k = int(nr.value)
            if k == 0:
                return None, None, None
            out = torch.empty((3, self.m - 1, k), dtype=torch.float64, device=self.device)
            _lib.check(self.lib.l1b_pivot_breakpoints(self.X.data_ptr(), self.n, self.m, int(pivot),
                                                      ctypes.byref(nr), out[0].data_ptr(), out[1].data_ptr(),
                                                      out[2].data_ptr(), k, self.ws.data_ptr(), self.ws.numel(),
                                                      self._s), "l1b_pivot_breakpoints")
            h = out.cpu().numpy()
        return h[0], h[1], h[2]

    def tableau(self, pivot: int, target: int = -1):
        """Sorted tableau columns of one pivot (l1b_pivot_tableau, ratios.py:40-67 / 109-135):
        ratios, weights, inclusive prefix [c][k] (f64) and source rows [c][k] (i64) for
        target ``target`` (c = 0) or every target j != pivot; None for a zero pivot column."""
        nr = ctypes.c_int64()
        ncol = self.m - 1 if target < 0 else 1
        with torch.cuda.device(self.device):
            _lib.check(self.lib.l1b_pivot_tableau(self.X.data_ptr(), self.n, self.m, int(pivot), int(target),
                                                  ctypes.byref(nr), None, None, None, None, 0, self.ws.data_ptr(),
                                                  self.ws.numel(), self._s), "l1b_pivot_tableau")
            k = int(nr.value)
            if k == 0:
                return None
            out = torch.empty((3, ncol, k), dtype=torch.float64, device=self.device)
            rows = torch.empty((ncol, k), dtype=torch.int64, device=self.device)
            _lib.check(self.lib.l1b_pivot_tableau(self.X.data_ptr(), self.n, self.m, int(pivot), int(target),
                                                  ctypes.byref(nr), out[0].data_ptr(), out[1].data_ptr(),
                                                  out[2].data_ptr(), rows.data_ptr(), k, self.ws.data_ptr(),
                                                  self.ws.numel(), self._s), "l1b_pivot_tableau")
            h = out.cpu().numpy()
            r = rows.cpu().numpy()
        return h[0], h[1], h[2], r

    def bound_entries(self, lams, pivots, from_pos=None, from_count: int = 0, from_ranges=None):
        """One bounding pass per (pivot, penalty) entry (l1b_bound_entries); with
        from_pos, continuing from those entries of the last bound call (or of
        the multi-penalty pass's ranges, from_ranges)."""
        piv = np.ascontiguousarray(np.asarray(pivots, dtype=np.int64))
        lam = np.ascontiguousarray(np.asarray(lams, dtype=np.float64))
        fp = None if from_pos is None else np.ascontiguousarray(np.asarray(from_pos, dtype=np.int64))
        with torch.cuda.device(self.device):
            b = torch.empty((2, piv.size), dtype=torch.float64, device=self.device)
            rc = self.lib.l1b_bound_entries(
                self.X.data_ptr(), self.n, self.m, lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                piv.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), piv.size,
                None if fp is None else fp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(from_count),
                None if from_ranges is None else from_ranges.data_ptr(),
                b[0].data_ptr(), b[1].data_ptr(), self.ws.data_ptr(), self.ws.numel(), self._s)
            _lib.check(rc, "l1b_bound_entries")
            bh = b.cpu().numpy()
        return bh[0], bh[1]

    def fit_entries_seeded(self, lams, pivots, seed, seed_count: int):
        """Seeded exact fit of (pivot, penalty) entries (l1b_fit_entries_seeded)."""
        piv = np.ascontiguousarray(np.asarray(pivots, dtype=np.int64))
        lam = np.ascontiguousarray(np.asarray(lams, dtype=np.float64))
        sd = np.ascontiguousarray(np.asarray(seed, dtype=np.int64))
        k = piv.size
        with torch.cuda.device(self.device):
            V = torch.empty((k, self.m), dtype=torch.float64, device=self.device)
            eo = torch.empty((3, k), dtype=torch.float64, device=self.device)
            rc = self.lib.l1b_fit_entries_seeded(
                self.X.data_ptr(), self.n, self.m, lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                piv.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), k,
                sd.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(seed_count), V.data_ptr(), eo[0].data_ptr(),
                eo[1].data_ptr(), eo[2].data_ptr(), self.ws.data_ptr(), self.ws.numel(), self._s)
        _lib.check(rc, "l1b_fit_entries_seeded")
        return V, eo[0], eo[1], eo[2]

    def _sweep_winners(self, lam, all_piv, lbm, ubm, uniq, ub_exchange, ranges=None, npiv: int = 0):
        """Winners of a penalty sweep after one multi-penalty pass: every
        penalty's survivors are refined and fitted together as one entry list
        (one launch per cascade level instead of one per penalty)."""
        L = uniq.size
        tops = np.array([float(np.min(ubm[i])) for i in range(L)])
        if ub_exchange is not None:  # every penalty's best upper bound over all shards, one collective
            tops = np.asarray(ub_exchange(tops), dtype=np.float64).reshape(L)
        ent_l, ent_k = [], []
        for i in range(L):
            k = np.nonzero(~(lbm[i] > self._prune_threshold(tops[i])))[0]
            ent_l.append(np.full(k.size, i, dtype=np.int64))
            ent_k.append(k)
        # entry lists are bounded by the workspace's pivot capacity: penalties
        # go in batches whose survivors fit
        batches, cur, size = [], [], 0
        for i in range(L):
            c = ent_k[i].size
            if cur and size + c > self.max_pivots:
                batches.append(cur)
                cur, size = [], 0
            cur.append(i)
            size += c
        if cur:
            batches.append(cur)
        wins = {}
        self.last_candidates = 0
        for bl in batches:
            li = np.concatenate([ent_l[i] for i in bl])  # entry -> penalty index
            kk = np.concatenate([ent_k[i] for i in bl])  # entry -> shard pivot position
            seed, seed_n = None, 0
            src = None
            if ranges is not None:  # level 0 continues from the multi pass's per-penalty ranges
                seed, seed_n, src = li * npiv + kk, L * npiv, ranges
            for level in range(REFINE_PASSES + 1):
                counts = np.bincount(li, minlength=L)
                if kk.size == 0 or (level > 0 and np.all(counts <= REFINE_MIN)):
                    break
                lb2, ub2 = self.bound_entries(uniq[li], all_piv[kk], seed, seed_n, src)
                src = None
                np.minimum.at(tops, li, ub2)
                ok = ~(lb2 > np.array([self._prune_threshold(t) for t in tops])[li])
                sel = np.nonzero(ok)[0]
                li, kk, seed, seed_n = li[sel], kk[sel], sel, lb2.size
            self.last_candidates += int(kk.size)
            if kk.size:
                V, err, pen, obj = self.fit_entries_seeded(uniq[li], all_piv[kk], seed, seed_n)
                obj_h = obj.cpu().numpy()
                ids, groups = [], []
                for i in bl:
                    e = np.nonzero(li == i)[0]
                    if e.size:
                        ids.append(i)
                        # rows e of V, gathered only for the re-scored candidates (one gather for all)
                        groups.append((float(uniq[i]), all_piv[kk[e]], (V, e), obj_h[e]))
                wins.update(zip(ids, self._winners(groups)))
        return [wins.get(int(np.searchsorted(uniq, x))) for x in lam]

    def bound_pivots_multi(self, lams, p_begin: int = 0, p_stride: int = 1, npiv: int | None = None,
                           ranges: bool = False):
        """One bounding pass for several strictly ascending penalties: lb, ub [L][npiv]
        (host); with ranges, also every (penalty, pivot, target)'s next range
        [L][npiv][m] (device float pairs) for bound_entries to continue from."""
        lam = np.ascontiguousarray(np.asarray(lams, dtype=np.float64))
        if npiv is None:
            npiv = shard(self.m - p_begin, 0, p_stride)[2] if p_stride > 1 else self.m - p_begin
        with torch.cuda.device(self.device):
            b = torch.empty((2, lam.size, npiv), dtype=torch.float64, device=self.device)
            rg = torch.empty((lam.size, npiv, self.m, 2), dtype=torch.float32, device=self.device) if ranges else None
            rc = self.lib.l1b_bound_pivots_multi(
                self.X.data_ptr(), self.n, self.m, lam.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), lam.size,
                p_begin, p_stride, npiv, b[0].data_ptr(), b[1].data_ptr(), None if rg is None else rg.data_ptr(),
                self.ws.data_ptr(), self.ws.numel(), self._s)
            _lib.check(rc, "l1b_bound_pivots_multi")
            bh = b.cpu().numpy()
        if ranges:
            return bh[0], bh[1], rg
        return bh[0], bh[1]

    def bound_pivot_list(self, lam: float, pivots, passes: int = REFINE_PASSES):
        """Bounds for an explicit pivot list; passes 2-3 refine the optimum's range."""
        piv = np.ascontiguousarray(np.asarray(pivots, dtype=np.int64))
        with torch.cuda.device(self.device):
            b = torch.empty((2, piv.size), dtype=torch.float64, device=self.device)
            rc = self.lib.l1b_bound_pivot_list(self.X.data_ptr(), self.n, self.m, float(lam),
                                               piv.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), piv.size,
                                               int(passes), b[0].data_ptr(), b[1].data_ptr(), self.ws.data_ptr(),
                                               self.ws.numel(), self._s)
            _lib.check(rc, "l1b_bound_pivot_list")
            bh = b.cpu().numpy()
        return bh[0], bh[1]

    def bound_columns(self, count: int):
        """Per-column bounds [count][m] of the last bound call over ``count`` pivots (diagnostics, tests)."""
        lb = np.empty((count, self.m), dtype=np.float64)
        ub = np.empty_like(lb)
        with torch.cuda.device(self.device):
            _lib.check(self.lib.l1b_bound_columns(self.n, self.m, count, self.ws.data_ptr(), self.ws.numel(),
                                                  lb.ctypes.data, ub.ctypes.data, self._s),
                       "l1b_bound_columns")
        return lb, ub

    def bound_pivot_list_continue(self, lam: float, pivots, from_pos, from_npiv: int):
        """One more bounding pass for pivots[k] = entry from_pos[k] of the last bound call's list."""
        piv = np.ascontiguousarray(np.asarray(pivots, dtype=np.int64))
        fp = np.ascontiguousarray(np.asarray(from_pos, dtype=np.int64))
        with torch.cuda.device(self.device):
            b = torch.empty((2, piv.size), dtype=torch.float64, device=self.device)
            rc = self.lib.l1b_bound_pivot_list_continue(
                self.X.data_ptr(), self.n, self.m, float(lam), piv.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                piv.size, fp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), int(from_npiv), b[0].data_ptr(),
                b[1].data_ptr(), self.ws.data_ptr(), self.ws.numel(), self._s)
            _lib.check(rc, "l1b_bound_pivot_list_continue")
            bh = b.cpu().numpy()
        return bh[0], bh[1]

    def residual_exact_batch(self, V: torch.Tensor, pivots) -> np.ndarray:
        """residual_exact for the rows of V [C][m] (pivot pivots[k]) in one batch."""
        piv = np.ascontiguousarray(np.asarray(pivots, dtype=np.int64))
        V = V.contiguous()
        with torch.cuda.device(self.device):
            out = torch.empty(piv.size, dtype=torch.float64, device=self.device)
            _lib.check(self.lib.l1b_residual_exact_batch(
                self.X.data_ptr(), self.n, self.m, V.data_ptr(), V.stride(0),
                piv.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), piv.size, out.data_ptr(), self.ws.data_ptr(),
                self.ws.numel(), self._s), "l1b_residual_exact_batch")
            return out.cpu().numpy()

    def _candidates(self, obj_h) -> np.ndarray:
        o = obj_h
        best = float(o.min())
        if math.isinf(best):
            return np.nonzero(o == best)[0][:1]
        return np.nonzero(o <= best + RESCORE_RTOL * abs(best) + RESCORE_ATOL * self._abs_scale() + 1e-300)[0]

    def _winners(self, groups) -> list[PivotWinner]:
        """fit.py:98-102 for several (lam, pivots, V, obj) groups of fitted
        pivots: the near-minimal ones of every group are re-scored with the
        reference's rounding in one batch, the first strict minimum wins."""
        picks = []
        for lam, pivots, V, obj_h in groups:
            if np.isnan(obj_h).any():
                # FittedLine's invariant rejects a NaN objective (core.py:120-124):
                # only lam=inf with an all-zero pivot column produces one.
                raise ValueError(f"objective nan for lam={lam!r} (zero pivot column at infinite penalty)")
            picks.append(self._candidates(obj_h))
        pivs = np.concatenate([np.asarray(g[1])[c] for g, c in zip(groups, picks)]).astype(np.int64)
        # a group's V is a [k][m] tensor or (V, e): rows e of a shared [K][m] tensor
        lazy = all(isinstance(g[2], tuple) for g in groups) and len({id(g[2][0]) for g in groups}) == 1
        if pivs.size == 1:  # the common case: one candidate, no batching copies
            V = groups[0][2]
            row = V[0][int(V[1][picks[0][0]])] if isinstance(V, tuple) else V[int(picks[0][0])]
            errs = [self.residual_exact(row, int(pivs[0]))]
            vhs = row.cpu().numpy()[None, :]
        else:
            if lazy:
                Vb = groups[0][2][0]
                idx = np.concatenate([g[2][1][c] for g, c in zip(groups, picks)]).astype(np.int64)
                rows = Vb[torch.from_numpy(idx).to(Vb.device)]
            else:
                rows = torch.cat([(V[0][torch.as_tensor(V[1], device=V[0].device)] if isinstance(V, tuple) else V)
                                  [torch.as_tensor(c, device=(V[0] if isinstance(V, tuple) else V).device)]
                                  for (_, _, V, _), c in zip(groups, picks)])
            errs = self.residual_exact_batch(rows, pivs)
            vhs = rows.cpu().numpy()
        out, at = [], 0
        for (lam, _, _, _), c in zip(groups, picks):
            win = None
            for k in range(c.size):  # ascending pivot order
                vh = vhs[at + k].copy()
                e = float(errs[at + k])
                pn = float(np.abs(vh).sum())
                z = e + float(lam) * pn
                if win is None or z < win.objective:
                    win = PivotWinner(int(pivs[at + k]), float(lam), vh, e, pn, z)
            out.append(win)
            at += c.size
        return out

    def _winner(self, lam: float, pivots, V, obj_h) -> PivotWinner:
        """fit.py:98-102 among fitted pivots (one group of _winners)."""
        return self._winners([(lam, pivots, V, obj_h)])[0]

    def _abs_scale(self) -> float:
        if self._scale is None:
            self._scale = self.absmax() * self.n * self.m
        return self._scale

    def shard_winners(self, lams, p_begin: int = 0, p_stride: int = 1,
                      npiv: int | None = None, prune: bool | None = None,
                      ub_exchange=None) -> list[PivotWinner | None]:
        """Exact winner of the shard for every lambda (fit.py:98-102 semantics).

        With ``prune`` (None: auto_prune()) every pivot is first bounded by one FP32 pass
        (l1b_bound_pivots) and only the pivots whose lower bound does not
        exceed the smallest upper bound are fitted exactly -- the others
        provably cannot win, so the result is the same as fitting all.

        ``ub_exchange(top) -> global top`` (sharded fits) replaces the
        shard's best upper bound by the best over all shards before pruning;
        a shard whose pivots are all provably beaten then returns None for
        that lambda.  Called once per lambda, or once with the vector of a
        sweep's distinct penalties (distributed.exchange_calls).
        """
        lam = np.atleast_1d(np.asarray(lams, dtype=np.float64))
        if npiv is None:
            npiv = shard(self.m - p_begin, 0, p_stride)[2] if p_stride > 1 else self.m - p_begin
        all_piv = p_begin + p_stride * np.arange(npiv, dtype=np.int64)
        out = []
        if lam.size == 1:
            # one penalty: the whole cascade in one C call (no Python round trips)
            return [self.fit_line_device(float(lam[0]), p_begin, p_stride, npiv, prune, ub_exchange)]
        if prune is None:
            prune = self.auto_prune()
        if not prune:
            V, err, pen, obj = self.fit_pivots(lam, p_begin, p_stride, npiv, want_v=True)
            obj_h = obj.cpu().numpy()
            return self._winners([(float(lam[l]), all_piv, V[l], obj_h[l]) for l in range(lam.size)])
        # several penalties: one bounding pass for all of them (the histogram
        # is penalty-free; each penalty gets its own bounds from it)
        uniq = np.unique(lam[np.isfinite(lam)])
        if uniq.size > 1 and all(np.isfinite(lam)):
            # the per-penalty next ranges (8 B per (penalty, pivot, target)) let the
            # first refinement level continue instead of re-sampling
            keep_ranges = uniq.size * npiv * self.m * 8 <= (4 << 30) and os.environ.get("L1B200_SWEEP_RANGES", "1") != "0"
            if os.environ.get("L1B200_PY_SWEEP", "0") == "1":  # the same cascade driven from Python (cross-check)
                res = self.bound_pivots_multi(uniq, p_begin, p_stride, npiv, ranges=keep_ranges)
                rg = res[2] if keep_ranges else None
                return self._sweep_winners(lam, all_piv, res[0], res[1], uniq, ub_exchange, rg, npiv)
            return self.fit_lines_device(lam, p_begin, p_stride, npiv, ub_exchange, keep_ranges)
        for l in range(lam.size):
            lb, ub = self.bound_pivots(float(lam[l]), p_begin, p_stride, npiv)
            fresh = False
            top = float(np.min(ub))
            if ub_exchange is not None:
                top = float(ub_exchange(top))  # the best upper bound over every shard
            keep = np.nonzero(~(lb > self._prune_threshold(top)))[0]  # NaN-safe: keep unless provably worse
            if keep.size == 0:  # another shard holds a pivot provably better than all of ours
                self.last_candidates = 0
                out.append(None)
                continue
            seed, seed_n = keep, npiv  # positions in the last bound call's pivot list
            for level in range(REFINE_PASSES + (1 if fresh else 0)):
                if keep.size <= REFINE_MIN and not (fresh and level == 0):
                    break
                # refine the survivors: one more pass each, over the range
                # where the last pass proved each column's optimum lies, so
                # the bounds tighten by orders of magnitude per level (after
                # a multi-penalty pass: first one pass at this penalty alone)
                if fresh and level == 0:
                    lb2, ub2 = self.bound_pivot_list(float(lam[l]), all_piv[keep], passes=1)
                else:
                    lb2, ub2 = self.bound_pivot_list_continue(float(lam[l]), all_piv[keep], seed, seed_n)
                top = min(top, float(np.min(ub2)))
                sel = np.nonzero(~(lb2 > self._prune_threshold(top)))[0]
                keep, seed, seed_n = keep[sel], sel, keep.size
            self.last_candidates = int(keep.size)
            piv = all_piv[keep]
            # exact fits of the candidates, started on the ranges the bounds left
            V, err, pen, obj = self.fit_pivot_list_seeded(float(lam[l]), piv, seed, seed_n)
            out.append(self._winner(float(lam[l]), piv, V[0], obj.cpu().numpy()[0]))
        return out

    def fit_line_device(self, lam: float, p_begin: int = 0, p_stride: int = 1, npiv: int | None = None,
                        prune: bool | None = None, ub_exchange=None) -> PivotWinner | None:
        """shard_winners for one penalty via l1b_fit_line (the same cascade in C++).

        ``ub_exchange(top) -> global top`` is handed to the library as its
        exchange hook (called once, only when pruning; a shard whose pivots
        are all beaten returns None)."""
        if npiv is None:
            npiv = shard(self.m - p_begin, 0, p_stride)[2] if p_stride > 1 else self.m - p_begin
        piv, cand = ctypes.c_int64(), ctypes.c_int64()
        err, pen, obj = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        failed = []

        def _exchange(top, ctx):
            try:
                return float(ub_exchange(top))
            except BaseException as e:  # noqa: BLE001 -- re-raised after the C call
                failed.append(e)
                return float("nan")  # no threshold: nothing is pruned
        hook = _lib.UB_EXCHANGE_FN(0) if ub_exchange is None else _lib.UB_EXCHANGE_FN(_exchange)
        if ub_exchange is not None and prune is None:
            prune = self.auto_prune()  # every rank must take the same path
        with torch.cuda.device(self.device):
            v = torch.empty(self.m, dtype=torch.float64, device=self.device)
            rc = self.lib.l1b_fit_line(self.X.data_ptr(), self.n, self.m, float(lam), p_begin, p_stride, npiv,
                                       -1 if prune is None else int(bool(prune)), hook, None, ctypes.byref(piv),
                                       v.data_ptr(), ctypes.byref(err), ctypes.byref(pen), ctypes.byref(obj),
                                       ctypes.byref(cand), self.ws.data_ptr(), self.ws.numel(), self._s)
            if failed:
                raise failed[0]
            if rc == _lib.L1B_EINVAL and math.isinf(lam):
                raise ValueError(f"objective nan for lam={lam!r} (zero pivot column at infinite penalty)")
            _lib.check(rc, "l1b_fit_line")
            vh = v.cpu().numpy()
        self.last_candidates = int(cand.value)
        if piv.value < 0:
            return None
        return PivotWinner(int(piv.value), float(lam), vh, float(err.value), float(pen.value), float(obj.value))

    def fit_lines_device(self, lams, p_begin: int, p_stride: int, npiv: int, ub_exchange=None,
                         keep_ranges: bool = True) -> list[PivotWinner | None]:
        """A pruned penalty sweep (>= 2 distinct finite penalties) via l1b_fit_lines: the cascade of
        _sweep_winners in C++.  ``ub_exchange(tops) -> global tops`` (a vector over the distinct
        penalties) is handed to the library as its exchange hook."""
        lam = np.ascontiguousarray(np.asarray(lams, dtype=np.float64))
        L = int(np.unique(lam).size)
        failed = []

        def _exchange(ptr, count, ctx):
            try:
                a = np.ctypeslib.as_array(ptr, shape=(count,))
                a[:] = np.asarray(ub_exchange(a.copy()), dtype=np.float64).reshape(count)
            except BaseException as e:  # noqa: BLE001 -- re-raised after the C call
                failed.append(e)
        hook = _lib.UB_EXCHANGE_VEC_FN(0) if ub_exchange is None else _lib.UB_EXCHANGE_VEC_FN(_exchange)
        k = lam.size
        piv = np.zeros(k, dtype=np.int64)
        err, pen, obj = np.zeros(k), np.zeros(k), np.zeros(k)
        cand = ctypes.c_int64()
        with torch.cuda.device(self.device):
            bounds = torch.empty(2 * L * npiv, dtype=torch.float64, device=self.device)
            rg = torch.empty(L * npiv * self.m * 2, dtype=torch.float32, device=self.device) if keep_ranges else None
            V = torch.empty((k, self.m), dtype=torch.float64, device=self.device)
            dp = lambda a, t: a.ctypes.data_as(ctypes.POINTER(t))  # noqa: E731
            rc = self.lib.l1b_fit_lines(
                self.X.data_ptr(), self.n, self.m, dp(lam, ctypes.c_double), k, p_begin, p_stride, npiv, hook, None,
                bounds.data_ptr(), None if rg is None else rg.data_ptr(), 0 if rg is None else rg.numel() * 4,
                dp(piv, ctypes.c_int64), V.data_ptr(), dp(err, ctypes.c_double), dp(pen, ctypes.c_double),
                dp(obj, ctypes.c_double), ctypes.byref(cand), self.ws.data_ptr(), self.ws.numel(), self._s)
            if failed:
                raise failed[0]
            _lib.check(rc, "l1b_fit_lines")
            Vh = V.cpu().numpy()
        self.last_candidates = int(cand.value)
        return [None if piv[j] < 0 else PivotWinner(int(piv[j]), float(lam[j]), Vh[j].copy(), float(err[j]),
                                                    float(pen[j]), float(obj[j])) for j in range(k)]

    def auto_prune(self) -> bool:
        """Whether shard_winners bounds before fitting: the bound pass costs a
        pass of its own, not worth it for small fits.  Depends on the matrix
        only, so every rank of a sharded fit decides alike."""
        return self.m > 32 and self.m * self.m * self.n >= (1 << 24)

    def _prune_threshold(self, top: float) -> float:
        if not np.isfinite(top):
            return np.inf
        return top + PRUNE_RTOL * abs(top) + RESCORE_ATOL * self._abs_scale()

    def selftest_divide(self, n_pairs: int = 1 << 26, seed: int = 1) -> int:
        with torch.cuda.device(self.device):
            cnt = torch.zeros(1, dtype=torch.int64, device=self.device)
            _lib.check(self.lib.l1b_selftest_divide(seed, n_pairs, cnt.data_ptr(), self._s),
                       "l1b_selftest_divide")
            return int(cnt.item())
