"""The reference's sorted-ratio API (``ratios.py``, ``fit.solve_column``,
``oracle.dual_certificate``) with the tableau built on the device.

* ``pivot_tableau(data, pivot)``            <- ratios.py:109-135 (``PivotTableau``)
* ``build_column(data, pivot, target)``     <- ratios.py:40-67 (``RatioColumn``)
* ``window_bounds(col, k)``                 <- ratios.py:70-86
* ``solve_column(col, lam)``                <- fit.py:27-48
* ``dual_certificate(col, value, lam)``     <- oracle.py:141-174 (``DualCertificate``)

The NumPy sort and cumsum the reference spends 84 % of a pivot fit on
(``ratios.py:119-125``) run in ``l1b_pivot_tableau``: exact
IEEE ratios, the stable (ratio, row) order with +-0 tied, and the prefix sums
accumulated sequentially in sorted order -- so every array is bit-identical to
the reference's.  What the reference then does on one column (a window test,
an O(n) multiplier construction) is plain arithmetic on those arrays and stays
on the host next to them: ``window_bounds`` / ``solve_column`` evaluate the
reference's formulas on the device-built column (the batched GPU versions of
the same test are the fit kernels), and ``dual_certificate`` assembles the
multipliers of the reference's KKT construction and checks them with the same
tolerances.  ``certify.certify_line`` is the batched device check of whole lines.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .api import _as_data, _check_lam, _engine
from .certify import OptimalityRefuted
from .core import DualCertificate, EmptyPivotError, RatioColumn

__all__ = ["EmptyPivotError", "RatioColumn", "PivotTableau", "DualCertificate", "build_column", "pivot_tableau",
           "window_bounds", "solve_column", "dual_certificate"]


@dataclass(frozen=True)
class PivotTableau:
    """Every ratio column of one pivot (ratios.py:89-106): column c describes
    target ``targets[c]``; rows are sorted positions."""

    pivot: int
    targets: np.ndarray
    ratios: np.ndarray
    weights: np.ndarray
    source_rows: np.ndarray
    prefix: np.ndarray
    prefix_prev: np.ndarray
    totals: np.ndarray


def _pair_ok(m: int, pivot: int, target: int) -> None:
    """ratios.py:31-37: index errors first, then the pivot == target case."""
    if not 0 <= pivot < m:
        raise IndexError(f"pivot column {pivot} out of range")
    if not 0 <= target < m:
        raise IndexError(f"target column {target} out of range")
    if pivot == target:
        raise ValueError("pivot and target must differ")


def build_column(data, pivot: int, target: int) -> RatioColumn:
    """Sorted ratios of one target column against a pivot (ratios.py:40-67)."""
    d = _as_data(data)
    pivot, target = int(pivot), int(target)
    _pair_ok(d.m, pivot, target)
    tab = _engine(data, d).tableau(pivot, target)
    if tab is None:
        raise EmptyPivotError(f"column {pivot} is identically zero")
    r, w, pre, rows = (a[0] for a in tab)
    return RatioColumn(pivot=pivot, target=target, ratios=r, weights=w, source_rows=rows, prefix_weights=pre,
                       total_weight=float(pre[-1]))


def pivot_tableau(data, pivot: int) -> PivotTableau:
    """All ratio columns of one pivot (ratios.py:109-135), arrays [n_p][m - 1]."""
    d = _as_data(data)
    pivot = int(pivot)
    if not 0 <= pivot < d.m:
        raise IndexError(f"pivot column {pivot} out of range")
    tab = _engine(data, d).tableau(pivot)
    if tab is None:
        raise EmptyPivotError(f"column {pivot} is identically zero")
    r, w, pre, rows = (np.ascontiguousarray(a.T) for a in tab)
    prev = np.zeros_like(pre)
    prev[1:] = pre[:-1]
    return PivotTableau(pivot=pivot, targets=np.array([j for j in range(d.m) if j != pivot], dtype=np.intp),
                        ratios=r, weights=w, source_rows=rows.astype(np.intp), prefix=pre, prefix_prev=prev,
                        totals=pre[-1].copy())


def window_bounds(col: RatioColumn, k: int) -> tuple[float, float]:
    """Admission window (lower, upper] of sorted position k (ratios.py:70-86):
    lower = T - 2 P[k], upper = T - 2 P[k-1] (T for k = 0)."""
    if not 0 <= k < len(col):
        raise IndexError(f"position {k} out of range for column of {len(col)}")
    T = col.total_weight
    below = float(col.prefix_weights[k - 1]) if k else 0.0
    return T - 2.0 * float(col.prefix_weights[k]), T - 2.0 * below


def solve_column(col: RatioColumn, lam: float) -> float:
    """Optimal v_j of one column (fit.py:27-48): the position whose window holds
    sign(ratio) * lam (zero ratios probe +lam); 0.0 when none does."""
    lam = _check_lam(lam)
    T = col.total_weight
    edges = T - 2.0 * col.prefix_weights          # lower bound of each window
    tops = np.concatenate(([T], edges[:-1]))      # upper bound (the previous lower)
    probe = np.where(col.ratios >= 0.0, lam, -lam)
    inside = np.flatnonzero((edges < probe) & (probe <= tops))
    if __debug__:
        assert inside.size <= 1, "admission windows overlapped"
    return float(col.ratios[inside[0]]) if inside.size else 0.0


def _kkt_failures(col: RatioColumn, value: float, lam: float, pi: np.ndarray, gamma: float) -> list[str]:
    """The conditions oracle.py:93-116 checks, with its tolerance 1e-9 * max(1, T, lam):
    box feasibility, balance, complementary slackness, |gamma| = lam off zero, zero gap."""
    tol = 1e-9 * max(1.0, col.total_weight, lam)
    w, r = col.weights, col.ratios
    out = []
    if (np.abs(pi) > w + tol).any():
        out.append("multiplier exceeds its weight box")
    if abs(gamma) > lam + tol:
        out.append("penalty multiplier exceeds lam")
    if abs(float(pi.sum()) + gamma) > tol:
        out.append("multipliers do not balance")
    if ((np.abs(pi) < w - tol) & (np.abs(r - value) * w > tol)).any():
        out.append("slack multiplier on a nonzero residual")
    if value != 0.0 and abs(abs(gamma) - lam) > tol:
        out.append("nonzero snap value needs |gamma| == lam")
    primal = float((w * np.abs(r - value)).sum() + lam * abs(value))
    gap = primal - float((r * pi).sum())
    if abs(gap) > 1e-9 * max(1.0, abs(primal)):
        out.append(f"duality gap {gap:.3e}")
    return out


def dual_certificate(col: RatioColumn, value: float, lam: float) -> DualCertificate:
    """Dual multipliers proving ``value`` optimal for the column at ``lam``
    (oracle.py:141-174), or OptimalityRefuted naming what fails.

    A value at sorted position k: rows below k pull with -w, rows above with
    +w, gamma = -sgn(r_k) lam, and row k balances the rest.  The value 0 (a
    killed column): every row at its signed weight, the zero ratios absorbing
    as much of the imbalance as their boxes allow, gamma the remainder.
    """
    if lam < 0.0:
        raise ValueError("penalty weight must be nonnegative")
    lam = float(lam)
    n = len(col)
    failed = []
    for k in np.flatnonzero(col.ratios == value):
        gamma = (-1.0 if col.ratios[k] >= 0.0 else 1.0) * lam
        pi = np.where(np.arange(n) > k, col.weights, -col.weights)
        pi[k] = -gamma - (float(pi.sum()) - float(pi[k]))
        why = _kkt_failures(col, value, lam, pi, gamma)
        if not why:
            return DualCertificate(pivot=col.pivot, target=col.target, lam=lam, pi=pi, gamma=gamma)
        failed.append(f"position {k}: " + "; ".join(why))
    if value == 0.0:
        pi = col.weights * np.sign(col.ratios)
        rest = float(pi.sum())
        for i in np.flatnonzero(col.ratios == 0.0):
            take = float(np.clip(-rest, -col.weights[i], col.weights[i]))
            pi[i] = take
            rest += take
        gamma = -float(pi.sum())
        why = _kkt_failures(col, value, lam, pi, gamma)
        if not why:
            return DualCertificate(pivot=col.pivot, target=col.target, lam=lam, pi=pi, gamma=gamma)
        failed.append("killed column: " + "; ".join(why))
    if not failed:
        failed.append("value matches no ratio and is not zero")
    raise OptimalityRefuted(f"column {col.target} vs pivot {col.pivot} at lam={lam}: " + " | ".join(failed))
