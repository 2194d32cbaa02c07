"""The reference's optimality checks on the device (SURVEY.md 8f "next" row 3):
``brute_force_column`` / ``brute_force_pivot`` / ``brute_force_line`` and
``sweep_validate`` / ``SweepReport`` (``oracle.py:39-224``).

The brute force evaluates the column objective at every kink candidate
(``l1b_brute_force_columns``: O(n^2) per column, summed over the rows in the
reference's order) -- a route independent of the sort-free solver that
``fit_line`` uses; ``sweep_validate`` compares a solution path, ``fit_line``
and the brute force on a weight grid, as the reference does, at sizes its
Python loops cannot reach.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .api import _as_data, _check_lam, _engine, fit_lines
from .core import EmptyPivotError, FittedLine
from .engine import DeviceFit

__all__ = ["brute_force_column", "brute_force_pivot", "brute_force_line", "sweep_validate", "SweepReport"]


def _columns(eng: DeviceFit, pivot: int, lam: float):
    with torch.cuda.device(eng.device):
        t = torch.empty(eng.m - 1, dtype=torch.float64, device=eng.device)
        f = torch.empty_like(t)
        _lib.check(eng.lib.l1b_brute_force_columns(eng.X.data_ptr(), eng.n, eng.m, int(pivot), float(lam),
                                                   t.data_ptr(), f.data_ptr(), eng._s), "l1b_brute_force_columns")
        return t.cpu().numpy(), f.cpu().numpy()


def brute_force_column(data, pivot: int, target: int, lam: float) -> tuple[float, float]:
    """min_t sum_i |x_it - t x_ip| + lam |t| over the kinks (oracle.py:39-58): (t, f(t))."""
    if lam < 0.0:
        raise ValueError("penalty weight must be nonnegative")
    d = _as_data(data)
    if not np.any(d.values[:, pivot]):
        raise EmptyPivotError(f"column {pivot} is identically zero")
    t, f = _columns(_engine(data, d), pivot, lam)
    c = target if target < pivot else target - 1
    return float(t[c]), float(f[c])


def _pivot_line(eng: DeviceFit, d, pivot: int, lam: float) -> FittedLine:
    if not np.any(d.values[:, pivot]):
        v = np.zeros(d.m)
    else:
        t, _ = _columns(eng, pivot, lam)
        v = np.insert(t, pivot, 1.0)
    with torch.cuda.device(eng.device):
        err = eng.residual_exact(torch.from_numpy(v).to(eng.device), pivot)
    pen = float(np.abs(v).sum())
    return FittedLine(v=v, preserved=pivot, lam=float(lam), error=err, penalty_norm=pen, objective=err + lam * pen)


def brute_force_pivot(data, pivot: int, lam: float) -> FittedLine:
    """One pivot's line, column by column by brute force (oracle.py:61-71)."""
    d = _as_data(data)
    return _pivot_line(_engine(data, d), d, int(pivot), float(lam))


def brute_force_line(data, lam: float) -> FittedLine:
    """Minimum over pivots of the brute-force lines (oracle.py:74-81)."""
    d = _as_data(data)
    eng = _engine(data, d)
    best = None
    for p in range(d.m):
        line = _pivot_line(eng, d, p, float(lam))
        if best is None or line.objective < best.objective:
            best = line
    return best


@dataclass
class SweepReport:
    """Cross-validation of a solution path on a grid of weights (oracle.py:177-190)."""

    lambdas: np.ndarray
    path_objectives: np.ndarray
    fit_objectives: np.ndarray
    brute_objectives: np.ndarray
    max_rel_discrepancy: float
    failures: list = field(default_factory=list)

    @property
    def ok(self) -> bool:
        return not self.failures and self.max_rel_discrepancy <= 1e-9


def sweep_validate(data, path, grid_size: int = 200, threads: int | None = None) -> SweepReport:
    """The path against fresh fits and the brute force on [0, 1.1 max breakpoint]
    (oracle.py:193-224); the fits of the grid run as one batched sweep."""
    d = _as_data(data)
    failures = []
    try:
        path.check_invariants()
    except ValueError as bad:
        failures.append(str(bad))
    hi = 1.1 * path.breakpoints[-1] if path.breakpoints else 1.0
    grid = np.linspace(0.0, hi, grid_size)
    z_path = np.array([path.objective_at(lam) for lam in grid])
    z_fit = np.array([ln.objective for ln in fit_lines(d, [_check_lam(x) for x in grid], threads)])
    z_brute = np.array([brute_force_line(d, lam).objective for lam in grid])
    scale = np.maximum(1.0, np.abs(z_brute))
    rel = np.maximum(np.abs(z_path - z_fit), np.abs(z_path - z_brute)) / scale
    worst = int(np.argmax(rel))
    if rel[worst] > 1e-9:
        failures.append(f"objective mismatch {rel[worst]:.3e} at lam={grid[worst]!r}")
    return SweepReport(lambdas=grid, path_objectives=z_path, fit_objectives=z_fit, brute_objectives=z_brute,
                       max_rel_discrepancy=float(rel[worst]), failures=failures)
