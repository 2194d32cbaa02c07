"""Device-side optimality certificates (SURVEY.md 8f "next" row 3).

The reference certifies a column value with explicit dual multipliers
(``oracle.py:141-174``, ``dual_certificate``): feasibility, complementary
slackness and strong duality.  For the column problem
f_j(t) = sum_i |x_ij - t x_ip| + lam |t| such multipliers exist exactly when
0 lies in the subdifferential of f_j at t, which ``l1b_certify_columns``
checks for every column of a line at once with exact weight sums
(``csrc/path.cuh``).  ``certify_line`` returns the per-column slack;
``check_line`` raises ``OptimalityRefuted`` (as ``dual_certificate`` does)
naming the refuted columns.  Only the line's own pivot is certified, as in
the reference's use (``test_acceptance.py:87-102``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .api import _as_data, _engine

__all__ = ["OptimalityRefuted", "LineCertificate", "certify_line", "check_line"]


class OptimalityRefuted(Exception):
    """A claimed column value admits no feasible, complementary dual (oracle.py:35-36)."""


@dataclass(frozen=True)
class LineCertificate:
    pivot: int
    lam: float
    slack: np.ndarray       # per column, weight units; >= -tolerance certifies (inf: the pivot / degenerate)
    tolerance: np.ndarray
    refuted: tuple[int, ...]

    @property
    def ok(self) -> bool:
        return not self.refuted


def certify_line(data, line, lam: float | None = None, tol: float = 1e-9) -> LineCertificate:
    """Per-column optimality of ``line`` (a FittedLine: v, preserved, lam) at ``lam``.

    The tolerance mirrors ``oracle._verify`` (1e-9 * max(1, T_p, lam)) plus
    the fixed-point weights' rounding (n * 2^-s_p; zero on grid inputs).
    """
    d = _as_data(data)
    lam = float(line.lam if lam is None else lam)
    if not lam >= 0.0:
        raise ValueError("penalty weight must be nonnegative")
    p = int(line.preserved)
    v = np.ascontiguousarray(np.asarray(line.v, dtype=np.float64))
    if v.shape != (d.m,) or not np.all(np.isfinite(v)):
        raise ValueError("line direction must be a finite vector of length m")
    colp = np.abs(d.values[:, p])
    T = float(colp.sum())
    if not np.any(colp):  # degenerate pivot: the line must be the zero line (fit.py:66-72)
        bad = tuple(int(j) for j in np.nonzero(v)[0])
        return LineCertificate(p, lam, np.full(d.m, np.inf), np.zeros(d.m), bad)
    eng = _engine(data, d)
    with torch.cuda.device(eng.device):
        vd = torch.from_numpy(v).to(eng.device)
        sl = torch.empty(d.m, dtype=torch.float64, device=eng.device)
        _lib.check(eng.lib.l1b_certify_columns(eng.X.data_ptr(), eng.n, eng.m, p, vd.data_ptr(), lam,
                                               sl.data_ptr(), eng.ws.data_ptr(), eng.ws.numel(), eng._s),
                   "l1b_certify_columns")
        slack = sl.cpu().numpy()
    s_p = 51 - math.frexp(T)[1]
    tolv = np.full(d.m, tol * max(1.0, T, lam) + d.n * math.ldexp(1.0, -s_p))
    refuted = [int(j) for j in np.nonzero(slack < -tolv)[0]]
    if v[p] != 1.0:
        refuted = sorted(set(refuted) | {p})
    return LineCertificate(p, lam, slack, tolv, tuple(refuted))


def check_line(data, line, lam: float | None = None, tol: float = 1e-9) -> LineCertificate:
    """certify_line, raising OptimalityRefuted unless every column is certified."""
    cert = certify_line(data, line, lam, tol)
    if not cert.ok:
        raise OptimalityRefuted(
            f"pivot {cert.pivot} at lam={cert.lam}: columns {list(cert.refuted)[:16]} are not optimal")
    return cert
