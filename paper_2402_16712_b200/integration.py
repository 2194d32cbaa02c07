"""Route an installed reference package (``l1line``) through the GPU path.

The reference binds ``fit_line`` by value at import in several modules
(subspace.py:11, oracle.py:21, cli.py:22 -- SURVEY.md 8b), so rebinding the
package attribute alone would not redirect them.  ``use_gpu()`` patches every
binding site with wrappers that run this package's kernels and return the
reference's own ``FittedLine`` / ``SubspaceFit`` objects, so the reference's
CLI, oracle and tests run unchanged on the B200.
"""

from __future__ import annotations

import importlib

__all__ = ["use_gpu"]

_PATCHED = {}


def use_gpu(module: str = "l1line") -> None:
    """Patch ``l1line`` in place so fit_line / fit_for_pivot / fit_subspace, the sorted
    tableau (build_column / pivot_tableau) and the breakpoint maps (pivot_breakpoints /
    major_breakpoints, so solution_path too) use the GPU."""
    from . import api

    l1 = importlib.import_module(module)
    ref_core = importlib.import_module(f"{module}.core")

    def _conv(line):
        return ref_core.FittedLine(v=line.v, preserved=line.preserved, lam=line.lam,
                                   error=line.error, penalty_norm=line.penalty_norm,
                                   objective=line.objective)

    def fit_line(data, lam, threads=None):
        return _conv(api.fit_line(data, lam, threads))

    def fit_for_pivot(data, pivot, lam):
        return _conv(api.fit_for_pivot(data, pivot, lam))

    def fit_subspace(data, lam, k, threads=None):
        sub = importlib.import_module(f"{module}.subspace")
        fit = api.fit_subspace(data, lam, k, threads)
        return sub.SubspaceFit(tuple(_conv(c) for c in fit.components), fit.degenerate)

    def _ref_path():
        return importlib.import_module(f"{module}.path")

    def pivot_breakpoints(data, pivot):
        from . import path
        pb = path.pivot_breakpoints(data, pivot)
        return _ref_path().PivotBreakpoints(pivot=pb.pivot, entries=pb.entries, lambda_max=pb.lambda_max)

    def major_breakpoints(data, threads=None):
        # Algorithm 2 on the device; the reference's merge_path / solution_path
        # (Algorithm 3) then run unchanged on the result
        from . import path
        rp = _ref_path()
        grid, sols = path.major_breakpoints(data, threads)
        pivots = {p: rp.PivotBreakpoints(pivot=pb.pivot, entries=pb.entries, lambda_max=pb.lambda_max)
                  for p, pb in sols.pivots.items()}
        return grid, rp.PivotSolutions(data, pivots, sols.degenerate)

    def read_matrix(path, has_header=False):
        # the native CSV reader, returning the reference's own DataMatrix
        from . import io
        d = io.read_matrix(path, has_header)
        return ref_core.DataMatrix(d.values, column_names=d.column_names)

    def _conv_path(path):
        return ref_core.SolutionPath(tuple(
            ref_core.PathSegment(lambda_lo=sg.lambda_lo, lambda_hi=sg.lambda_hi, line=_conv(sg.line),
                                 z_lo=sg.z_lo, z_hi=sg.z_hi) for sg in path.segments))

    def merge_path(lambdas, solutions, data):
        from . import path
        return _conv_path(path.merge_path(lambdas, solutions, data))

    def solution_path(data, threads=None):
        from . import path
        return _conv_path(path.solution_path(data, threads))

    def build_column(data, pivot, target):
        # the device-sorted column as the reference's own RatioColumn
        from . import tableau
        c = tableau.build_column(data, pivot, target)
        return ref_core.RatioColumn(pivot=c.pivot, target=c.target, ratios=c.ratios, weights=c.weights,
                                    source_rows=c.source_rows, prefix_weights=c.prefix_weights,
                                    total_weight=c.total_weight)

    def pivot_tableau(data, pivot):
        from . import tableau
        rr = importlib.import_module(f"{module}.ratios")
        t = tableau.pivot_tableau(data, pivot)
        return rr.PivotTableau(pivot=t.pivot, targets=t.targets, ratios=t.ratios, weights=t.weights,
                               source_rows=t.source_rows, prefix=t.prefix, prefix_prev=t.prefix_prev,
                               totals=t.totals)

    targets = {
        "build_column": build_column,
        "pivot_tableau": pivot_tableau,
        "merge_path": merge_path,
        "solution_path": solution_path,
        "read_matrix": read_matrix,
        "fit_line": fit_line,
        "fit_for_pivot": fit_for_pivot,
        "fit_subspace": fit_subspace,
        "pivot_breakpoints": pivot_breakpoints,
        "major_breakpoints": major_breakpoints,
    }
    for modname in ("", ".ratios", ".fit", ".subspace", ".oracle", ".cli", ".path", ".io"):
        try:
            mod = importlib.import_module(module + modname)
        except ImportError:
            continue
        for name, fn in targets.items():
            if hasattr(mod, name):
                _PATCHED.setdefault((mod.__name__, name), getattr(mod, name))
                setattr(mod, name, fn)
    _ = l1


def restore() -> None:
    """Undo use_gpu()."""
    for (modname, name), fn in _PATCHED.items():
        setattr(importlib.import_module(modname), name, fn)
    _PATCHED.clear()
