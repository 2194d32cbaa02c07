"""B200-native sparse l1 best-fit lines (arXiv 2402.16712, Algorithm 1).

A drop-in for the hot path of the reference package ``l1line``: the same
``fit_line`` / ``fit_for_pivot`` / ``fit_subspace`` API and ``FittedLine``
results, computed by hand-written sm_100a CUDA kernels behind a C ABI
(``include/l1b200.h``).  Importing the package is cheap and works without a
GPU (types, data generation); the first fit loads ``csrc/libl1b200.so`` and
requires a CUDA device -- there is no CPU fallback.
"""

from .core import (DataMatrix, DualCertificate, EmptyPivotError, FittedLine, PathSegment, RatioColumn, SolutionPath,
                   SubspaceFit)
from .datagen import gen_line_data, gen_outlier_data, laplace

__version__ = "0.1.0"

_API = ("fit_line", "fit_lines", "fit_for_pivot", "degenerate_line", "fit_subspace", "deflate",
        "residual_error", "resolve_threads", "discordance", "l0_fraction")
_PATH = ("pivot_breakpoints", "major_breakpoints", "PivotBreakpoints", "PivotSolutions", "merge_path",
         "solution_path")
_CERT = ("certify_line", "check_line", "LineCertificate", "OptimalityRefuted")
_IO = ("read_matrix", "write_matrix", "CsvParseError", "write_path", "read_path", "write_sweep")
_VALIDATE = ("brute_force_column", "brute_force_pivot", "brute_force_line", "sweep_validate", "SweepReport")
_TABLEAU = ("build_column", "pivot_tableau", "PivotTableau", "window_bounds", "solve_column", "dual_certificate")

__all__ = ["DataMatrix", "DualCertificate", "EmptyPivotError", "FittedLine", "PathSegment", "RatioColumn", "SolutionPath",
           "SubspaceFit", "gen_line_data", "gen_outlier_data", "laplace", "use_gpu", *_API, *_PATH, *_CERT, *_IO,
           *_VALIDATE, *_TABLEAU, "__version__"]


def __getattr__(name):
    # The device API pulls in torch; load it on first use only.
    if name in _API:
        from . import api
        return getattr(api, name)
    if name in _PATH:
        from . import path
        return getattr(path, name)
    if name in _CERT:
        from . import certify
        return getattr(certify, name)
    if name in _IO:
        from . import io
        return getattr(io, name)
    if name in _VALIDATE:
        from . import validate
        return getattr(validate, name)
    if name in _TABLEAU:
        from . import tableau
        return getattr(tableau, name)
    if name == "use_gpu":
        from .integration import use_gpu
        return use_gpu
    raise AttributeError(name)
