"""Algorithm 3 (merge_path, path.py:166-277) natively (l1b_merge_path) against
the reference's solution_path (tests/golden/paths.npz), fed the reference's own
breakpoint maps (tests/golden/breakpoints.npz): every segment's bounds, line
and objectives bit for bit.  Host-only: runs without a GPU."""

import numpy as np
import pytest

from conftest import load_golden
from paper_2402_16712_b200 import DataMatrix
from paper_2402_16712_b200.path import PivotBreakpoints, PivotSolutions, merge_path

BP = load_golden("breakpoints.npz")
PATHS = load_golden("paths.npz")


def _solutions(name, X):
    pivots = {}
    for p in range(X.shape[1]):
        key = f"{name}_p{p}_entries"
        if key not in BP.files:
            continue
        rows = BP[key]
        entries = {}
        for t, bp, v in rows:
            entries.setdefault(int(t), []).append((float(bp), float(v)))
        lmax = {int(t): float(l) for t, l in BP[f"{name}_p{p}_lmax"]}
        pivots[p] = PivotBreakpoints(pivot=p, entries={t: tuple(e) for t, e in entries.items()}, lambda_max=lmax)
    return PivotSolutions(DataMatrix(X), pivots, tuple(int(p) for p in BP[f"{name}_degenerate"]))


@pytest.mark.parametrize("name", [str(n) for n in BP["names"]])
def test_merge_path_matches_reference(name):
    X = BP[f"{name}_X"]
    path = merge_path(BP[f"{name}_grid"], _solutions(name, X), X)
    segs = path.segments
    want = {k: PATHS[f"{name}_{k}"] for k in ("lo", "hi", "zlo", "zhi", "piv", "v", "err", "pen", "obj")}
    assert len(segs) == want["piv"].size, name
    got = {
        "lo": np.asarray([s.lambda_lo for s in segs]), "hi": np.asarray([s.lambda_hi for s in segs]),
        "zlo": np.asarray([s.z_lo for s in segs]), "zhi": np.asarray([s.z_hi for s in segs]),
        "piv": np.asarray([s.line.preserved for s in segs], dtype=np.int64),
        "v": np.asarray([s.line.v for s in segs]), "err": np.asarray([s.line.error for s in segs]),
        "pen": np.asarray([s.line.penalty_norm for s in segs]), "obj": np.asarray([s.line.objective for s in segs]),
    }
    for k in want:
        assert got[k].tobytes() == want[k].reshape(got[k].shape).tobytes(), (name, k)
    path.check_invariants()
