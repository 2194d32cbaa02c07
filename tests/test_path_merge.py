"""Algorithm 3 (merge_path, path.py:166-277) on the device
(l1b_merge_path_device) against the reference's solution_path
(tests/golden/paths.npz), fed the reference's own breakpoint maps
(tests/golden/breakpoints.npz): every segment's bounds, line and objectives
bit for bit; and against the host C++ restatement (l1b_merge_path) on a
larger grid."""

import numpy as np
import pytest

from conftest import load_golden
from paper_2402_16712_b200 import DataMatrix
from paper_2402_16712_b200.path import PivotBreakpoints, PivotSolutions, merge_path

pytestmark = pytest.mark.gpu

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


def _host_merge(lam, sols, X):
    """l1b_merge_path (host C++, the same arithmetic) for cross-checking."""
    import ctypes

    from paper_2402_16712_b200 import _lib
    from paper_2402_16712_b200.path import _events, _snap_indices
    ep, et, ev, eb = _events(sols)
    k = _snap_indices(lam, eb)
    order = np.argsort(k, kind="stable")
    ep, et, ev = (np.ascontiguousarray(a[order]) for a in (ep, et, ev))
    off = np.ascontiguousarray(np.searchsorted(k[order], np.arange(lam.size + 1)).astype(np.int64))
    piv = np.asarray(sorted(sols.pivots), dtype=np.int64)
    deg = np.asarray(sorted(sols.degenerate), dtype=np.int64)
    n, m = X.shape
    cap = 1 << 16
    o = {nm: np.empty(cap) for nm in ("lo", "hi", "err", "pen", "obj", "zlo", "zhi")}
    opiv = np.empty(cap, dtype=np.int64)
    ov = np.empty((cap, m))
    cnt = ctypes.c_int64()
    P = lambda a: a.ctypes.data  # noqa: E731
    Xc = np.ascontiguousarray(X)
    lamc = np.ascontiguousarray(lam)
    rc = _lib.load().l1b_merge_path(P(Xc), n, m, P(lamc), lam.size, P(piv), piv.size, P(deg), deg.size, P(off),
                                    P(ep), P(et), P(ev), cap, P(o["lo"]), P(o["hi"]), P(opiv), P(ov), P(o["err"]),
                                    P(o["pen"]), P(o["obj"]), P(o["zlo"]), P(o["zhi"]), ctypes.byref(cnt))
    assert rc == 0
    c = int(cnt.value)
    return {k: v[:c] for k, v in o.items()}, opiv[:c], ov[:c]


def test_device_merge_equals_host_merge_and_fast_route():
    """400x40 (a 233k-weight grid): the device merge, the host C++ merge and the
    array-built solution_path give bit-identical segments."""
    import paper_2402_16712_b200 as l1b
    from paper_2402_16712_b200.path import major_breakpoints, solution_path
    d, _ = l1b.gen_line_data(40, 400, seed=0, noise_scale=1.0)
    X = np.array(d.values)
    lam, sols = major_breakpoints(d)
    dev = merge_path(lam, sols, d)
    host, hpiv, hv = _host_merge(lam, sols, X)
    fast = solution_path(d)
    for path in (dev, fast):
        segs = path.segments
        assert len(segs) == hpiv.size
        assert np.array_equal([s.line.preserved for s in segs], hpiv)
        assert np.asarray([s.line.v for s in segs]).tobytes() == hv.tobytes()
        for key, attr in (("lo", "lambda_lo"), ("hi", "lambda_hi"), ("zlo", "z_lo"), ("zhi", "z_hi")):
            assert np.asarray([getattr(s, attr) for s in segs]).tobytes() == host[key].tobytes(), key
        for key, attr in (("err", "error"), ("pen", "penalty_norm"), ("obj", "objective")):
            assert np.asarray([getattr(s.line, attr) for s in segs]).tobytes() == host[key].tobytes(), key
