"""Pin the CPU oracle (test infrastructure) to the reference.

Every check compares oracle/ against vectors the reference produced
(tests/golden/make_golden.py) or against the reference's own known-answer
tests, bit for bit.  Only when this file passes may the oracle judge the GPU.
"""

import numpy as np
import pytest

import oracle
from conftest import TOY, iter_random_small, iter_random_small_lines, load_golden


def test_pairwise_sum_matches_numpy():
    # NumPy's pairwise reduction order (core.py:93 relies on it)
    rng = np.random.default_rng(0)
    for n in list(range(0, 300)) + [1000, 4097, 10_000, 123_457]:
        a = np.abs(rng.standard_normal(n)) * rng.uniform(0.1, 1e6, size=n)
        assert oracle.pairwise_sum(a) == float(a.sum()), n
    for shape in [(200, 50), (2000, 3), (333, 77)]:
        A = np.abs(rng.standard_normal(shape))
        assert oracle.pairwise_sum(A) == float(A.sum()), shape


def test_residual_error_kats(toy):
    # pkg/tests/test_core.py:54-66
    assert oracle.residual_error(toy, np.array([1.0, 0.0, 0.0, 0.0]), 0) == 41.0
    assert oracle.residual_error(toy, np.array([1.0, -0.5, 0.4, -1.0]), 0) == pytest.approx(36.1, abs=1e-12)
    assert oracle.residual_error(toy, np.zeros(4), 0) == 58.0


def test_residual_error_matches_numpy_formula():
    rng = np.random.default_rng(4)
    for _ in range(20):
        n, m = int(rng.integers(1, 300)), int(rng.integers(2, 40))
        X = rng.standard_normal((n, m)) * 10
        v = rng.standard_normal(m)
        p = int(rng.integers(m))
        want = float(np.abs(X - np.outer(X[:, p], v)).sum())
        assert oracle.residual_error(X, v, p) == want


def test_toy_column_sorted_with_weights(toy):
    # pkg/tests/test_ratios.py:8-17
    r, w, rows, pre = oracle.build_column(toy, 0, 3)
    assert r.tolist() == [-1.5, -1.0, -1.0, -0.2, 1.0 / 3.0]
    assert w.tolist() == [4.0, 2.0, 3.0, 5.0, 3.0]
    assert rows.tolist() == [0, 2, 3, 4, 1]
    assert pre.tolist() == [4.0, 6.0, 9.0, 14.0, 17.0]


def test_toy_column_values_at_known_weights(toy):
    # pkg/tests/test_fit.py:18-27 (boundaries at 1 inclusive and 11 dead)
    r, _, _, pre = oracle.build_column(toy, 0, 3)
    for lam, want in [(0.0, -1.0), (0.5, -1.0), (1.0, -0.2), (10.999, -0.2), (11.0, 0.0), (50.0, 0.0)]:
        assert oracle.solve_column(r, pre, lam) == want


def test_fit_for_pivot_known_lines(toy):
    # pkg/tests/test_fit.py:93-103
    line = oracle.fit_for_pivot(toy, 3, 0.0)
    assert line.v.tolist() == [-2.0 / 3.0, 1.0 / 3.0, -0.5, 1.0]
    assert line.error == 34.5 and line.penalty_norm == 2.5
    assert oracle.fit_for_pivot(toy, 0, 2.0).v.tolist() == [1.0, -0.5, 0.0, -0.2]
    assert oracle.fit_for_pivot(toy, 0, 5.0).v.tolist() == [1.0, 0.0, 0.0, -0.2]


def test_fit_line_toy_goldens(toy):
    # pkg/tests/test_fit.py:106-114, test_acceptance.py:80-84
    assert oracle.fit_line(toy, 0.0).preserved == 3
    assert oracle.fit_line(toy, 5.0).preserved == 0
    for lam, z in [(0.0, 34.5), (3.0, 42.0), (3.5, 43.0), (11.0, 52.0)]:
        assert oracle.fit_line(toy, lam).objective == pytest.approx(z, abs=1e-12)


def test_tie_prefers_smaller_pivot():
    X = np.array([[1.0, 1.0, 3.0], [2.0, 2.0, -1.0], [-1.0, -1.0, 2.0]])
    for lam in (0.0, 0.5, 2.0):
        assert oracle.fit_line(X, lam).preserved == 0


def test_zero_column_degenerates():
    X = np.array([[0.0, 2.0, 1.0], [0.0, -1.0, 3.0]])
    line = oracle.fit_for_pivot(X, 0, 1.0)
    assert not line.v.any() and line.error == float(np.abs(X).sum()) and line.penalty_norm == 0.0
    assert oracle.fit_line(X, 100.0).objective == float(np.abs(X).sum())


def test_random_small_golden_bit_exact():
    lvs = iter_random_small_lines()
    for t, X, lams, (pV, pE, pP, pO), lpiv, lobj, lerr, lpen in iter_random_small():
        V, E, P, O = oracle.fit_pivots(X, lams, threads=2)
        assert V.tobytes() == pV.tobytes(), t
        assert E.tobytes() == pE.tobytes() and P.tobytes() == pP.tobytes(), t
        assert O.tobytes() == pO.tobytes(), t
        lines = oracle.fit_line_multi(X, lams, threads=2)
        for k, line in enumerate(lines):
            assert line.preserved == lpiv[k], (t, k)
            assert line.objective == lobj[k] and line.error == lerr[k] and line.penalty_norm == lpen[k]
            assert line.v.tobytes() == lvs[t][k].tobytes()


@pytest.mark.parametrize("tag", ["raw", "grid"])
def test_c1_golden_bit_exact(tag):
    g = load_golden("c1.npz")
    X = g["X"] if tag == "raw" else g["Xq"]
    lams = g["lams"]
    V, E, P, O = oracle.fit_pivots(X, lams)
    assert V.tobytes() == g[f"{tag}_pV"].tobytes()
    assert O.tobytes() == g[f"{tag}_pO"].tobytes()
    for k, line in enumerate(oracle.fit_line_multi(X, lams)):
        assert line.preserved == g[f"{tag}_piv"][k]
        assert line.v.tobytes() == g[f"{tag}_v"][k].tobytes()
        assert line.objective == g[f"{tag}_obj"][k]


def test_grid_medium_golden_bit_exact():
    g = load_golden("grid_medium.npz")
    V, E, P, O = oracle.fit_pivots(g["X"], g["lams"])
    assert V.tobytes() == g["pV"].tobytes() and O.tobytes() == g["pO"].tobytes()


def test_subspace_golden():
    g = load_golden("subspace.npz")
    for tag in ("toy", "rand", "grid"):
        comps, degen = oracle.fit_subspace(g[f"{tag}_X"], float(g[f"{tag}_lam"]), int(g[f"{tag}_k"]))
        assert degen == bool(g[f"{tag}_degenerate"])
        assert [c.preserved for c in comps] == g[f"{tag}_piv"].tolist()
        assert np.array([c.v for c in comps]).tobytes() == g[f"{tag}_v"].tobytes()
        assert np.array([c.objective for c in comps]).tobytes() == g[f"{tag}_obj"].tobytes()
    comps, degen = oracle.fit_subspace(g["rank1_X"], 0.0, 2)
    assert degen and len(comps) == int(g["rank1_n"])


def test_thread_count_does_not_change_bits():
    # pkg/tests/test_fit.py:150-159 for the oracle's OpenMP loop
    rng = np.random.default_rng(3)
    X = rng.uniform(-10, 10, size=(25, 6))
    for lam in (0.0, 1.7, 8.0):
        base = oracle.fit_line(X, lam, threads=1)
        for t in (2, 4, 8):
            other = oracle.fit_line(X, lam, threads=t)
            assert other.v.tobytes() == base.v.tobytes() and other.objective == base.objective
