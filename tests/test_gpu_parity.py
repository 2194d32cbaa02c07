"""GPU parity: the CUDA path against the reference's goldens and the oracle.

Bar (BASELINE.json north_star): pivot, selected ratios and sparsity pattern
exactly; objective and directions within 1e-5 relative.  We hold a tighter
bar: directions bit-identical to the reference on every input whose prefix
sums are exact in f64 (all goldens, grid-quantised data, integer data), and
the winning line's error / penalty / objective bit-identical whenever its
direction is (the winner is re-scored in NumPy's summation order).  On raw
data the direction is compared tie-aware: a differing column
is accepted only if both values give the same column objective to 1e-12.
"""

import math

import numpy as np
import pytest
import torch

import oracle
import paper_2402_16712_b200 as l1b
from conftest import TOY, iter_random_small, iter_random_small_lines, load_golden
from paper_2402_16712_b200.engine import DeviceFit, shard

pytestmark = pytest.mark.gpu

OBJ_RTOL = 1e-12
# Per-pivot objectives are reduced in a fixed device order, not NumPy's, so
# they match to rounding: relative 1e-12, plus an absolute floor of 1e-13 of
# sum|X| for objectives that are (near) zero.  The winner's objective is
# re-scored in NumPy's order and compared bit for bit.
OBJ_ATOL = 1e-13


def assert_obj_close(O, Oref, X, rtol=OBJ_RTOL):
    np.testing.assert_allclose(O, Oref, rtol=rtol, atol=OBJ_ATOL * float(np.abs(X).sum()) + 1e-300)


def _col_obj(X, p, j, t, lam):
    return float(np.abs(X[:, j] - t * X[:, p]).sum()) + lam * abs(t)


def _assert_v_tie_aware(X, p, lam, got, want, what=""):
    if got.tobytes() == want.tobytes():
        return 0
    bad = np.nonzero(got.view(np.int64) != want.view(np.int64))[0]
    for j in bad:
        a, b = _col_obj(X, p, j, got[j], lam), _col_obj(X, p, j, want[j], lam)
        assert abs(a - b) <= 1e-12 * max(1.0, abs(b)), (what, p, j, got[j], want[j], a, b)
    return len(bad)


def _pivots(X, lams, **kw):
    eng = DeviceFit(X)
    V, E, P, O = eng.fit_pivots(lams, **kw)
    torch.cuda.synchronize()
    return eng, V.cpu().numpy(), E.cpu().numpy(), P.cpu().numpy(), O.cpu().numpy()


@pytest.mark.parametrize("n,m", [(1, 3), (2, 3), (37, 11), (61, 7), (129, 5), (300, 17), (2000, 2000), (3000, 7001),
                                 (100000, 500)])
def test_residual_exact_matches_numpy_bits(n, m):
    """l1b_residual_exact == residual_error (core.py:93) bit for bit, up to C4's n*m."""
    rng = np.random.default_rng(n + m)
    X = rng.standard_normal((n, m))
    v = rng.standard_normal(m)
    p = m // 2
    v[p] = 1.0
    want = float(np.abs(X - np.outer(X[:, p], v)).sum())
    eng = DeviceFit(X, max_pivots=1)
    got = eng.residual_exact(torch.from_numpy(v).to(eng.device), p)
    assert got == want, (got, want)


def test_division_selftest_bit_exact():
    eng = DeviceFit(TOY)
    assert eng.selftest_divide(n_pairs=1 << 28, seed=7) == 0


# ------------------------------------------------------ reference KATs --

def test_fit_for_pivot_known_lines():
    # pkg/tests/test_fit.py:93-103
    line = l1b.fit_for_pivot(TOY, 3, 0.0)
    assert line.v.tolist() == [-2.0 / 3.0, 1.0 / 3.0, -0.5, 1.0]
    assert line.error == 34.5 and line.penalty_norm == 2.5
    assert l1b.fit_for_pivot(TOY, 0, 2.0).v.tolist() == [1.0, -0.5, 0.0, -0.2]
    assert l1b.fit_for_pivot(TOY, 0, 5.0).v.tolist() == [1.0, 0.0, 0.0, -0.2]


def test_toy_column_walk():
    # pkg/tests/test_fit.py:18-27: column (p=0, j=3) -1 -> -1/5 -> 0 at lam 1 and 11
    for lam, want in [(0.0, -1.0), (0.5, -1.0), (1.0, -0.2), (10.999, -0.2), (11.0, 0.0), (50.0, 0.0)]:
        assert l1b.fit_for_pivot(TOY, 0, lam).v[3] == want


def test_fit_line_toy_goldens():
    # pkg/tests/test_fit.py:106-114, test_acceptance.py:80-84
    assert l1b.fit_line(TOY, 0.0).preserved == 3
    assert l1b.fit_line(TOY, 5.0).preserved == 0
    for lam in (0.0, 1.0, 2.5, 3.5, 7.0, 12.0):
        got, want = l1b.fit_line(TOY, lam), oracle.fit_line(TOY, lam)
        assert (got.preserved, got.v.tobytes(), got.objective) == (want.preserved, want.v.tobytes(), want.objective)
    for lam, z in [(0.0, 34.5), (3.0, 42.0), (3.5, 43.0), (11.0, 52.0)]:
        assert l1b.fit_line(TOY, lam).objective == pytest.approx(z, abs=1e-12)


def test_tie_prefers_smaller_pivot():
    X = np.array([[1.0, 1.0, 3.0], [2.0, 2.0, -1.0], [-1.0, -1.0, 2.0]])
    for lam in (0.0, 0.5, 2.0):
        assert l1b.fit_line(X, lam).preserved == 0


def test_zero_column_and_zero_line():
    # pkg/tests/test_fit.py:125-147
    X = np.array([[0.0, 2.0, 1.0], [0.0, -1.0, 3.0]])
    line = l1b.fit_for_pivot(X, 0, 1.0)
    assert not line.v.any() and line.error == float(np.abs(X).sum()) and line.penalty_norm == 0.0
    assert l1b.fit_line(X, 0.0).preserved in (1, 2)
    big = l1b.fit_line(X, 100.0)
    assert not big.v.any() and big.objective == float(np.abs(X).sum())


def test_infinite_lambda():
    got, want = l1b.fit_line(TOY, math.inf), oracle.fit_line(TOY, math.inf)
    assert got.preserved == want.preserved == 0
    assert got.v.tobytes() == want.v.tobytes() and got.error == want.error and math.isinf(got.objective)


# ------------------------------------------------------------- goldens --

def test_random_small_golden():
    lvs = iter_random_small_lines()
    for t, X, lams, (pV, pE, pP, pO), lpiv, lobj, lerr, lpen in iter_random_small():
        if X.shape[0] < 1:
            continue
        _, V, E, P, O = _pivots(X, lams)
        V = V.transpose(1, 0, 2)  # [m][L][m] like the golden
        assert V.tobytes() == pV.tobytes(), t
        assert_obj_close(O.T, pO, X)
        lines = l1b.fit_lines(X, lams)
        for k, line in enumerate(lines):
            assert line.preserved == lpiv[k], (t, k)
            assert line.v.tobytes() == lvs[t][k].tobytes(), (t, k)
            assert (line.objective, line.error, line.penalty_norm) == (lobj[k], lerr[k], lpen[k]), (t, k)


@pytest.mark.parametrize("tag", ["raw", "grid"])
def test_c1_golden(tag):
    g = load_golden("c1.npz")
    X = g["X"] if tag == "raw" else g["Xq"]
    lams = g["lams"]
    _, V, E, P, O = _pivots(X, lams)
    assert V.transpose(1, 0, 2).tobytes() == g[f"{tag}_pV"].tobytes()
    assert_obj_close(O.T, g[f"{tag}_pO"], X)
    for k, line in enumerate(l1b.fit_lines(X, lams)):
        assert line.preserved == g[f"{tag}_piv"][k]
        assert line.v.tobytes() == g[f"{tag}_v"][k].tobytes()
        assert line.objective == g[f"{tag}_obj"][k] and line.error == g[f"{tag}_err"][k]


def test_grid_medium_golden():
    g = load_golden("grid_medium.npz")
    _, V, E, P, O = _pivots(g["X"], g["lams"])
    assert V.transpose(1, 0, 2).tobytes() == g["pV"].tobytes()
    assert_obj_close(O.T, g["pO"], g["X"])
    for k, line in enumerate(l1b.fit_lines(g["X"], g["lams"])):
        assert line.preserved == g["l_piv"][k] and line.objective == g["l_obj"][k]


def test_subspace_golden():
    g = load_golden("subspace.npz")
    for tag in ("toy", "rand", "grid"):
        fit = l1b.fit_subspace(g[f"{tag}_X"], float(g[f"{tag}_lam"]), int(g[f"{tag}_k"]))
        assert fit.degenerate == bool(g[f"{tag}_degenerate"])
        piv = [c.preserved for c in fit.components]
        assert piv == g[f"{tag}_piv"].tolist(), tag
        # component 1 is bit-exact; later ones see device-deflated data whose
        # rounding differs from BLAS dgemv at the 1e-16 level
        c0 = fit.components[0]
        assert c0.v.tobytes() == g[f"{tag}_v"][0].tobytes() and c0.objective == g[f"{tag}_obj"][0]
        np.testing.assert_allclose([c.objective for c in fit.components], g[f"{tag}_obj"], rtol=1e-9)
        np.testing.assert_allclose(np.array([c.v for c in fit.components]), g[f"{tag}_v"], rtol=1e-9, atol=1e-12)
    fit = l1b.fit_subspace(g["rank1_X"], 0.0, 2)
    assert fit.degenerate and len(fit) == int(g["rank1_n"])


# --------------------------------------------------- oracle at scale --

def _grid(X, bits=20):
    return np.round(X * 2.0**bits) / 2.0**bits


@pytest.mark.parametrize("n,m,seed", [(400, 48, 0), (3000, 24, 1), (1, 6, 2), (7, 2, 3), (1000, 33, 4),
                                      (6000, 16, 5),     # two selection passes (n > 4096)
                                      (70000, 10, 6)])   # three passes, 32-bit row indices (n > 65535)
def test_grid_data_bit_exact_vs_oracle(n, m, seed):
    d, _ = l1b.gen_line_data(m, n, seed=seed, noise_scale=1.0)
    X = _grid(d.values)
    lams = [0.0, 1.0, 0.3 * float(np.abs(X).sum(axis=0).max()), 1e9]
    _, V, E, P, O = _pivots(X, lams)
    Vo, Eo, Po, Oo = oracle.fit_pivots(X, lams)
    assert V.transpose(1, 0, 2).tobytes() == Vo.tobytes()
    assert_obj_close(O.T, Oo, X, rtol=1e-11)
    for k, line in enumerate(l1b.fit_lines(X, lams)):
        want = oracle.fit_line(X, lams[k])
        assert line.preserved == want.preserved and line.v.tobytes() == want.v.tobytes()
        assert line.objective == want.objective


@pytest.mark.parametrize("kind", ["integers", "sparse", "signed_zeros", "duplicate_rows", "noiseless"])
def test_adversarial_ties_vs_oracle(kind):
    """Exercises the tie paths: 64-bit refinement, the +-0 group in row order."""
    rng = np.random.default_rng(hash(kind) % 2**32)
    n, m = 600, 20
    if kind == "integers":
        X = np.round(rng.uniform(-4, 4, size=(n, m)))
    elif kind == "sparse":
        X = np.round(rng.uniform(-10, 10, size=(n, m)) * 8) / 8   # dyadic: prefix sums exact
        X[rng.random(X.shape) < 0.7] = 0.0
    elif kind == "signed_zeros":
        X = np.round(rng.uniform(-3, 3, size=(n, m)))
        X[rng.random(X.shape) < 0.4] = -0.0
    elif kind == "duplicate_rows":
        base = np.round(rng.uniform(-10, 10, size=(40, m)) * 64) / 64
        X = base[rng.integers(0, 40, size=n)]
    else:  # rank one: every ratio of a column identical up to rounding
        X = np.outer(rng.uniform(-100, 100, size=n), rng.uniform(-1, 1, size=m))
    lams = [0.0, 0.5, 3.0, 50.0]
    _, V, E, P, O = _pivots(X, lams)
    Vo, Eo, Po, Oo = oracle.fit_pivots(X, lams)
    if kind == "noiseless":
        # raw products: prefix sums are not exact, compare tie-aware
        for p in range(m):
            for k, lam in enumerate(lams):
                _assert_v_tie_aware(X, p, lam, V[k, p], Vo[p, k], kind)
    else:
        assert V.transpose(1, 0, 2).tobytes() == Vo.tobytes()
    np.testing.assert_allclose(O.T, Oo, rtol=1e-10, atol=1e-9)


def test_extreme_exponents_take_exact_division_path():
    rng = np.random.default_rng(9)
    X = rng.uniform(-10, 10, size=(300, 12))
    X[:, 3] *= 2.0**600
    X[:, 7] *= 2.0**-700
    X[5, 2] = 5e-324  # a subnormal entry
    lams = [0.0, 2.0]
    _, V, E, P, O = _pivots(X, lams)
    Vo, Eo, Po, Oo = oracle.fit_pivots(X, lams)
    for p in range(X.shape[1]):
        for k, lam in enumerate(lams):
            _assert_v_tie_aware(X, p, lam, V[k, p], Vo[p, k], "extreme")
    assert_obj_close(O.T, Oo, X, rtol=1e-10)


def test_raw_c2_shape_sampled_pivots_vs_oracle():
    """Full 2000 x 2000 C2 input: every pivot on the GPU, 12 sampled on the CPU."""
    d, _ = l1b.gen_line_data(2000, 2000, seed=0, noise_scale=1.0)
    X = d.values
    eng = DeviceFit(X)
    V, E, P, O = eng.fit_pivots([1.0])
    V, O = V.cpu().numpy()[0], O.cpu().numpy()[0]
    best = int(np.argmin(O))
    sample = sorted({0, 1, 1329, 308, best, 1999, *np.random.default_rng(0).integers(0, 2000, 6).tolist()})
    for p in sample:
        want = oracle.fit_for_pivot(X, p, 1.0)
        nbad = _assert_v_tie_aware(X, p, 1.0, V[p], want.v, "c2")
        assert nbad <= 2
        assert O[p] == pytest.approx(want.objective, rel=1e-11)
    line = eng.shard_winners([1.0])[0]
    # C2 at lam=1 -> pivot 1329, z = 4561881.260523822
    assert line.pivot == 1329
    assert line.objective == pytest.approx(4561881.260523822, rel=1e-12)


def test_grid_c2_winner_bit_exact():
    d, _ = l1b.gen_line_data(2000, 2000, seed=0, noise_scale=1.0)
    X = _grid(d.values)
    eng = DeviceFit(X)
    win = eng.shard_winners([1.0, 2500.0])
    for w in win:
        want = oracle.fit_for_pivot(X, w.pivot, w.lam)
        assert w.v.tobytes() == want.v.tobytes()
        assert (w.error, w.penalty_norm, w.objective) == (want.error, want.penalty_norm, want.objective)


def test_batched_lambdas_equal_single_calls_and_are_deterministic():
    d, _ = l1b.gen_outlier_data(50, 200, 20, seed=0)
    X = d.values
    lams = [0.0, 0.1, 7.5, 120.0, 900.0]
    eng = DeviceFit(X)
    V1, _, _, O1 = eng.fit_pivots(lams)
    V2, _, _, O2 = eng.fit_pivots(lams)
    assert torch.equal(V1, V2) and torch.equal(O1, O2)
    for k, lam in enumerate(lams):
        Vs, _, _, Os = eng.fit_pivots([lam])
        assert torch.equal(Vs[0], V1[k]) and torch.equal(Os[0], O1[k])
    # sharded pivots give byte-identical per-pivot results
    for stride in (2, 3):
        for r in range(stride):
            npiv = (50 - r + stride - 1) // stride
            Vs, _, _, Os = eng.fit_pivots(lams, p_begin=r, p_stride=stride, npiv=npiv)
            assert torch.equal(Vs, V1[:, r::stride]) and torch.equal(Os, O1[:, r::stride])


def test_use_gpu_patches_reference_bindings():
    import sys
    import types
    # a stand-in for an installed l1line with by-value bindings
    core = types.ModuleType("fake_l1line.core")
    core.FittedLine = l1b.FittedLine
    pkg = types.ModuleType("fake_l1line")
    pkg.fit_line = None
    pkg.__path__ = []
    sub = types.ModuleType("fake_l1line.subspace")
    sub.fit_line = None
    sub.SubspaceFit = l1b.SubspaceFit
    from paper_2402_16712_b200 import path as our_path
    pth = types.ModuleType("fake_l1line.path")
    pth.major_breakpoints = None
    pth.PivotBreakpoints = our_path.PivotBreakpoints
    pth.PivotSolutions = our_path.PivotSolutions
    sys.modules.update({"fake_l1line": pkg, "fake_l1line.core": core, "fake_l1line.subspace": sub,
                        "fake_l1line.path": pth})
    try:
        from paper_2402_16712_b200.integration import restore, use_gpu
        use_gpu("fake_l1line")
        assert pkg.fit_line(TOY, 0.0).preserved == 3 and sub.fit_line(TOY, 5.0).preserved == 0
        grid, sols = pth.major_breakpoints(l1b.DataMatrix(TOY))  # what solution_path calls (path.py:280-282)
        assert grid.tolist() == [0.0, 1.0, 2.0, 3.0, 4.0, 5.0, 6.0, 11.0] and sorted(sols.pivots) == [0, 1, 2, 3]
        restore()
        assert pkg.fit_line is None and pth.major_breakpoints is None
    finally:
        for k in ("fake_l1line", "fake_l1line.core", "fake_l1line.subspace", "fake_l1line.path"):
            sys.modules.pop(k, None)


# ---------------------------------------------------- pivot pruning bounds --

def _bounds_hold(X, lam):
    eng = DeviceFit(X)
    _, _, _, O = eng.fit_pivots([lam], want_v=False)
    o = O.cpu().numpy()[0]
    tol = 1e-12 * np.abs(o) + OBJ_ATOL * float(np.abs(X).sum())
    # fit_line's lean first pass (per-pivot sums only), unsteered and steered
    for steer in (0, 2):
        lb, ub = eng.bound_pivot_sums(lam, steer=steer)
        assert np.all(lb <= o + tol), (lam, steer, np.max(lb - o))
        assert np.all(o <= ub + tol), (lam, steer, np.max(o - ub))
    lb, ub = eng.bound_pivots(lam)
    assert np.all(lb <= o + tol), (lam, np.max(lb - o))
    assert np.all(o <= ub + tol), (lam, np.max(o - ub))
    # per column: lb_pj <= f_pj* <= ub_pj with f_pj* from the exact directions
    V, _, _, _ = eng.fit_pivots([lam], want_v=True)
    V = V.cpu().numpy()[0]
    F = np.abs(X[None, :, :] - X.T[:, :, None] * V[:, None, :]).sum(axis=1) + lam * np.abs(V)
    F[np.arange(X.shape[1]), np.arange(X.shape[1])] = 0.0  # the pivot's own column: v = 1, no error
    ftol = 1e-12 * F + OBJ_ATOL * float(np.abs(X).sum())
    cols = bool(np.all(np.isfinite(lb)))  # outside the FP32 window nothing is bounded per column
    if cols:
        lbc, ubc = eng.bound_columns(X.shape[1])
        np.fill_diagonal(lbc, 0.0)
        np.fill_diagonal(ubc, 0.0)
        assert np.all(lbc <= F + ftol) and np.all(F <= ubc + ftol), lam
    # the multi-pass refinement on a pivot list (every other pivot, reversed),
    # and the cascade: one more pass continuing from the all-pivot pass above
    piv = np.arange(X.shape[1])[::-2].copy()
    for passes in (2, 3, "continue"):
        if passes == "continue":
            eng.bound_pivots(lam)
            lb2, ub2 = eng.bound_pivot_list_continue(lam, piv, piv, X.shape[1])
        else:
            lb2, ub2 = eng.bound_pivot_list(lam, piv, passes=passes)
        assert np.all(lb2 <= o[piv] + tol[piv]), (lam, passes, np.max(lb2 - o[piv]))
        assert np.all(o[piv] <= ub2 + tol[piv]), (lam, passes, np.max(o[piv] - ub2))
        if not cols:
            continue
        lbc, ubc = eng.bound_columns(piv.size)
        Fp = F[piv]
        for k, p in enumerate(piv):
            lbc[k, p] = ubc[k, p] = 0.0
        assert np.all(lbc <= Fp + ftol[piv]) and np.all(Fp <= ubc + ftol[piv]), (lam, passes)
    return lb, ub, o


@pytest.mark.parametrize("lam_kind", ["zero", "small", "mid", "large"])
def test_bounds_contain_every_pivot_objective(lam_kind):
    """l1b_bound_pivots: lb <= z_p <= ub for every pivot (C1, grid and ragged data)."""
    g = load_golden("c1.npz")
    cases = [g["X"], g["Xq"]]
    d, _ = l1b.gen_line_data(40, 700, seed=11, noise_scale=1.0)
    cases.append(d.values)
    rng = np.random.default_rng(5)
    Z = np.round(rng.uniform(-10, 10, size=(300, 20)) * 4) / 4
    Z[rng.random(Z.shape) < 0.3] = 0.0
    cases.append(Z)
    for X in cases:
        T = float(np.abs(X).sum(axis=0).max())
        lam = {"zero": 0.0, "small": 1.0, "mid": 0.2 * T, "large": 0.9 * T}[lam_kind]
        _bounds_hold(X, lam)


def test_pruned_fit_equals_full_fit():
    """The pruned fit_line path returns exactly what fitting every pivot returns."""
    for seed, (m, n) in enumerate([(60, 900), (200, 300), (30, 5000)]):
        d, _ = l1b.gen_line_data(m, n, seed=seed, noise_scale=1.0)
        X = d.values
        T = float(np.abs(X).sum(axis=0).max())
        lams = [0.0, 1.0, 0.1 * T, 0.5 * T, 2.0 * T, math.inf]
        eng = DeviceFit(X)
        full = eng.shard_winners(lams, prune=False)
        pruned = eng.shard_winners(lams, prune=True)  # forced: these sizes are below the auto threshold
        for a, b in zip(full, pruned):
            assert a.pivot == b.pivot and a.v.tobytes() == b.v.tobytes()
            assert (a.error, a.penalty_norm, a.objective) == (b.error, b.penalty_norm, b.objective)


def test_staged_upload_is_exact():
    """engine._upload (l1b_upload: pooled streaming-store staging, two pinned
    chunks, the first a quarter chunk): byte-identical device copies for sizes
    around the chunk boundaries, several uploads queued back to back."""
    from paper_2402_16712_b200 import engine
    rng = np.random.default_rng(3)
    ch = engine._STAGE_DOUBLES
    dev = torch.device("cuda", torch.cuda.current_device())
    outs = []
    for rows, cols in [(1, 7), (ch // 4 // 8, 8), (ch // 4 // 8 + 1, 8), (ch // 1000, 1000), (3 * ch // 700 + 5, 700),
                       (1234, 2345)]:
        X = rng.standard_normal((rows, cols))
        X[0, 0] = -0.0
        outs.append((X, engine._upload(X, dev)))  # no synchronisation between uploads
    torch.cuda.synchronize()
    for X, d in outs:
        assert d.cpu().numpy().tobytes() == X.tobytes(), X.shape


def test_sweep_driver_matches_python_cascade(monkeypatch):
    """l1b_fit_lines (the sweep cascade in C++) returns exactly what the same
    cascade driven from Python returns (engine._sweep_winners): unsorted and
    repeated penalties, and a global-threshold hook that leaves some penalties
    to "another shard" (None)."""
    d, _ = l1b.gen_line_data(300, 1500, seed=12, noise_scale=1.0)
    X = d.values
    T = float(np.abs(X).sum(axis=0).max())
    lams = [5.0, 0.0, 1.0, 5.0, 0.3 * T, 0.05 * T]
    eng = DeviceFit(X)

    def run(py, exchange=None):
        monkeypatch.setenv("L1B200_PY_SWEEP", "1" if py else "0")
        return eng.shard_winners(lams, prune=True, ub_exchange=exchange)

    for exchange in (None, lambda tops: np.where(np.arange(tops.size) % 2 == 0, tops * (1 - 1e-3), tops)):
        a, b = run(False, exchange), run(True, exchange)
        assert len(a) == len(b) == len(lams)
        for x, y in zip(a, b):
            assert (x is None) == (y is None)
            if x is not None:
                assert x.pivot == y.pivot and x.v.tobytes() == y.v.tobytes()
                assert (x.error, x.penalty_norm, x.objective, x.lam) == (y.error, y.penalty_norm, y.objective, y.lam)
        if exchange is None:
            full = eng.shard_winners(lams, prune=False)
            assert [w.pivot for w in a] == [w.pivot for w in full]
            assert all(w.v.tobytes() == f.v.tobytes() and w.objective == f.objective for w, f in zip(a, full))


def test_raster_bands_leave_bounds_unchanged(monkeypatch):
    """k_bound's raster bands (CTAs pivot-group-major inside bands of target
    groups, used when the target tiles outgrow L2) only reorder the CTAs: the
    per-pivot bounds are integer sums, so every band width -- a ragged last band
    included -- gives the same bits, single- and multi-penalty, and the pruned
    fit is still the full fit."""
    d, _ = l1b.gen_line_data(330, 1500, seed=8, noise_scale=1.0)  # 6 target groups of 64
    X = d.values
    eng = DeviceFit(X)
    lams = [0.0, 1.0, 300.0]
    monkeypatch.delenv("L1B200_BAND", raising=False)
    ref = eng.bound_pivot_sums(1.0)
    refm = eng.bound_pivots_multi(lams)
    full = eng.shard_winners([1.0], prune=False)[0]
    for band in ("1", "4", "5"):
        monkeypatch.setenv("L1B200_BAND", band)
        got = eng.bound_pivot_sums(1.0)
        assert got[0].tobytes() == ref[0].tobytes() and got[1].tobytes() == ref[1].tobytes(), band
        gotm = eng.bound_pivots_multi(lams)
        assert all(np.array_equal(a, b) for a, b in zip(gotm[:2], refm[:2])), band
        w = eng.shard_winners([1.0], prune=True)[0]
        assert w.pivot == full.pivot and w.v.tobytes() == full.v.tobytes() and w.objective == full.objective


def test_pruned_fit_equals_full_fit_tall():
    """Tall columns (n >= 2 * KB_SREP_ROWS = 8192) start the bound pass from several
    averaged row samples (k_bound<..., TALL>); single- and multi-penalty pruned
    fits, also on deflated data, still return exactly the full fit.  The
    all-finite sweep takes the one-pass multi-penalty path (k_bound<..., MULTI,
    TALL> + the batched entry cascade); a sweep with +inf takes the per-penalty loop."""
    d, _ = l1b.gen_line_data(24, 40000, seed=5, noise_scale=1.0)
    X = d.values
    T = float(np.abs(X).sum(axis=0).max())
    eng = DeviceFit(X)
    for comp in range(2):
        for lams in ([1.0], [0.05 * T], [0.0, 1.0, 0.1 * T, 0.5 * T], [0.0, 1.0, 0.1 * T, 0.5 * T, math.inf]):
            full = eng.shard_winners(lams, prune=False)
            pruned = eng.shard_winners(lams, prune=True)
            for a, b in zip(full, pruned):
                assert a.pivot == b.pivot and a.v.tobytes() == b.v.tobytes()
                assert (a.error, a.penalty_norm, a.objective) == (b.error, b.penalty_norm, b.objective)
        eng.deflate(full[0].v)


@pytest.mark.parametrize("m,n", [(300, 2000), (40, 70000)])
def test_seeded_exact_fit_equals_batched_fit(m, n):
    """l1b_fit_pivot_list_seeded (warp-per-problem solver started on the bound
    ranges) returns bit-identical V (err / obj to 1e-12) to the batched exact path, for
    seeds from one-pass and three-pass bounds, and for stale seeds (ranges of
    other problems: the solver must widen them itself)."""
    d, _ = l1b.gen_line_data(m, n, seed=3, noise_scale=1.0)
    X = d.values
    T = float(np.abs(X).sum(axis=0).max())
    eng = DeviceFit(X)
    for lam in (0.0, 1.0, 0.3 * T):
        piv = np.arange(0, m, 7)
        V0, e0, _, o0 = eng.fit_pivot_list([lam], piv)
        V0, e0, o0 = V0.cpu().numpy(), e0.cpu().numpy(), o0.cpu().numpy()
        for passes in (1, 3):
            eng.bound_pivot_list(lam, piv, passes=passes)
            for seed in (np.arange(piv.size), np.arange(piv.size)[::-1].copy()):
                V1, e1, _, o1 = eng.fit_pivot_list_seeded(lam, piv, seed, piv.size)
                assert V1.cpu().numpy().tobytes() == V0.tobytes(), (lam, passes)
                # device error sums differ in summation order between the paths (the winner is re-scored
                # in NumPy order either way)
                np.testing.assert_allclose(e1.cpu().numpy(), e0, rtol=1e-12)
                np.testing.assert_allclose(o1.cpu().numpy(), o0, rtol=1e-12)


def test_sharded_pruning_with_global_threshold():
    """Two interleaved pivot shards pruned against the global best upper bound
    (what distributed.ub_exchange provides) combine to the unsharded winner;
    a shard may keep no pivot at all."""
    d, _ = l1b.gen_line_data(120, 1500, seed=8, noise_scale=1.0)
    X = d.values
    T = float(np.abs(X).sum(axis=0).max())
    m = X.shape[1]
    eng = DeviceFit(X)
    for lam in (1.0, 0.2 * T):
        want = eng.shard_winners([lam], prune=False)[0]
        shards = [shard(m, r, 3) for r in range(3)]
        tops = [float(np.min(eng.bound_pivots(lam, *sh)[1])) for sh in shards]
        wins = [eng.shard_winners([lam], *sh, prune=True, ub_exchange=lambda t: min(tops))[0] for sh in shards]
        wins = [w for w in wins if w is not None]
        best = min(wins, key=lambda w: (w.objective, w.pivot))
        assert best.pivot == want.pivot and best.v.tobytes() == want.v.tobytes()
        assert best.objective == want.objective


def test_multi_penalty_bound_pass():
    """l1b_bound_pivots_multi: one pass bounds every penalty of a sweep
    (lb <= z <= ub per penalty and pivot), and the pruned sweep equals the
    unpruned one."""
    d, _ = l1b.gen_line_data(70, 1200, seed=4, noise_scale=1.0)
    X = d.values
    T = float(np.abs(X).sum(axis=0).max())
    lams = np.array([0.0, 0.5, 3.0, 0.05 * T, 0.3 * T, 0.9 * T, 1.5 * T])
    eng = DeviceFit(X)
    lb, ub = eng.bound_pivots_multi(lams)
    _, _, _, O = eng.fit_pivots(lams, want_v=False)
    O = O.cpu().numpy()
    tol = 1e-12 * np.abs(O) + OBJ_ATOL * float(np.abs(X).sum())
    assert np.all(lb <= O + tol) and np.all(O <= ub + tol)
    full = eng.shard_winners(lams, prune=False)
    pruned = eng.shard_winners(lams[::-1], prune=True)[::-1]  # any order, repeated penalties allowed
    for a, b in zip(full, pruned):
        assert a.pivot == b.pivot and a.v.tobytes() == b.v.tobytes() and a.objective == b.objective


# ------------------------------------------- Algorithm 2 (path.py, "next") --

THIRD = 1.0 / 3.0


def test_pivot_breakpoints_toy_known_answers():
    """pkg/tests/test_path.py:33-70 (toy entry maps, death weights, breakpoint sets)."""
    from paper_2402_16712_b200 import pivot_breakpoints
    expected = {
        0: {1: ((0.0, -0.5), (3.0, 0.0)), 2: ((0.0, 0.4), (1.0, 0.0)),
            3: ((0.0, -1.0), (1.0, -0.2), (11.0, 0.0))},
        1: {0: ((0.0, -0.75), (4.0, 0.0)), 2: ((0.0, 0.5), (6.0, 0.0)), 3: ((0.0, -0.25), (4.0, 0.0))},
        2: {0: ((0.0, -2.0 * THIRD), (2.0, 0.0)), 1: ((0.0, 0.0),), 3: ((0.0, -0.5), (2.0, 0.0))},
        3: {0: ((0.0, -2.0 * THIRD), (11.0, 0.0)), 1: ((0.0, THIRD), (5.0, 0.0)), 2: ((0.0, -0.5), (3.0, 0.0))},
    }
    for pivot, entries in expected.items():
        pb = pivot_breakpoints(TOY, pivot)
        assert pb.pivot == pivot and pb.entries == entries
    assert pivot_breakpoints(TOY, 0).lambda_max == {1: 3.0, 2: 1.0, 3: 11.0}
    sets = [pivot_breakpoints(TOY, p).breakpoint_set() for p in range(4)]
    assert sets == [{1.0, 3.0, 11.0}, {4.0, 6.0}, {0.0, 2.0}, {3.0, 5.0, 11.0}]
    pb = pivot_breakpoints(TOY, 0)
    assert [pb.column_value(3, x) for x in (0.0, 0.999, 1.0, 11.0, 1e6)] == [-1.0, -1.0, -0.2, 0.0, 0.0]
    with pytest.raises(ValueError):
        pb.column_value(3, -0.5)
    with pytest.raises(IndexError):
        pivot_breakpoints(TOY, 4)


def test_major_breakpoints_match_reference_fixtures():
    """Every pivot's entry map, death weights and the merged grid equal the
    reference's (tests/golden/breakpoints.npz, from l1line.major_breakpoints),
    bit for bit: toy, ragged random instances with zeros / -0.0 / ties / zero
    columns, a 300x12 line and a 3000x6 grid-quantised tall case."""
    from paper_2402_16712_b200 import major_breakpoints
    from paper_2402_16712_b200.path import EmptyPivotError, pivot_breakpoints
    g = load_golden("breakpoints.npz")
    for name in g["names"]:
        X = g[f"{name}_X"]
        grid, sols = major_breakpoints(X)
        assert grid.tobytes() == g[f"{name}_grid"].tobytes(), name
        assert sols.degenerate == tuple(int(p) for p in g[f"{name}_degenerate"]), name
        for p in range(X.shape[1]):
            if p in sols.degenerate:
                with pytest.raises(EmptyPivotError):
                    pivot_breakpoints(X, p)
                continue
            pb = sols.pivots[p]
            rows = np.asarray([(t, bp, v) for t, e in pb.entries.items() for bp, v in e], dtype=np.float64)
            lmax = np.asarray([(t, pb.lambda_max[t]) for t in pb.entries], dtype=np.float64)
            assert rows.tobytes() == g[f"{name}_p{p}_entries"].tobytes(), (name, p)
            assert lmax.tobytes() == g[f"{name}_p{p}_lmax"].tobytes(), (name, p)
        assert sols.solution_at(int(np.argmax([p in sols.pivots for p in range(X.shape[1])])), 0.0).shape == (X.shape[1],)


# ------------------------------- optimality certificates (oracle.py, "next") --

def test_certificates_toy_and_refutations():
    """oracle.py:141-174 behaviour (pkg/tests/test_oracle.py:55-110): every
    solved toy column is certified; wrong values are refuted."""
    import types

    from paper_2402_16712_b200 import OptimalityRefuted, certify_line, check_line
    for lam in (0.0, 0.5, 2.0, 3.0, 7.0, 11.0, 15.0):
        for pivot in range(4):
            line = l1b.fit_for_pivot(TOY, pivot, lam)
            cert = check_line(TOY, line)
            assert cert.ok and np.isinf(cert.slack[pivot])
    base = l1b.fit_for_pivot(TOY, 0, 0.0)
    for j, val, lam in ((3, -1.5, 0.0), (3, -0.987, 0.0)):
        v = base.v.copy()
        v[j] = val
        bad = types.SimpleNamespace(v=v, preserved=0, lam=lam)
        assert certify_line(TOY, bad).refuted == (j,)
        with pytest.raises(OptimalityRefuted):
            check_line(TOY, bad)
    # column (0, 2): 0.4 until it dies at lam 1; at lam 5 only 0.0 is optimal
    v = l1b.fit_for_pivot(TOY, 0, 5.0).v.copy()
    assert v[2] == 0.0 and certify_line(TOY, types.SimpleNamespace(v=v, preserved=0, lam=5.0)).ok
    v[2] = 0.4
    assert 2 in certify_line(TOY, types.SimpleNamespace(v=v, preserved=0, lam=5.0)).refuted


def test_certificates_random_and_at_scale():
    """Random instances (test_oracle.py:94-110) and a 3000x400 winner: every column certified."""
    from paper_2402_16712_b200 import check_line
    from conftest import random_instance
    rng = np.random.default_rng(8)
    for _ in range(25):
        X = random_instance(rng, zeros=True)
        lam = float(rng.uniform(0.0, 0.7 * np.abs(X).sum()))
        check_line(X, l1b.fit_line(X, lam))
    d, _ = l1b.gen_line_data(400, 3000, seed=2, noise_scale=1.0)
    for lam in (1.0, 500.0):
        cert = check_line(d, l1b.fit_line(d, lam))
        assert cert.ok and np.isfinite(cert.slack).sum() == 399


def test_residual_exact_batch_equals_single():
    """l1b_residual_exact_batch == l1b_residual_exact (bit for bit) per candidate."""
    rng = np.random.default_rng(12)
    for n, m in ((37, 11), (2000, 300)):
        X = rng.standard_normal((n, m))
        eng = DeviceFit(X, max_pivots=1)
        piv = rng.integers(0, m, size=9)
        V = torch.from_numpy(rng.standard_normal((9, m))).to(eng.device)
        got = eng.residual_exact_batch(V, piv)
        for k in range(9):
            assert got[k] == eng.residual_exact(V[k], int(piv[k])), (n, m, k)


def test_c_driver_fit_line_equals_unpruned():
    """l1b_fit_line (the pruned cascade in C++) returns exactly the unpruned winner,
    forced pruning and auto, and agrees with the Python sweep path."""
    for seed, (m, n) in enumerate([(60, 900), (40, 5000)]):
        d, _ = l1b.gen_line_data(m, n, seed=seed + 20, noise_scale=1.0)
        X = d.values
        T = float(np.abs(X).sum(axis=0).max())
        eng = DeviceFit(X)
        for lam in (0.0, 1.0, 0.2 * T, 2.0 * T):
            want = eng.fit_line_device(lam, prune=False)
            for prune in (True, None):
                got = eng.fit_line_device(lam, prune=prune)
                assert got.pivot == want.pivot and got.v.tobytes() == want.v.tobytes()
                assert (got.error, got.penalty_norm, got.objective) == (want.error, want.penalty_norm, want.objective)
            sweep = eng.shard_winners([lam, lam + 1.0], prune=True)[0]
            assert sweep.pivot == want.pivot and sweep.v.tobytes() == want.v.tobytes()
            assert sweep.objective == want.objective


def test_integration_stub_runs():
    """The ctypes binding INTEGRATION.md proposes for l1line/gpu.py works as written
    (library path and FittedLine import adapted) and matches fit_line."""
    import os
    import re
    from conftest import ROOT
    from paper_2402_16712_b200 import _lib as lib_mod
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"```python\n(# l1line/gpu.py.*?)```", text, re.S).group(1)
    code = code.replace("from .core import FittedLine", "from paper_2402_16712_b200.core import FittedLine")
    code = code.replace('ctypes.CDLL("libl1b200.so")', f"ctypes.CDLL({lib_mod.LIB_PATH!r})")
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    d, _ = l1b.gen_line_data(80, 3000, seed=6, noise_scale=1.0)
    for lam in (1.0, 50.0):
        got = ns["fit_line"](d, lam)
        want = l1b.fit_line(d, lam)
        assert got.preserved == want.preserved and got.v.tobytes() == want.v.tobytes()
        assert got.objective == want.objective and got.error == want.error


def test_pruned_paths_random_stress():
    """A short run of tools/stress_prune.py's check (pruned == unpruned, bit for
    bit) over Gaussian, Cauchy, tied, sparse and badly scaled data, including
    sweeps whose survivors exceed the workspace's pivot capacity."""
    rng = np.random.default_rng(99)
    for t in range(12):
        m, n = int(rng.integers(34, 90)), int(rng.integers(50, 1500))
        X = [rng.standard_normal((n, m)), rng.standard_cauchy((n, m)), np.round(rng.uniform(-5, 5, (n, m))),
             rng.standard_normal((n, m)) * np.exp(rng.uniform(-8, 8, (1, m)))][t % 4]
        T = float(np.abs(X).sum(axis=0).max())
        lams = [0.0, 1.0, 0.1 * T, 0.8 * T]
        eng = DeviceFit(X)
        full = eng.shard_winners(lams, prune=False)
        for lam, want in zip(lams, full):
            got = eng.fit_line_device(lam, prune=True)
            assert got.pivot == want.pivot and got.v.tobytes() == want.v.tobytes() and got.objective == want.objective
        for a, b in zip(eng.shard_winners(lams, prune=True), full):
            assert a.pivot == b.pivot and a.v.tobytes() == b.v.tobytes() and a.objective == b.objective


def test_block_solver_heavy_ties_and_signed_zero():
    """Tall data (block-per-problem exact solver): a crossing key shared by
    thousands of rows (grid data) and a column whose weighted median is a
    zero ratio (its sign from the crossing row) -- the case a random stress
    run found; pruned == unpruned bit for bit."""
    rng = np.random.default_rng(31)
    n, m = 9000, 36
    X = np.round(rng.standard_normal((n, m)) * 4) / 4
    X[rng.random(n) < 0.7, 5] = 0.0
    X[rng.random(n) < 0.2, 5] = -0.0
    X[:, 9] = 0.0
    eng = DeviceFit(X)
    for lam in (0.0, 1.0, 50.0):
        want = eng.fit_line_device(lam, prune=False)
        got = eng.fit_line_device(lam, prune=True)
        assert got.pivot == want.pivot and got.v.tobytes() == want.v.tobytes() and got.objective == want.objective
        for p in (0, 5):  # every column of two pivots through the seeded block solver
            lb, ub = eng.bound_pivot_list(lam, [p], passes=3)
            V, _, _, _ = eng.fit_pivot_list_seeded(lam, [p], [0], 1)
            V0, _, _, _ = eng.fit_pivot_list([lam], [p])
            assert V[0, 0].cpu().numpy().tobytes() == V0[0, 0].cpu().numpy().tobytes()


def test_solution_path_matches_reference():
    """solution_path = device breakpoints (k_breakpoints) + native merge: the
    reference's paths (tests/golden/paths.npz) bit for bit."""
    from paper_2402_16712_b200 import solution_path
    bp = load_golden("breakpoints.npz")
    g = load_golden("paths.npz")
    for name in bp["names"]:
        path = solution_path(bp[f"{name}_X"])
        segs = path.segments
        assert np.asarray([s.line.preserved for s in segs]).tolist() == g[f"{name}_piv"].tolist(), name
        assert np.asarray([s.lambda_lo for s in segs]).tobytes() == g[f"{name}_lo"].tobytes(), name
        assert np.asarray([s.line.v for s in segs]).tobytes() == g[f"{name}_v"].tobytes(), name
        assert np.asarray([s.line.objective for s in segs]).tobytes() == g[f"{name}_obj"].tobytes(), name


def test_pruned_path_outside_fp32_window():
    """Magnitudes beyond the FP32 steering window (|x| ~ 2^80, and a column
    near 2^-70): the bounds prune nothing and every problem goes to the exact
    straggler solver -- the pruned API path still returns the exact winner."""
    rng = np.random.default_rng(41)
    X = rng.standard_normal((600, 40)) * 2.0 ** 80
    X[:, 3] *= 2.0 ** -150
    eng = DeviceFit(X)
    for lam in (0.0, 1e24):
        want = eng.fit_line_device(lam, prune=False)
        got = eng.fit_line_device(lam, prune=True)
        assert got.pivot == want.pivot and got.v.tobytes() == want.v.tobytes() and got.objective == want.objective


def test_brute_force_and_sweep_validate():
    """oracle.py's brute force on the device: toy KAT (test_oracle.py:23-36),
    brute-force objectives == fit_line's exactly on random data, and the
    reference's sweep_validate (test_acceptance.py:110-120) on a device path."""
    from paper_2402_16712_b200 import brute_force_column, brute_force_line, solution_path, sweep_validate
    t, f = brute_force_column(TOY, 0, 1, 0.0)
    want = oracle.fit_for_pivot(TOY, 0, 0.0)
    assert t == want.v[1]
    rng = np.random.default_rng(17)
    for _ in range(6):
        X = rng.uniform(-10, 10, size=(int(rng.integers(5, 40)), int(rng.integers(3, 8))))
        lam = float(rng.uniform(0, np.abs(X).sum()))
        b = brute_force_line(X, lam)
        g = l1b.fit_line(X, lam)
        assert b.objective == g.objective or abs(b.objective - g.objective) <= 1e-12 * max(1.0, abs(g.objective))
    X = rng.uniform(-10, 10, size=(30, 5))
    rep = sweep_validate(X, solution_path(X), grid_size=40)
    assert rep.ok, rep.failures


def test_subspace_rejects_zero_direction_like_reference():
    """subspace.py:71-75 deflates after every component (the last one too) and
    deflate (subspace.py:32-33) raises on v = 0: a degenerate winning line at a
    huge penalty makes the reference's fit_subspace raise, even for k = 1."""
    X = np.array([[0.0, 2.0, 1.0], [0.0, -1.0, 3.0], [0.0, 4.0, -2.0]])
    with pytest.raises(ValueError, match="zero vector"):
        l1b.fit_subspace(X, 100.0, 1)
    with pytest.raises(ValueError, match="zero vector"):
        l1b.deflate(X, np.zeros(3))


@pytest.mark.parametrize("n,zeros", [(40000, False), (70001, True)])
def test_pivot_runs_tall_pivot(n, zeros):
    """Pivots with more than 16384 nonzero rows (chunk sorts + global merges,
    l1b_pivot_breakpoints' tall path) give the sorted tableau runs of
    path.py:76-102 bit for bit: ratios.py:40-67's column (the oracle's
    build_column, itself pinned to the reference) and path.py:86-89's run
    arithmetic (center = (T - P) - P_prev, start = +-center - w, right = start + 2 w)."""
    rng = np.random.default_rng(n)
    d, _ = l1b.gen_line_data(5, n, seed=7, noise_scale=1.0)
    X = np.array(d.values)
    X = np.round(X * 64.0) / 64.0  # heavy exact ties: the row tie-break decides the order
    if zeros:
        X[rng.random(n) < 0.3, 2] = 0.0
        X[rng.random(n) < 0.1, 0] = -0.0
    eng = DeviceFit(X)
    for p in (0, 2):
        R, S, T = eng.pivot_runs(p)
        cols = [j for j in range(X.shape[1]) if j != p]
        for c, j in enumerate(cols):
            r, w, rows, pref = oracle.build_column(X, p, j)
            prev = np.concatenate(([0.0], pref[:-1]))
            center = (pref[-1] - pref) - prev
            start = np.where(r >= 0.0, center, -center) - w
            right = start + 2.0 * w
            assert R[c].tobytes() == r.tobytes(), (p, j)
            assert S[c].tobytes() == start.tobytes() and T[c].tobytes() == right.tobytes(), (p, j)


# ------------------------------------------- the sorted-ratio API (ratios.py) --

def test_tableau_and_certificates_match_reference():
    """pivot_tableau / build_column (ratios.py:40-67, 109-135) from the device
    sort equal the reference's arrays bit for bit (ties, exact zeros, -0.0,
    zero pivot columns -> EmptyPivotError), solve_column / window_bounds agree,
    and dual_certificate (oracle.py:141-174) returns the reference's
    multipliers -- or refutes exactly where it does (tests/golden/tableau.npz)."""
    from paper_2402_16712_b200.certify import OptimalityRefuted
    g = load_golden("tableau.npz")
    for name in g["names"]:
        X = g[f"{name}_X"]
        d = l1b.DataMatrix(X)
        n, m = X.shape
        lams = g[f"{name}_lams"]
        for p in range(m):
            if f"{name}_p{p}_empty" in g.files:
                with pytest.raises(l1b.EmptyPivotError):
                    l1b.pivot_tableau(d, p)
                with pytest.raises(l1b.EmptyPivotError):
                    l1b.build_column(d, p, (p + 1) % m)
                continue
            tab = l1b.pivot_tableau(d, p)
            for key in ("ratios", "weights", "source_rows", "prefix", "prefix_prev", "totals", "targets"):
                want = g[f"{name}_p{p}_{key}"]
                got = getattr(tab, key)
                assert got.shape == want.shape and got.tobytes() == want.astype(got.dtype).tobytes(), (name, p, key)
        cert = g[f"{name}_cert"]
        for row in cert:
            p, j, li, case, val, ok, gamma = int(row[0]), int(row[1]), int(row[2]), int(row[3]), row[4], row[5], row[6]
            col = l1b.build_column(d, p, j)
            lam = float(lams[li])
            if case == 0:
                assert l1b.solve_column(col, lam) == val
                for k in (0, len(col) - 1):
                    lo, hi = l1b.window_bounds(col, k)
                    assert hi == col.total_weight - 2.0 * (float(col.prefix_weights[k - 1]) if k else 0.0)
                    assert lo == col.total_weight - 2.0 * float(col.prefix_weights[k])
            if ok:
                c = l1b.dual_certificate(col, float(val), lam)
                assert c.gamma == gamma and c.pi.tobytes() == row[7:7 + len(col)].tobytes(), (name, p, j, li, case)
            else:
                with pytest.raises(OptimalityRefuted):
                    l1b.dual_certificate(col, float(val), lam)


def test_build_column_errors_like_reference():
    """ratios.py:31-37: IndexError for out-of-range columns, ValueError for pivot == target."""
    with pytest.raises(IndexError):
        l1b.build_column(TOY, 4, 0)
    with pytest.raises(IndexError):
        l1b.build_column(TOY, 0, -1)
    with pytest.raises(ValueError):
        l1b.build_column(TOY, 2, 2)
    with pytest.raises(IndexError):
        l1b.pivot_tableau(TOY, 9)
    col = l1b.build_column(TOY, 0, 3)  # pkg/tests/test_ratios.py:8-17
    assert col.ratios.tolist() == [-1.5, -1.0, -1.0, -0.2, 1.0 / 3.0]
    assert col.weights.tolist() == [4.0, 2.0, 3.0, 5.0, 3.0] and col.source_rows.tolist() == [0, 2, 3, 4, 1]
    assert col.prefix_weights.tolist() == [4.0, 6.0, 9.0, 14.0, 17.0] and col.total_weight == 17.0
    with pytest.raises(IndexError):
        l1b.window_bounds(col, 5)


def test_engine_cache_reuses_upload():
    """fit_for_pivot over every pivot of one DataMatrix uploads X once (the device
    replica is cached by the read-only values array) and matches fit_line's pivot."""
    from paper_2402_16712_b200 import api
    d, _ = l1b.gen_line_data(40, 300, seed=2, noise_scale=1.0)
    api._ENGINES.clear()
    lines = [l1b.fit_for_pivot(d, p, 1.0) for p in range(d.m)]
    assert len(api._ENGINES) == 1
    best = min(range(d.m), key=lambda p: (lines[p].objective, p))
    assert l1b.fit_line(d, 1.0).preserved == best and len(api._ENGINES) == 1
    w = np.array(d.values)  # a writable copy is never cached
    l1b.fit_for_pivot(w, 0, 1.0)
    assert len(api._ENGINES) == 1


def test_bounds_and_fits_deterministic_across_runs():
    """compute-sanitizer is closed on this GPU pool (profiles/r02/compute_sanitizer_refused.txt),
    so races are caught by determinism: k_bound's bounds are exact integer sums and
    every exact result a fixed-order reduction, so a TMA-ring or histogram race
    would change bytes between identical runs (tools/race_stress.py runs 40 reps)."""
    import hashlib
    d, _ = l1b.gen_line_data(300, 3000, seed=9, noise_scale=1.0)
    X = np.array(d.values)
    eng = DeviceFit(X)
    T = float(np.abs(X).sum(axis=0).max())

    def run():
        h = hashlib.blake2b(digest_size=16)
        lb, ub = eng.bound_pivots(1.0)
        clb, cub = eng.bound_columns(eng.m)
        for a in (lb, ub, clb, cub, *eng.bound_pivots_multi([0.0, 1.0, 0.3 * T])[:2]):
            h.update(np.ascontiguousarray(a).tobytes())
        w = eng.shard_winners([1.0])[0]
        h.update(w.v.tobytes())
        return h.hexdigest()
    first = run()
    for _ in range(4):
        assert run() == first
