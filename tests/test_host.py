"""CPU-only checks: datagen bytes, host contracts, C-ABI export list, sharding."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_2402_16712_b200 as l1b
from conftest import ROOT, TOY, load_golden
from paper_2402_16712_b200 import _lib
from paper_2402_16712_b200.engine import shard


# ---------------------------------------------------------------- datagen --

def test_datagen_bytes_match_reference():
    g = load_golden("datagen.npz")
    for (m, n, seed, ns) in ((7, 11, 0, 1.0), (5, 9, 3, 0.0), (12, 30, 42, 2.5)):
        d, v = l1b.gen_line_data(m, n, seed=seed, noise_scale=ns)
        assert d.values.tobytes() == g[f"line_{m}_{n}_{seed}_X"].tobytes()
        assert v.tobytes() == g[f"line_{m}_{n}_{seed}_v"].tobytes()
    for (m, n, k, seed) in ((6, 13, 3, 1), (50, 200, 20, 0)):
        d, v = l1b.gen_outlier_data(m, n, k, seed=seed)
        assert d.values.tobytes() == g[f"outl_{m}_{n}_{k}_{seed}_X"].tobytes()
        assert v.tobytes() == g[f"outl_{m}_{n}_{k}_{seed}_v"].tobytes()


def test_datagen_c2_checksum():
    g = load_golden("datagen.npz")
    d, v = l1b.gen_line_data(2000, 2000, seed=0, noise_scale=1.0)
    X = d.values
    assert X[:2].tobytes() == g["c2_head"].tobytes()
    assert X[-2:].tobytes() == g["c2_tail"].tobytes()
    assert X[::97, ::89].tobytes() == g["c2_stride"].tobytes()
    assert v.tobytes() == g["c2_v"].tobytes()


def test_datagen_validation():
    with pytest.raises(ValueError):
        l1b.gen_line_data(1, 5, 0)
    with pytest.raises(ValueError):
        l1b.gen_line_data(3, 0, 0)
    with pytest.raises(ValueError):
        l1b.gen_outlier_data(4, 10, 2, 0)


# ------------------------------------------------------------- core types --

def test_datamatrix_contract():
    # core.py:48-68 / pkg/tests/test_core.py:15-52
    d = l1b.DataMatrix(TOY)
    assert d.n == 5 and d.m == 4 and not d.values.flags.writeable
    with pytest.raises(ValueError):
        l1b.DataMatrix(np.zeros(3))
    with pytest.raises(ValueError):
        l1b.DataMatrix(np.zeros((0, 3)))
    with pytest.raises(ValueError):
        l1b.DataMatrix(np.zeros((3, 1)))
    with pytest.raises(ValueError, match="row 1, column 2"):
        bad = np.zeros((3, 3))
        bad[1, 2] = np.nan
        l1b.DataMatrix(bad)
    with pytest.raises(ValueError):
        l1b.DataMatrix(TOY, column_names=("a", "b"))
    assert l1b.DataMatrix(TOY, column_names=list("abcd")).column_names == tuple("abcd")


def test_fitted_line_invariants():
    # core.py:113-124 / pkg/tests/test_core.py:77-109
    v = np.array([1.0, -0.5, 0.0])
    line = l1b.FittedLine(v=v, preserved=0, lam=2.0, error=3.0, penalty_norm=1.5, objective=6.0)
    assert not line.v.flags.writeable and line.objective_at(0.0) == 3.0
    with pytest.raises(ValueError):
        l1b.FittedLine(v=v, preserved=1, lam=2.0, error=3.0, penalty_norm=1.5, objective=6.0)
    with pytest.raises(ValueError):
        l1b.FittedLine(v=v, preserved=0, lam=2.0, error=3.0, penalty_norm=1.5, objective=6.5)
    with pytest.raises(ValueError):
        l1b.FittedLine(v=v, preserved=0, lam=-1.0, error=3.0, penalty_norm=1.5, objective=1.5)
    l1b.FittedLine(v=np.zeros(3), preserved=2, lam=1.0, error=3.0, penalty_norm=0.0, objective=3.0)


def test_lambda_and_threads_validation():
    from paper_2402_16712_b200.api import _check_lam, resolve_threads
    assert _check_lam(math.inf) == math.inf
    for bad in (-1.0, math.nan, -1e-300):
        with pytest.raises(ValueError):
            _check_lam(bad)
    assert resolve_threads(3) == 3
    with pytest.raises(ValueError):
        resolve_threads(0)


def test_lambda_rejected_before_any_device_work():
    for fn in (lambda: l1b.fit_line(TOY, -1.0), lambda: l1b.fit_lines(TOY, [0.0, float("nan")]),
               lambda: l1b.fit_for_pivot(TOY, 0, -0.5)):
        with pytest.raises(ValueError):
            fn()
    with pytest.raises(IndexError):
        l1b.fit_for_pivot(TOY, 4, 1.0)
    with pytest.raises(ValueError):
        l1b.fit_subspace(TOY, 1.0, 4)
    with pytest.raises(ValueError):
        l1b.fit_subspace(TOY, math.inf, 2)


# -------------------------------------------------------------- sharding --

def test_shard_partitions_pivots():
    for m in (2, 3, 50, 2000, 10_001):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                b, s, k = shard(m, r, world)
                seen += [b + i * s for i in range(k)]
            assert sorted(seen) == list(range(m))
    with pytest.raises(ValueError):
        shard(10, 3, 3)


# -------------------------------------------------------------------- ABI --

def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "l1b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(l1b_\w+)\(", txt, re.M)))


def test_abi_library_exports_every_header_symbol():
    syms = _header_symbols()
    assert len(syms) >= 9
    assert sorted(_lib.ABI_SYMBOLS) == syms
    lib = _lib.load()  # loads without a GPU
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.l1b_version() == 1
    assert lib.l1b_status_string(0) == b"ok"
    assert lib.l1b_status_string(-1) == b"invalid argument"


def test_host_copy_is_memcpy():
    """l1b_host_copy (the upload's staging copy, hostcopy.inc): the same bytes as
    memcpy for any alignment and size, through the thread pool and without it."""
    lib = _lib.load()
    rng = np.random.default_rng(5)
    src = rng.integers(0, 256, (5 << 20) + 77, dtype=np.uint8)
    for size, so, do, threads in [(0, 0, 0, 8), (1, 3, 5, 8), (31, 1, 0, 1), (4096, 0, 7, 8),
                                  ((1 << 20) + 7, 5, 3, 8), ((5 << 20) + 60, 17, 11, 8), ((3 << 20) + 1, 0, 0, 3),
                                  ((2 << 20) + 9, 2, 1, 64)]:
        dst = np.zeros(size + do + 64, dtype=np.uint8)
        assert lib.l1b_host_copy(dst.ctypes.data + do, src.ctypes.data + so, size, threads) == _lib.L1B_OK
        assert np.array_equal(dst[do:do + size], src[so:so + size]), (size, so, do, threads)
        assert not dst[:do].any() and not dst[do + size:].any()
    assert lib.l1b_host_copy(None, None, 8, 4) == _lib.L1B_EINVAL


def test_abi_workspace_and_argument_checks():
    lib = _lib.load()
    assert lib.l1b_workspace_bytes(2000, 2000, 1, 2000) > 2000 * 2000 * 32
    assert lib.l1b_workspace_bytes(0, 5, 1, 1) == 0
    assert lib.l1b_workspace_bytes(5, 1, 1, 1) == 0
    # invalid shapes are rejected before any CUDA call
    assert lib.l1b_prepare(None, 5, 4, None, 0, None) == _lib.L1B_EINVAL
    lam = (ctypes.c_double * 1)(-1.0)
    assert lib.l1b_fit_pivots(1, 5, 4, lam, 1, 0, 1, 4, None, 1, 1, 1, 1, 1 << 30, None) == _lib.L1B_EINVAL
    lam[0] = 1.0
    assert lib.l1b_fit_pivots(1, 5, 4, lam, 1, 3, 1, 2, None, 1, 1, 1, 1, 1 << 30, None) == _lib.L1B_EINVAL
    # l1b_fit_lines: >= 2 distinct finite nonnegative penalties, a valid shard
    hook = _lib.UB_EXCHANGE_VEC_FN(0)
    out_i = (ctypes.c_int64 * 3)()
    out_d = [(ctypes.c_double * 3)() for _ in range(3)]

    def fit_lines(vals, p_begin=0, npiv=4):
        lams = (ctypes.c_double * len(vals))(*vals)
        return lib.l1b_fit_lines(1, 5, 4, lams, len(vals), p_begin, 1, npiv, hook, None, 1, None, 0, out_i, 1,
                                 out_d[0], out_d[1], out_d[2], None, 1, 1 << 30, None)
    assert fit_lines([1.0, 1.0]) == _lib.L1B_EINVAL             # one distinct penalty: l1b_fit_line
    assert fit_lines([1.0, float("inf")]) == _lib.L1B_EINVAL    # non-finite
    assert fit_lines([1.0, -2.0]) == _lib.L1B_EINVAL            # negative
    assert fit_lines([1.0, 2.0], p_begin=3, npiv=2) == _lib.L1B_EINVAL  # shard past the last pivot


def test_abi_sass_is_sm100a():
    import subprocess
    so = _lib.LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_breakpoint_grid_dedup_matches_reference_rule():
    """path.major_breakpoints' vectorised dedup == path.py:146-152's sequential rule."""
    from paper_2402_16712_b200.path import DEDUP_TOL, _dedup
    rng = np.random.default_rng(0)
    for t in range(100):
        v = np.concatenate([rng.uniform(0, 1e-7, 40), np.round(rng.uniform(0, 5, 80), 2),
                            rng.uniform(0, 1e-8, 20) + 3.0, np.zeros(5), rng.uniform(0, 1e-9, 10) + 1.0])
        vals = sorted([0.0] + v.tolist())
        ref = [vals[0]]
        for x in vals[1:]:
            if x - ref[-1] > DEDUP_TOL:
                ref.append(x)
        assert np.asarray(ref).tobytes() == _dedup(np.concatenate([[0.0], v])).tobytes(), t


def test_discordance_and_l0_fraction():
    """subspace.py:79-110 mirrors (pkg/tests/test_subspace.py's properties)."""
    v = np.array([3.0, 0.0, -4.0])
    assert l1b.discordance(v, -2.5 * v) <= 1e-15
    assert l1b.discordance([1.0, 0.0], [0.0, 2.0]) == 1.0
    assert l1b.l0_fraction([0.0, 1e-12, 0.5, -2.0]) == 0.5
    with pytest.raises(ValueError):
        l1b.discordance([0.0, 0.0], [1.0, 0.0])
    with pytest.raises(ValueError):
        l1b.l0_fraction(v, tol=-1.0)


def test_pivot_events_equal_breakpoint_maps():
    """path._pivot_events (solution_path's array route) yields exactly the entries
    of path._maps (pivot_breakpoints' tuples, path.py:76-102) in the same order:
    live runs clamped at 0, the death entry last among equal weights, dead runs dropped."""
    from paper_2402_16712_b200 import path as P

    rng = np.random.default_rng(11)
    for trial in range(30):
        m, k = int(rng.integers(2, 7)), int(rng.integers(1, 12))
        p = int(rng.integers(m))
        rs = np.round(rng.normal(size=(m - 1, k)), 1)
        st = np.round(rng.normal(size=(m - 1, k)) * 3, 0)           # ties and zeros in the starts
        rt = st + 2.0 * np.abs(np.round(rng.normal(size=(m - 1, k)), 0))
        rt[rng.random(rt.shape) < 0.3] = -1.0                       # dead runs

        class Eng:
            def pivot_runs(self, pivot):
                return rs, st, rt
        Eng.m = m
        tgt, w, v = P._pivot_events(Eng(), p)
        maps = P._maps(p, m, rs, st, rt)
        want = [(t, bp, val) for t, entries in maps.entries.items() for bp, val in entries]
        got = list(zip(tgt.tolist(), w.tolist(), v.tolist()))
        assert got == want, trial
