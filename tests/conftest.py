"""Shared fixtures.  Mirrors the reference's pkg/tests/conftest.py:8-33.

Tests marked ``gpu`` need a B200 (run with ``-m gpu`` on the GPU box);
everything else runs on a CPU-only machine.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# Five points in four dimensions (pkg/tests/conftest.py:8-14).
TOY = np.array([
    [4.0, -2.0, 3.0, -6.0],
    [-3.0, 4.0, 2.0, -1.0],
    [2.0, 3.0, -3.0, -2.0],
    [-3.0, 4.0, 2.0, 3.0],
    [5.0, 3.0, 2.0, -1.0],
])


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture
def toy() -> np.ndarray:
    return TOY.copy()


def random_instance(rng, n=None, m=None, zeros=False) -> np.ndarray:
    """pkg/tests/conftest.py:22-33: small uniform matrix, optional exact zeros."""
    if n is None:
        n = int(rng.integers(2, 21))
    if m is None:
        m = int(rng.integers(2, 7))
    X = rng.uniform(-10.0, 10.0, size=(n, m))
    if zeros:
        X[rng.random(size=X.shape) < 0.25] = 0.0
        if not X.any():
            X[0, 0] = 1.0
    return X


def load_golden(name: str):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def iter_random_small():
    """Yield (X, lams, pivot results, line results) from golden/random_small.npz."""
    g = load_golden("random_small.npz")
    shapes, X = g["shapes"], g["X"]
    lams = g["lams"]
    ox = opv = ope = 0
    for t, (n, m) in enumerate(shapes):
        n, m = int(n), int(m)
        L = lams.shape[1]
        Xt = X[ox:ox + n * m].reshape(n, m)
        ox += n * m
        pV = g["pV"][opv:opv + m * L * m].reshape(m, L, m)
        opv += m * L * m
        pE = g["pE"][ope:ope + m * L].reshape(m, L)
        pP = g["pP"][ope:ope + m * L].reshape(m, L)
        pO = g["pO"][ope:ope + m * L].reshape(m, L)
        ope += m * L
        yield t, Xt, lams[t], (pV, pE, pP, pO), g["lpiv"][t], g["lobj"][t], g["lerr"][t], g["lpen"][t]


def iter_random_small_lines():
    g = load_golden("random_small.npz")
    ov = 0
    out = []
    for t, (n, m) in enumerate(g["shapes"]):
        L = g["lams"].shape[1]
        out.append(g["lv"][ov:ov + L * int(m)].reshape(L, int(m)))
        ov += L * int(m)
    return out
