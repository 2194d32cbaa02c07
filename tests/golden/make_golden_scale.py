"""At-scale parity fixtures from the REFERENCE implementation (BASELINE.json configs C2-C5).

Run in the build container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_scale.py c2 c3 c4 c5

The full matrices are regenerated from their seeds on the GPU box
(``paper_2402_16712_b200.datagen`` is byte-identical to ``l1line.datagen``,
tests/test_host.py), so only the reference's ANSWERS are committed here, a few
kilobytes per configuration:

* the winning line of every (config, penalty): pivot, v bytes, error,
  penalty, objective -- ``l1line.fit_line`` (fit.py:88-102);
* every pivot's objective and an 8-byte BLAKE2b digest of its v bytes, so the
  device's per-pivot results can be checked pivot by pivot, not just the argmin.

Per-pivot lines are computed with the reference's own functions in the
reference's own order: ``fit_for_pivot`` (fit.py:75-85) through
``map_indices`` (parallel.py:36-43), then the strict-``<`` argmin of
fit.py:98-102 -- exactly what ``fit_line`` does, with the per-pivot results
kept.  For the 32-penalty sweep (C3) each pivot's tableau is built once with
``pivot_tableau`` (ratios.py:109-135) and snapped for every penalty with
``_snap_all`` (fit.py:51-63) + ``FittedLine.build`` (core.py:126-133): the
tableau takes no penalty, so this is bit-identical to 32 ``fit_for_pivot``
calls (fit.py:79-85) at 1/15 of the time.  C4 follows ``fit_subspace``
(subspace.py:54-76) with the reference's ``deflate`` (subspace.py:22-36).
C5 (10000x10000; ~9 CPU-hours for a full fit) keeps 17 pivots: 16 evenly
spaced plus the device winner 1422, each through ``fit_for_pivot``.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import l1line  # noqa: E402
from l1line.fit import _snap_all  # noqa: E402
from l1line.parallel import map_indices  # noqa: E402
from l1line.ratios import EmptyPivotError, pivot_tableau  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
THREADS = int(os.environ.get("L1LINE_THREADS", os.cpu_count() or 1))


def vdigest(v: np.ndarray) -> np.uint64:
    return np.frombuffer(hashlib.blake2b(np.ascontiguousarray(v, dtype=np.float64).tobytes(),
                                         digest_size=8).digest(), dtype=np.uint64)[0]


def c3_lams(X: np.ndarray) -> list[float]:
    """lam_k = (k/31) * max_p sum_i |x_ip|, k = 0..31."""
    tmax = float(np.abs(X).sum(axis=0).max())
    return [(k / 31.0) * tmax for k in range(32)]


def _per_pivot(d, lams, threads=THREADS):
    """Reference lines of every pivot for every penalty: list[m] of list[L] FittedLine."""
    def one(p):
        if len(lams) == 1:
            return [l1line.fit_for_pivot(d, p, lams[0])]
        try:
            tab = pivot_tableau(d, p)
        except EmptyPivotError:
            return [l1line.degenerate_line(d, p, lam) for lam in lams]
        out = []
        for lam in lams:
            v = np.zeros(d.m)
            v[p] = 1.0
            v[tab.targets] = _snap_all(tab, float(lam))
            out.append(l1line.FittedLine.build(d, v, p, float(lam)))
        return out
    return map_indices(one, d.m, threads)


def _winner(lines):
    best = lines[0]
    for line in lines[1:]:
        if line.objective < best.objective:     # fit.py:98-102
            best = line
    return best


def _pack(prefix, per_pivot, L):
    """Arrays for L penalties: winner record + per-pivot objective / digest / nnz."""
    m = len(per_pivot)
    out = {}
    wins = [_winner([per_pivot[p][k] for p in range(m)]) for k in range(L)]
    out[prefix + "piv"] = np.array([w.preserved for w in wins], dtype=np.int64)
    out[prefix + "v"] = np.stack([w.v for w in wins])
    out[prefix + "err"] = np.array([w.error for w in wins])
    out[prefix + "pen"] = np.array([w.penalty_norm for w in wins])
    out[prefix + "obj"] = np.array([w.objective for w in wins])
    out[prefix + "pobj"] = np.array([[per_pivot[p][k].objective for p in range(m)] for k in range(L)])
    out[prefix + "pdig"] = np.array([[vdigest(per_pivot[p][k].v) for p in range(m)] for k in range(L)],
                                    dtype=np.uint64)
    out[prefix + "pnnz"] = np.array([[np.count_nonzero(per_pivot[p][k].v) for p in range(m)] for k in range(L)],
                                    dtype=np.int32)
    return out


def grid(X):
    return np.round(X * 2.0**20) / 2.0**20


def c2():
    """C2: gen_line_data(2000, 2000, seed=0, noise_scale=1.0), raw and grid, lam in {1, 2500}."""
    X, _ = l1line.gen_line_data(2000, 2000, seed=0, noise_scale=1.0)
    X = np.asarray(X.values)
    lams = [1.0, 2500.0]
    out = {"lams": np.array(lams)}
    for tag, Xv in (("raw_", X), ("grid_", grid(X))):
        d = l1line.DataMatrix(Xv)
        for k, lam in enumerate(lams):
            t0 = time.time()
            pp = _per_pivot(d, [lam])
            out.update(_pack(f"{tag}{k}_", pp, 1))
            w = _winner([p[0] for p in pp])
            # the winner must be what fit_line itself reports (same code, fit.py:88-102)
            print(f"c2 {tag}lam={lam}: pivot {w.preserved} obj {w.objective!r} "
                  f"nnz {np.count_nonzero(w.v)} ({time.time() - t0:.0f} s)", flush=True)
    np.savez_compressed(os.path.join(OUT, "scale_c2.npz"), **out)


def c3():
    """C3: the 32-penalty sweep on C2's raw data."""
    X, _ = l1line.gen_line_data(2000, 2000, seed=0, noise_scale=1.0)
    d = l1line.DataMatrix(np.asarray(X.values))
    lams = c3_lams(d.values)
    t0 = time.time()
    pp = _per_pivot(d, lams)
    out = {"lams": np.array(lams)}
    out.update(_pack("raw_", pp, len(lams)))
    print(f"c3: pivots {out['raw_piv'].tolist()} ({time.time() - t0:.0f} s)", flush=True)
    np.savez_compressed(os.path.join(OUT, "scale_c3.npz"), **out)


def c4():
    """C4: gen_line_data(500, 100000, seed=0, noise_scale=1.0), fit_subspace(k=3) at lam=1."""
    X, _ = l1line.gen_line_data(500, 100000, seed=0, noise_scale=1.0)
    cur = X
    lam, k = 1.0, 3
    out = {"lams": np.array([lam])}
    scale = max(1.0, float(np.abs(X.values).max()))
    for c in range(k):
        assert float(np.abs(cur.values).max()) > 1e-10 * scale      # subspace.py:67
        t0 = time.time()
        pp = _per_pivot(cur, [lam])
        out.update(_pack(f"comp{c}_", pp, 1))
        w = _winner([p[0] for p in pp])
        print(f"c4 comp {c}: pivot {w.preserved} obj {w.objective!r} ({time.time() - t0:.0f} s)", flush=True)
        cur = l1line.deflate(cur, w.v)                                  # subspace.py:75
    np.savez_compressed(os.path.join(OUT, "scale_c4.npz"), **out)


C5_PIVOTS = sorted(set(np.linspace(0, 9999, 16).astype(int).tolist()) | {1422})


def c5():
    """C5: gen_line_data(10000, 10000, seed=0, noise_scale=1.0), 17 pivots at lam=1."""
    X, _ = l1line.gen_line_data(10000, 10000, seed=0, noise_scale=1.0)
    lam = 1.0
    t0 = time.time()
    # 4.8 GB of temporaries per in-flight pivot: cap workers by RAM
    lines = map_indices(lambda i: l1line.fit_for_pivot(X, C5_PIVOTS[i], lam), len(C5_PIVOTS), min(THREADS, 6))
    out = {"lams": np.array([lam]), "pivots": np.array(C5_PIVOTS, dtype=np.int64)}
    out["pobj"] = np.array([l.objective for l in lines])
    out["perr"] = np.array([l.error for l in lines])
    out["ppen"] = np.array([l.penalty_norm for l in lines])
    out["pdig"] = np.array([vdigest(l.v) for l in lines], dtype=np.uint64)
    out["pnnz"] = np.array([np.count_nonzero(l.v) for l in lines], dtype=np.int32)
    out["v1422"] = lines[C5_PIVOTS.index(1422)].v
    print(f"c5: {len(lines)} pivots ({time.time() - t0:.0f} s); best sampled "
          f"{C5_PIVOTS[int(np.argmin(out['pobj']))]}", flush=True)
    np.savez_compressed(os.path.join(OUT, "scale_c5.npz"), **out)


if __name__ == "__main__":
    for job in sys.argv[1:] or ["c2", "c3", "c4", "c5"]:
        {"c2": c2, "c3": c3, "c4": c4, "c5": c5}[job]()
