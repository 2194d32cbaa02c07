"""Run-to-run determinism as a race detector (compute-sanitizer is closed on
this GPU pool): every k_bound histogram sum and every exact-path result is an
exact integer or a fixed-order reduction, so a shared-memory race in the TMA
rings (a stage refilled while a warp still reads it, a histogram read before
every add landed) would show as a bound or a direction that changes between
identical runs.  Repeats each workload R times and compares bytes.

    python tools/race_stress.py [--reps 40]
"""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_16712_b200 as l1b  # noqa: E402
from paper_2402_16712_b200.engine import DeviceFit  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=40)
a = ap.parse_args()


def digest(*arrs):
    h = hashlib.blake2b(digest_size=12)
    for x in arrs:
        h.update(np.ascontiguousarray(x).tobytes())
    return h.hexdigest()


cases = {"c2-like 2000x600": l1b.gen_line_data(600, 2000, seed=0, noise_scale=1.0)[0].values,
         "tall 40000x64": l1b.gen_line_data(64, 40000, seed=1, noise_scale=1.0)[0].values,
         "outliers 300x120": l1b.gen_outlier_data(120, 300, 30, seed=2)[0].values}
bad = 0
for name, X in cases.items():
    X = np.array(X)
    eng = DeviceFit(X)
    T = float(np.abs(X).sum(axis=0).max())
    work = {
        "bound 1 pass (per-column LB/UB)": lambda: (eng.bound_pivots(1.0), eng.bound_columns(eng.m))[1],
        "bound 3 passes": lambda: eng.bound_pivot_list(1.0, np.arange(eng.m), passes=3),
        "multi-penalty bound": lambda: eng.bound_pivots_multi([0.0, 1.0, 0.3 * T])[:2],
        "exact all pivots": lambda: tuple(t.cpu().numpy() for t in eng.fit_pivots([1.0])),
        "pruned winner": lambda: (lambda w: (w.pivot, w.v, w.objective))(eng.shard_winners([1.0])[0]),
    }
    for what, fn in work.items():
        seen = set()
        for _ in range(a.reps):
            out = fn()
            torch.cuda.synchronize()
            seen.add(digest(*[np.asarray(o) for o in (out if isinstance(out, tuple) else (out,))]))
        status = "deterministic" if len(seen) == 1 else f"{len(seen)} DIFFERENT results"
        bad += len(seen) != 1
        print(f"{name:20s} {what:34s} x{a.reps}: {status}", flush=True)
print("race stress:", "clean" if bad == 0 else f"{bad} nondeterministic workloads")
sys.exit(1 if bad else 0)
