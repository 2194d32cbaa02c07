"""One C4 step (fit_subspace's fit -> deflate loop, 3 components, X resident)
for ncu launch lists; prints each component's pivot and exactly fitted pivots.

    python tools/profile_subspace.py [--k 3] [--lam 1.0]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_16712_b200 as l1b  # noqa: E402
from paper_2402_16712_b200.engine import DeviceFit  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--k", type=int, default=3)
ap.add_argument("--lam", type=float, default=1.0)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
d, _ = l1b.gen_line_data(500, 100000, seed=0, noise_scale=1.0)
eng = DeviceFit(np.array(d.values))
X0 = eng.X.clone()
for rep in range(a.reps):
    eng.X.copy_(X0)
    eng.prepare()
    for t in range(a.k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.set_steer(0 if t == 0 else -1)  # fit_subspace's policy (api.fit_subspace, bench.py)
        w = eng.shard_winners([a.lam])[0]
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(f"component {t}: pivot {w.pivot} objective {w.objective!r} exactly fitted {eng.last_candidates} "
              f"fit {1e3 * (t1 - t0):.2f} ms")
        if t + 1 < a.k:
            eng.deflate(w.v)
            torch.cuda.synchronize()
            print(f"  deflate+prepare {1e3 * (time.perf_counter() - t1):.2f} ms")
