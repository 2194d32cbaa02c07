"""How tight are the one-, two- and three-pass pivot bounds on a config's
components?  Prints, per component, the spread of the exact per-pivot
objectives, the bounds' relative gaps and how many pivots each pass prunes.

    python tools/bound_gaps.py [--config c4] [--comps 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_16712_b200 as l1b  # noqa: E402
from paper_2402_16712_b200.engine import DeviceFit  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--comps", type=int, default=3)
ap.add_argument("--lam", type=float, default=1.0)
a = ap.parse_args()
shapes = {"c2": (2000, 2000), "c4": (500, 100000), "c5": (10000, 10000)}
m, n = shapes[a.config]
d, _ = l1b.gen_line_data(m, n, seed=0, noise_scale=1.0)
eng = DeviceFit(np.array(d.values))
piv = np.arange(m)
for comp in range(a.comps):
    _, _, _, O = eng.fit_pivots([a.lam], want_v=False)
    O = O.cpu().numpy()[0]
    best = O.min()
    rel = (O - best) / best
    print(f"comp {comp}: best pivot {int(O.argmin())}; exact objectives above the best by "
          f"q10/50/90 = {np.quantile(rel, [0.1, 0.5, 0.9])}")
    for passes in (1, 2, 3):
        lb, ub = eng.bound_pivot_list(a.lam, piv, passes=passes)
        top = ub.min()
        gap = (ub - lb) / ub
        keep = int((lb <= top * (1 + 1e-9)).sum())
        print(f"  {passes} pass(es): gap q10/50/90 = {np.quantile(gap, [0.1, 0.5, 0.9])}, "
              f"ub-best {(top - best) / best:.2e}, survivors {keep}")
    w = eng.shard_winners([a.lam])[0]
    eng.deflate(w.v)
torch.cuda.synchronize()
