"""One full bench step (K0 prepare + pruned fit_line with exact re-scoring) on a
BASELINE config, for ncu launch lists.

    python tools/profile_step.py [--config c2|c3|c4|c5] [--lam 1.0]
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
ap.add_argument("--config", default="c2")
ap.add_argument("--lam", type=float, default=1.0)
a = ap.parse_args()
shapes = {"c2": (2000, 2000), "c3": (2000, 2000), "c4": (500, 100000), "c5": (10000, 10000)}
m, n = shapes[a.config]
d, _ = l1b.gen_line_data(m, n, seed=0, noise_scale=1.0)
X = np.array(d.values)
# C3: the 32-penalty grid of SURVEY.md 8d (lambda_k = k/31 max_p sum_i |x_ip|)
lams = [k / 31.0 * float(np.abs(X).sum(axis=0).max()) for k in range(32)] if a.config == "c3" else [a.lam]
eng = DeviceFit(X)
# DeviceFit() already ran K0 (prepare)
w = eng.shard_winners(lams)[0]
torch.cuda.synchronize()
print("winner", w.pivot, repr(w.objective), "exactly fitted pivots", eng.last_candidates)
