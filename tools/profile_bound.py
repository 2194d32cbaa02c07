"""One K0 prepare + one bound pass on a BASELINE config, for ncu: fit_line's lean
first pass (l1b_bound_pivot_sums, the kernel bench.py times), or with --full the
pass that also leaves per-column bounds (l1b_bound_pivots).

    python tools/profile_bound.py [--config c2] [--lam 1.0] [--full]
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
ap.add_argument("--full", action="store_true")
a = ap.parse_args()
shapes = {"c2": (2000, 2000), "c4": (500, 100000), "c5": (10000, 10000)}
m, n = shapes[a.config]
d, _ = l1b.gen_line_data(m, n, seed=0, noise_scale=1.0)
eng = DeviceFit(np.array(d.values))
lb, ub = eng.bound_pivots(a.lam) if a.full else eng.bound_pivot_sums(a.lam)
torch.cuda.synchronize()
print("min ub", float(ub.min()), "candidates", int((lb <= ub.min() * (1 + 1e-9)).sum()))
