"""Where solution_path's time goes (Algorithm 2 + 3) on gen_line_data inputs.

    python tools/profile_path.py [--m 100] [--n 1000]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2402_16712_b200 as l1b  # noqa: E402
from paper_2402_16712_b200 import path as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=100)
ap.add_argument("--n", type=int, default=1000)
a = ap.parse_args()
d, _ = l1b.gen_line_data(a.m, a.n, seed=0, noise_scale=1.0)
t0 = time.perf_counter()
lam, sols = P.major_breakpoints(d)
t1 = time.perf_counter()
E = sum(len(e) for pb in sols.pivots.values() for e in pb.entries.values())
path = P.merge_path(lam, sols, d)
t2 = time.perf_counter()
print(f"{a.n}x{a.m}: grid K={lam.size}, events E={E}, segments={len(path.segments)}; "
      f"major_breakpoints {t1 - t0:.2f} s, merge_path {t2 - t1:.2f} s", flush=True)
t3 = time.perf_counter()
fast = P.solution_path(d)
t4 = time.perf_counter()
assert len(fast.segments) == len(path.segments)
print(f"  solution_path (array route, device merge): {t4 - t3:.2f} s", flush=True)
