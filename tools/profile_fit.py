"""One prepare + one fit_pivots on a BASELINE config, for ncu launch lists / captures.

    python tools/profile_fit.py [--config c2] [--lam 1.0] [--reps 1]
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
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--time", action="store_true")
ap.add_argument("--strag", action="store_true", help="classify the straggler queue")
a = ap.parse_args()
shapes = {"c1": (50, 200), "c2": (2000, 2000), "c4": (500, 100000), "c5": (10000, 10000)}
m, n = shapes[a.config]
if a.config == "c1":
    d, _ = l1b.gen_outlier_data(m, n, n // 10, seed=0)
else:
    d, _ = l1b.gen_line_data(m, n, seed=0, noise_scale=1.0)
eng = DeviceFit(np.array(d.values))
for _ in range(a.reps):
    eng.prepare()
    V, E, P, O = eng.fit_pivots([a.lam], want_v=False)
torch.cuda.synchronize()
o = O.cpu().numpy()[0]
print("best pivot", int(np.argmin(o)), float(o.min()), "stragglers", eng.straggler_counts())
if a.time:
    ts = []
    for _ in range(5):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        eng.fit_pivots([a.lam], want_v=False)
        ev1.record()
        ev1.synchronize()
        ts.append(ev0.elapsed_time(ev1))
    print("fit_pivots ms", sorted(ts))

if a.strag:
    import ctypes
    from paper_2402_16712_b200 import _lib
    eng.fit_pivots([a.lam], want_v=False)
    dt = np.dtype([("kk", "<i4"), ("j", "<i4"), ("lo", "<u8"), ("hi", "<u8"), ("wb", "<f8"), ("G", "<f8")])
    buf = np.zeros(200000, dtype=dt)
    k = _lib.load().l1b_straggler_records(eng.n, eng.m, eng.max_pivots, eng.ws.data_ptr(), eng.ws.numel(),
                                          buf.ctypes.data, buf.size, torch.cuda.current_stream().cuda_stream)
    r = buf[:k]
    ZERO = 1 << 63
    lo_open = r["lo"] == 0
    hi_open = r["hi"] == np.uint64(2**64 - 1)
    span = (r["hi"].astype(np.float64) - r["lo"].astype(np.float64))
    print(f"stragglers {k}: lo-open {lo_open.sum()}, hi-open {hi_open.sum()}, finite {(~lo_open & ~hi_open).sum()}; "
          f"finite-span log2 quantiles {np.percentile(np.log2(span[~lo_open & ~hi_open] + 1), [10, 50, 90]) if (~lo_open & ~hi_open).any() else None}")
