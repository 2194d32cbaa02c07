"""Per-CTA phase durations of k_select from %globaltimer stamps (l1b_set_probe).

    python tools/phase_probe.py [--config c2] [--lam 1.0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_16712_b200 as l1b  # noqa: E402
from paper_2402_16712_b200 import _lib  # noqa: E402
from paper_2402_16712_b200.engine import DeviceFit  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--lam", type=float, default=1.0)
a = ap.parse_args()
shapes = {"c2": (2000, 2000), "c4": (500, 100000), "c5": (10000, 10000)}
m, n = shapes[a.config]
d, _ = l1b.gen_line_data(m, n, seed=0, noise_scale=1.0)
eng = DeviceFit(np.array(d.values))
ncta = ((m + 31) // 32) * ((m + 7) // 8)
buf = torch.zeros(ncta * 8, dtype=torch.int64, device=eng.device)
eng.fit_pivots([a.lam], want_v=False)
lib = _lib.load()
lib.l1b_set_probe(buf.data_ptr())
eng.fit_pivots([a.lam], want_v=False)
torch.cuda.synchronize()
lib.l1b_set_probe(None)
t = buf.cpu().numpy().reshape(ncta, 8).astype(np.float64)
t0 = t[:, 0].min()
names = ["sample", "F", "B", "resolve"]
dur = np.diff(t[:, :5], axis=1) / 1e3  # us
print(f"{ncta} CTAs, kernel span {(t[:, 4].max() - t0) / 1e6:.2f} ms")
for k, nm in enumerate(names):
    print(f"  {nm:8s} mean {dur[:, k].mean():8.1f} us  p50 {np.median(dur[:, k]):8.1f}  p99 {np.percentile(dur[:, k], 99):8.1f}"
          f"  share {100 * dur[:, k].sum() / dur.sum():5.1f}%")
life = (t[:, 4] - t[:, 0]) / 1e3
print(f"  CTA life mean {life.mean():.1f} us; sum of lives / span = {life.sum() / ((t[:, 4].max() - t0) / 1e3):.1f} CTAs resident on average")
