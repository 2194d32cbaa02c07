"""A small workload touching every kernel family, for compute-sanitizer
(racecheck / synccheck / memcheck, one tool per run):

    compute-sanitizer --tool racecheck python tools/sanitize_fit.py

256x256 pruned fit_line (k_bound -> refining passes -> seeded exact solver ->
exact re-score), the unpruned exact path (k_select / k_resolve / k_straggle),
a 4-penalty sweep (multi-penalty k_bound + entry cascade), a tall pivot's
tableau (chunk sorts + global merges), certificates, brute force, deflation.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2402_16712_b200 as l1b  # noqa: E402
from paper_2402_16712_b200.engine import DeviceFit  # noqa: E402

d, _ = l1b.gen_line_data(256, 256, seed=1, noise_scale=1.0)
X = np.array(d.values)
eng = DeviceFit(X)
w = eng.shard_winners([1.0], prune=True)[0]
print("pruned fit_line: pivot", w.pivot, "candidates", eng.last_candidates)
V, E, P, O = eng.fit_pivots([1.0])
torch.cuda.synchronize()
print("exhaustive argmin", int(O.cpu().numpy()[0].argmin()))
T = float(np.abs(X).sum(axis=0).max())
ws = eng.shard_winners([0.0, 1.0, 0.1 * T, 0.5 * T], prune=True)
print("sweep pivots", [x.pivot for x in ws])
line = l1b.fit_line(d, 1.0)
c = l1b.certify_line(d, line)
print("certified columns", int(np.isfinite(c.slack).sum()), "refuted", len(c.refuted))
col = l1b.build_column(d, line.preserved, (line.preserved + 1) % d.m)
l1b.dual_certificate(col, l1b.solve_column(col, 1.0), 1.0)
print("brute force", l1b.brute_force_pivot(X[:64, :16], 3, 1.0).preserved)
t, _ = l1b.gen_line_data(3, 20000, seed=2, noise_scale=1.0)
tab = l1b.pivot_tableau(t, 0)
print("tall tableau", tab.ratios.shape)
sub = l1b.fit_subspace(d, 1.0, 2)
print("subspace", [c.preserved for c in sub.components])
torch.cuda.synchronize()
print("sanitize workload ok")
