"""Randomised check that every pruned fit path (l1b_fit_line, the batched sweep)
returns exactly the unpruned winner: random shapes, Gaussian / Cauchy / tied /
sparse / line / badly scaled / grid data, four penalties each.

    python tools/stress_prune_large.py SEED SECONDS  (m 150-500, n 500-20000)
    STRESS_M=20-80 STRESS_N=16384-120000 python tools/stress_prune_large.py ...  (tall columns)
"""
import sys, os, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2402_16712_b200 as l1b
from paper_2402_16712_b200.engine import DeviceFit
M_LO, M_HI = map(int, os.environ.get("STRESS_M", "150-500").split("-"))
N_LO, N_HI = map(int, os.environ.get("STRESS_N", "500-20000").split("-"))
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
bad = 0; t0 = time.time(); cnt = 0
while time.time() - t0 < float(sys.argv[2]) if len(sys.argv) > 2 else 60:
    m = int(rng.integers(M_LO, M_HI)); n = int(rng.integers(N_LO, N_HI))
    kind = int(rng.integers(0, 7))
    if kind == 0:
        X = rng.standard_normal((n, m))
    elif kind == 1:
        X = rng.standard_cauchy((n, m))
    elif kind == 2:
        X = np.round(rng.uniform(-5, 5, (n, m)))          # heavy exact ties + zeros
    elif kind == 3:
        X = rng.standard_normal((n, m)); X[rng.random((n, m)) < 0.4] = 0.0
    elif kind == 4:
        d, _ = l1b.gen_line_data(m, n, seed=int(rng.integers(1 << 30)), noise_scale=float(rng.uniform(0.01, 5)))
        X = np.array(d.values)
    elif kind == 5:
        X = rng.standard_normal((n, m)) * np.exp(rng.uniform(-8, 8, (1, m)))   # wildly different column scales
    else:
        d, _ = l1b.gen_line_data(m, n, seed=int(rng.integers(1 << 30)), noise_scale=1.0)
        X = np.round(np.array(d.values) * 2**8) / 2**8
        X[:, int(rng.integers(m))] = 0.0                 # a degenerate pivot
    if not np.any(X):
        continue
    T = float(np.abs(X).sum(axis=0).max())
    lams = [0.0, float(rng.uniform(0, 3)), float(rng.uniform(0, 0.3)) * T, float(rng.uniform(0.3, 1.5)) * T]
    eng = DeviceFit(X)
    full = eng.shard_winners(lams, prune=False)
    for lam, want in zip(lams, full):
        try:
            got = eng.fit_line_device(lam, prune=True)
        except Exception as e:
            print("ERROR", e, "kind", kind, X.shape, "lam", lam, flush=True)
            os.makedirs("gpurun_out", exist_ok=True)
            np.save("gpurun_out/fail_X.npy", X); np.save("gpurun_out/fail_lam.npy", np.array([lam]))
            raise
        if not (got.pivot == want.pivot and got.v.tobytes() == want.v.tobytes() and got.objective == want.objective):
            bad += 1
            print("MISMATCH kind", kind, "shape", X.shape, "lam", lam, got.pivot, want.pivot, got.objective, want.objective, flush=True)
    sweep = eng.shard_winners(lams, prune=True)
    for lam, a, b in zip(lams, sweep, full):
        if not (a.pivot == b.pivot and a.v.tobytes() == b.v.tobytes() and a.objective == b.objective):
            bad += 1
            print("SWEEP MISMATCH kind", kind, "shape", X.shape, "lam", lam, a.pivot, b.pivot, flush=True)
    cnt += 1
print("instances", cnt, "mismatches", bad)
