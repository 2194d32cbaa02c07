"""Time the UNMODIFIED reference package (l1line 0.1.0, installed offline into
baseline/_ref from /root/reference/pkg) on this host's cores: C2, the
reference CLI's own bench recipe (cli.py:246-260) -- gen_line_data(2000,
2000, seed=0, noise_scale=1.0), fit_line(data, 1.0, threads=os.cpu_count()),
perf_counter around fit_line only.  Not part of bench.py's contract (the
reference arm there is the oracle C port, which travels without the
reference tree); this records what the real package takes on the GPU host.

    python tools/time_reference_pkg.py [--lam 1.0] [--repeat 1]
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import l1line  # noqa: E402


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


ap = argparse.ArgumentParser()
ap.add_argument("--lam", type=float, default=1.0)
ap.add_argument("--m", type=int, default=2000)
ap.add_argument("--n", type=int, default=2000)
ap.add_argument("--repeat", type=int, default=1)
a = ap.parse_args()
data, _ = l1line.gen_line_data(a.m, a.n, seed=0, noise_scale=1.0)
threads = os.cpu_count()
best = None
for _ in range(a.repeat):
    t0 = time.perf_counter()
    line = l1line.fit_line(data, a.lam, threads=threads)
    dt = time.perf_counter() - t0
    best = dt if best is None else min(best, dt)
print(json.dumps({"package": "l1line " + getattr(l1line, "__version__", "0.1.0"), "module": l1line.__file__,
                  "config": {"n": a.n, "m": a.m, "lam": a.lam, "generator": "gen_line_data(seed=0, noise_scale=1.0)"},
                  "threads": threads, "cpu_model": cpu_model(), "seconds_per_fit": best,
                  "pivot": line.preserved, "objective": repr(line.objective),
                  "nonzeros": int((line.v != 0).sum())}))
