"""Benchmark: Algorithm 1 (fit_line) on the B200 against the CPU reference path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One JSON line on rank 0.  A "step" is one complete fit_line over one
synthetic input (BASELINE.json configs[1] = C2: gen_line_data(m=2000,
n=2000, seed=0, noise_scale=1), lambda = 1 -- the reference CLI's bench
recipe, cli.py:246-260).  Metric: BASELINE.json's "ms per sparse L1 line fit
at 2000x2000 and weighted-median solves/sec"; ``value`` is solves/s for the
whole job (m(m-1) weighted-median problems per fit), ``ms_per_step`` is ms
per fit.  (solves/s is nominal under pruning: every problem is bounded, only
the surviving pivots' problems are solved exactly -- results identical.)

* value       -- X resident in HBM; device time of K fits with CUDA events on
                 the launching stream, L2 flushed (256 MB write) before every
                 timed fit, max over ranks.  A fit = K0 prepare + the pruned
                 cascade (one k_bound pass over every problem, refining passes
                 over the survivors, the seeded exact solver) + exact
                 re-scoring of the winner in NumPy's summation order.
* e2e         -- the public API (paper_2402_16712_b200.fit_line) from a host
                 numpy array: H2D of X, the fit, D2H of the line, per step.
* roofline    -- k_bound, the dominant kernel: one shared-memory histogram
                 atomic per (pivot, target, row) element over its event-timed
                 duration, against the conflict-free red.shared rate measured
                 here (l1b_atoms_probe); exact_fit_view reports the exhaustive
                 exact path (k_select & co.) against the FP64 pipe.
* cpu_baseline -- the reference package itself (l1line, installed offline in
                 baseline/_ref) on this host's cores, or the oracle C port where
                 it is absent; a bounded, evenly spread pivot sample,
                 extrapolated to a full fit.  rank 0, N=1 only.

--impl reference times the reference arm: on C1/C2 the unmodified l1line's
own fit_for_pivot + thread pool over ONE complete fit whose pivots are split
across the timed steps (each pivot timed once, the argmin printed); elsewhere
the oracle C port (C3: full fit; C4/C5: strided sample, extrapolated).
Multi-GPU (torchrun, one process per GPU, NCCL): pivots are interleaved over
ranks, the winner is combined with one all_gather + one
broadcast; total work is fixed, so scaling is "strong".
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (generator, m, n, lams, description)
    "c1": ("outlier", 50, 200, [0.1], "synthetic 200x50 + 10% outliers, lambda=0.1"),
    "c2": ("line", 2000, 2000, [1.0], "paper benchmark 2000x2000 synthetic, lambda=1"),
    "c3": ("line", 2000, 2000, None, "lambda sweep of 32 penalties on 2000x2000"),
    "c4": ("line", 500, 100000, [1.0], "tall 100000x500, 3 components via deflation"),
    "c5": ("line", 10000, 10000, [1.0], "10000x10000, pivots sharded across GPUs"),
}
COMPONENTS = {"c4": 3}
METRIC = "ms per sparse L1 line fit at 2000×2000 and weighted-median solves/sec vs CPU"


def _make_data(cfg):
    import paper_2402_16712_b200 as l1b
    kind, m, n, lams, _ = CONFIGS[cfg]
    if kind == "outlier":
        d, _ = l1b.gen_outlier_data(m, n, n // 10, seed=0)
    else:
        d, _ = l1b.gen_line_data(m, n, seed=0, noise_scale=1.0)
    X = d.values
    if lams is None:  # C3 grid: lambda_k = (k/31) max_p sum_i |x_ip|
        tmax = float(np.abs(X).sum(axis=0).max())
        lams = [k / 31.0 * tmax for k in range(32)]
    return X, lams


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during timing."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.02):
        self.samples, self.reasons, self.ok = [], 0, False
        self.period, self.index = period, index
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # noqa: BLE001 -- clocks are best-effort metadata
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [v for k, v in self.REASONS.items() if self.reasons & k and v != "gpu_idle"]
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(self.samples)}


def cpu_reference(X, lams, budget_s: float, threads: int | None = None):
    """Time the CPU oracle (C port of the reference algorithm) on a pivot sample.

    Batches of `threads` pivots, evenly strided over the whole range (so the
    sample does not depend on where the cheap or costly pivots sit), one
    pivot per worker thread, until `budget_s` elapses or every pivot is done;
    returns (solves/s, seconds per full fit (extrapolated), sample).
    """
    from concurrent.futures import FIRST_COMPLETED, ThreadPoolExecutor, wait
    n, m = X.shape
    threads = threads or os.cpu_count() or 1
    order = np.argsort((np.arange(m) * 0.6180339887498949) % 1.0, kind="stable")  # low-discrepancy order
    ref = _reference_package() if len(lams) == 1 else None
    if ref is not None:  # the reference package itself: fit_for_pivot, one task per pivot
        l1line, _ = ref
        data = l1line.DataMatrix(X)

        def one(p):
            l1line.fit_for_pivot(data, int(p), float(lams[0]))
    else:
        import oracle

        def one(p):
            oracle.fit_pivots(X, lams, int(p), int(p) + 1, threads=1, want_v=False)
    # a window of 2 x threads tasks in flight, refilled as they finish, until the
    # budget is spent: every worker stays busy (no per-batch tail)
    done, nxt, t0 = 0, 0, time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as pool:
        live = set()
        while nxt < m and len(live) < 2 * threads:
            live.add(pool.submit(one, order[nxt]))
            nxt += 1
        while live:
            fin, live = wait(live, return_when=FIRST_COMPLETED)
            done += len(fin)
            if time.perf_counter() - t0 < budget_s:
                while nxt < m and len(live) < 2 * threads:
                    live.add(pool.submit(one, order[nxt]))
                    nxt += 1
    dt = time.perf_counter() - t0
    solves = done * (m - 1) * len(lams)
    per_fit = dt * m / done / len(lams)
    what = "l1line.fit_for_pivot (baseline/_ref)" if ref is not None else "oracle C port"
    if ref is None and len(lams) > 1:
        what += (" (one tableau per pivot shared by every penalty: faster than the reference's one fit_line "
                 "per penalty)")
    return (solves / dt, per_fit, f"{what}: {done}/{m} pivots (evenly spread) x {len(lams)} lambda of the same "
            f"input on {threads} threads, {dt:.1f}s", "reference" if ref is not None else "port")


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _argmin_strict(O):
    """fit.py:98-102: first pivot with the smallest objective (strict '<' in pivot order)."""
    best = 0
    for p in range(1, O.size):
        if O[p] < O[best]:
            best = p
    return best


def run_reference(args):
    """The reference algorithm on this host's cores (the oracle C port, OpenMP over
    pivots like parallel.py:36-43).

    C1-C3: the timed steps partition the pivots -- step k fits pivots
    [k m / K, (k + 1) m / K) -- so every pivot of ONE complete fit is timed
    exactly once and nothing is extrapolated; the strict-'<' argmin over all
    of them (fit.py:98-102) is printed, so the run also checks the GPU's
    winner.  C4 / C5 (minutes to hours of CPU per fit): the steps partition an
    evenly strided pivot sample and the fit time is extrapolated (labelled).
    """
    world, rank, _ = _dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        if rank != 0:
            dist.barrier()
            dist.destroy_process_group()
            return
    X, lams = _make_data(args.config)
    n, m = X.shape
    threads = os.cpu_count() or 1
    ncomp = COMPONENTS.get(args.config, 1)
    ref = _reference_package() if args.config in ("c1", "c2") and not args.port else None
    if ref is not None:
        return _run_reference_package(args, ref, X, lams, threads, world)
    import oracle
    full = args.config in ("c1", "c2", "c3")
    if full:
        pivots = np.arange(m)
    else:  # an evenly strided sample of about 4 pivots per thread
        cnt = min(m, 4 * threads)
        pivots = np.unique(np.linspace(0, m - 1, cnt).astype(np.int64))
    K = max(1, args.steps)
    whole = args.config == "c1"  # a complete fit takes milliseconds: every step is one
    bounds = [int(round(k * pivots.size / K)) for k in range(K + 1)]
    if whole:
        bounds = None
    for w in range(args.warmup):  # untimed: one batch of `threads` pivots
        lo = (w * threads) % m
        oracle.fit_pivots(X, lams, lo, min(m, lo + threads), threads=threads, want_v=False)
    t_steps, objs = [], []
    t_wall = time.perf_counter()
    for k in range(K):
        sel = pivots if whole else pivots[bounds[k]:bounds[k + 1]]
        t0 = time.perf_counter()
        O_parts = []
        if sel.size:
            if full:  # a contiguous range
                _, _, _, O = oracle.fit_pivots(X, lams, int(sel[0]), int(sel[-1]) + 1, threads=threads,
                                               want_v=False)
                O_parts.append(O)
            else:  # a strided sample: one pivot per worker thread
                O_parts.append(_fit_pivot_set(oracle, X, lams, sel, threads)[3])
        t_steps.append(time.perf_counter() - t0)
        objs = O_parts if whole else objs + O_parts
    wall = time.perf_counter() - t_wall
    O = np.concatenate(objs, axis=0) if objs else np.zeros((0, len(lams)))
    # seconds per complete workload pass
    t_fit = float(np.mean(t_steps)) if whole else float(np.sum(t_steps)) * (m / pivots.size) * ncomp
    solves = m * (m - 1) * len(lams) * ncomp
    v = solves / t_fit
    result = None
    if full:
        win = [_argmin_strict(O[:, l]) for l in range(len(lams))]
        result = {"pivot": win[:4], "objective": [float(O[w, l]) for l, w in enumerate(win)][:4]}
    sample = (f"a complete fit per step (all {m} pivots x {len(lams)} lambda)" if whole else
              f"one complete fit: all {m} pivots x {len(lams)} lambda, each timed once across the {K} steps"
              if full else
              f"{pivots.size} of {m} pivots (evenly strided) x {len(lams)} lambda, extrapolated x{m / pivots.size:.1f}"
              + (f" x {ncomp} components (component 1's data)" if ncomp > 1 else ""))
    if args.config == "c3":
        sample += ("; the port builds each pivot's tableau once for all 32 penalties (the reference calls "
                   "fit_line 32 times and re-sorts every time, fit.py:79), so this arm is faster than the reference")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(t_steps)),
        "ms_per_fit": 1e3 * t_fit, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_dict(args, X, lams, world),
        "cpu_baseline": {"value": v, "unit": "solves/s", "cores": threads, "kind": "port",
                         "cpu_model": _cpu_model(), "sample": sample,
                         "extrapolated": not full, "fits_in_driver_run": bool(full),
                         "timed_s": float(np.sum(t_steps)), "wall_s": wall},
        "result": result,
        "e2e": {"value": v, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def _reference_package():
    """The unmodified reference package (l1line 0.1.0), installed offline into
    baseline/_ref, or None where it is absent."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "l1line")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    try:
        import l1line
        from l1line.parallel import map_indices
    except Exception:  # noqa: BLE001 -- fall back to the port
        return None
    return l1line, map_indices


def _run_reference_package(args, ref, X, lams, threads, world):
    """The reference's own fit_line (fit.py:88-102) on all host cores, timed in
    K steps without splitting it: fit_for_pivot (fit.py:75-85) for every pivot
    through one ThreadPoolExecutor.map over range(m) -- exactly what
    parallel.map_indices (parallel.py:36-43) does inside fit_line -- and the
    in-order results timestamped at the K chunk boundaries (pivot k m / K), so
    step k is the time the fit spent between two boundaries, the steps add up
    to one complete fit (no per-step pool start or tail), and the strict '<'
    argmin in pivot order (fit.py:98-102) over all of them is its answer.
    C1 (milliseconds per fit) runs l1line.fit_line itself once per step."""
    from concurrent.futures import ThreadPoolExecutor
    l1line, map_indices = ref
    n, m = X.shape
    data = l1line.DataMatrix(X)
    lam = float(lams[0])
    K = max(1, args.steps)
    whole = args.config == "c1"
    for w in range(args.warmup):  # untimed: one batch of `threads` pivots
        lo = (w * threads) % m
        map_indices(lambda i: l1line.fit_for_pivot(data, lo + i, lam), min(threads, m - lo), threads)
    t_steps, best = [], None
    if whole:
        for k in range(K):
            t0 = time.perf_counter()
            best = l1line.fit_line(data, lam, threads=threads)
            t_steps.append(time.perf_counter() - t0)
    else:
        bounds = [(k + 1) * m // K for k in range(K)]
        lines = []
        with ThreadPoolExecutor(max_workers=min(threads, m)) as pool:
            t_prev = time.perf_counter()
            nxt = 0
            for i, line in enumerate(pool.map(lambda p: l1line.fit_for_pivot(data, p, lam), range(m))):
                lines.append(line)
                while nxt < K and i + 1 == bounds[nxt]:
                    t = time.perf_counter()
                    t_steps.append(t - t_prev)
                    t_prev = t
                    nxt += 1
        best = lines[0]
        for line in lines[1:]:
            if line.objective < best.objective:  # fit.py:98-102
                best = line
    t_fit = float(np.mean(t_steps)) if whole else float(np.sum(t_steps))
    v = m * (m - 1) / t_fit
    sample = ("l1line.fit_line, a complete fit per step" if whole else
              f"one complete l1line fit: fit_for_pivot on all {m} pivots through one ThreadPoolExecutor.map "
              f"(parallel.map_indices' mechanism), timed in {K} steps at pivot boundaries k*m/K")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "solves/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(t_steps)),
        "ms_per_fit": 1e3 * t_fit, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_dict(args, X, lams, world),
        "cpu_baseline": {"value": v, "unit": "solves/s", "cores": threads, "kind": "reference",
                         "package": "l1line 0.1.0 (baseline/_ref, unmodified)", "cpu_model": _cpu_model(),
                         "sample": sample, "extrapolated": False, "fits_in_driver_run": True,
                         "timed_s": float(np.sum(t_steps))},
        "result": {"pivot": [best.preserved], "objective": [best.objective]},
        "e2e": {"value": v, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def _fit_pivot_set(oracle, X, lams, pivots, threads):
    """oracle.fit_pivots over an arbitrary pivot set, threads in parallel (one pivot each)."""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(threads, len(pivots))) as ex:
        parts = list(ex.map(lambda p: oracle.fit_pivots(X, lams, int(p), int(p) + 1, threads=1, want_v=False),
                            pivots))
    return (None, np.concatenate([q[1] for q in parts]), np.concatenate([q[2] for q in parts]),
            np.concatenate([q[3] for q in parts]))


def _config_dict(args, X, lams, world):
    n, m = X.shape
    return {"workload": args.config, "description": CONFIGS[args.config][4], "n": n, "m": m,
            "n_lambdas": len(lams), "lambda": lams[0] if len(lams) == 1 else [lams[0], lams[-1]],
            "components": COMPONENTS.get(args.config, 1),
            "solves_per_step": m * (m - 1) * len(lams) * COMPONENTS.get(args.config, 1),
            "ratio_elements_per_fit": m * (m - 1) * n,
            "parallelism": f"pivot-shard x{world}" if world > 1 else "1 gpu",
            "l2": "flushed (256 MB write) before every timed step"}


def _sync_time(stream, fn):
    """Device time of fn() on `stream` with CUDA events (ms) and its result."""
    import torch
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    out = fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b), out


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2402_16712_b200 as l1b
    from paper_2402_16712_b200 import _lib
    from paper_2402_16712_b200.distributed import combine_winners, ub_exchange
    from paper_2402_16712_b200.engine import DeviceFit, shard

    world, rank, local = _dist_env()
    # one process per GPU over NCCL; L1B200_DIST_BACKEND=gloo lets several
    # ranks share a GPU (plumbing check only: the ranks never wait on one
    # another's kernels, only on host-side collectives)
    backend = os.environ.get("L1B200_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    lib = _lib.load()
    X, lams = _make_data(args.config)
    n, m = X.shape
    ncomp = COMPONENTS.get(args.config, 1)
    p_begin, p_stride, npiv = shard(m, rank, world)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    eng = DeviceFit(X, device=dev, max_pivots=max(1, npiv))
    X0 = eng.X.clone() if ncomp > 1 else None

    # sharded pruning: one all-reduce(MIN) of the best upper bound per lambda
    ex = ub_exchange() if world > 1 and eng.auto_prune() else None

    def step():
        """One workload pass with X resident: fit_line (every lambda), or
        fit_subspace's fit -> deflate loop (subspace.py:54-76) for C4."""
        if X0 is not None:
            eng.X.copy_(X0)
        eng.prepare()
        out = []
        scale = max(1.0, eng.absmax()) if ncomp > 1 else 1.0
        for t in range(ncomp):
            if ncomp > 1 and eng.absmax() <= 1e-10 * scale:
                break
            if ncomp > 1:  # fit_subspace's steering policy (api.fit_subspace)
                eng.set_steer(0 if t == 0 else -1)
            wins = eng.shard_winners(lams, p_begin, p_stride, npiv, ub_exchange=ex)
            if world > 1:
                wins = combine_winners(wins, m)
            out.append(wins)
            if t + 1 < ncomp:
                eng.deflate(wins[0].v)
        return out

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    # ---- device-resident timing (value) ----------------------------------
    launches0 = lib.l1b_kernel_launches()
    times = []
    barrier()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            ms, res = _sync_time(stream, step)
            times.append(ms)
    barrier()
    launches = (lib.l1b_kernel_launches() - launches0) / args.steps
    ms_total = max_over_ranks(float(np.sum(times)))
    solves_step = m * (m - 1) * len(lams) * ncomp
    value = solves_step * args.steps / (ms_total / 1e3)

    # ---- dominant kernel: K1 (k_select + stragglers) alone, same stream ----
    if X0 is not None:
        eng.X.copy_(X0)
    eng.prepare()
    sel_ms = []
    for _ in range(max(3, min(args.steps, 5))):
        flush.fill_(1)
        ms, _ = _sync_time(stream, lambda: eng.fit_pivots(lams, p_begin, p_stride, npiv, want_v=False))
        sel_ms.append(ms)
    sel_ms = float(np.median(sel_ms))
    strag = eng.straggler_counts(npiv)[0]
    # the pruned step's dominant kernel: k_bound, the bounding pass over every
    # problem exactly as the step runs it (fit_line's lean first pass; a
    # sweep's multi-penalty pass), timed by the library's CUDA events on its
    # stream
    bnd_ms, kb_ms = [], []
    ulams = sorted(set(float(x) for x in lams))
    multi = len(ulams) > 1 and all(np.isfinite(ulams))  # a sweep bounds every penalty in one pass
    for _ in range(max(3, min(args.steps, 5))):
        flush.fill_(1)
        ms, _ = _sync_time(stream, (lambda: eng.bound_pivots_multi(ulams, p_begin, p_stride, npiv)) if multi
                           else (lambda: eng.bound_pivot_sums(lams[0], p_begin, p_stride, npiv)))
        bnd_ms.append(ms)
        kb = ctypes.c_float()
        _lib.check(lib.l1b_last_bound_ms(ctypes.byref(kb)), "l1b_last_bound_ms")
        kb_ms.append(kb.value)
    bnd_ms = float(np.median(bnd_ms))
    kb_ms = float(np.median(kb_ms))
    cand = [None] * len(lams)
    for li, lam_l in enumerate(lams):
        eng.shard_winners([lam_l], p_begin, p_stride, npiv)
        cand[li] = eng.last_candidates

    # ---- FP64 peak probe ---------------------------------------------------
    probe = torch.zeros(1, dtype=torch.float64, device=dev)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    iters, blocks, thr = 1 << 14, nsm * 8, 256
    _lib.check(lib.l1b_dfma_probe(iters, blocks, thr, probe.data_ptr(), stream.cuda_stream), "probe")
    pms, _ = _sync_time(stream, lambda: _lib.check(
        lib.l1b_dfma_probe(iters, blocks, thr, probe.data_ptr(), stream.cuda_stream), "probe"))
    fp64_ops = 8.0 * iters * blocks * thr / (pms / 1e3)  # DFMA per second

    elems = npiv * (m - 1) * n * len(lams)  # ratio elements one fit_pivots call covers on this rank
    achieved = 11.0 * elems / (sel_ms / 1e3)

    # ---- shared-memory atomic peak probe (k_bound's binding operation) -----
    pu = torch.zeros(1, dtype=torch.int32, device=dev)
    a_iters, a_blocks, a_thr = 1 << 13, nsm * 2, 256
    _lib.check(lib.l1b_atoms_probe(a_iters, a_blocks, a_thr, pu.data_ptr(), stream.cuda_stream), "atoms")
    ams, _ = _sync_time(stream, lambda: _lib.check(
        lib.l1b_atoms_probe(a_iters, a_blocks, a_thr, pu.data_ptr(), stream.cuda_stream), "atoms"))
    atoms_peak = 8.0 * a_iters * a_blocks * a_thr / (ams / 1e3)  # lane atomics per second
    kb_elems = npiv * (m - 1) * n  # one histogram add per (pivot, target, row) per launch
    kb_rate = kb_elems / (kb_ms / 1e3)

    # ---- end to end through the public API (host numpy in, FittedLine out) --
    data = l1b.DataMatrix(X)  # built once, as the reference CLI does before timing fit_line
    from paper_2402_16712_b200 import api as _api
    if world == 1:
        def e2e_step():
            # no device replica carried over from the last step: every step
            # uploads X (the library keeps one per read-only input otherwise)
            _api.clear_device_cache()
            if ncomp > 1:
                return l1b.fit_subspace(data, lams[0], ncomp)
            return l1b.fit_lines(data, lams)
    else:
        from paper_2402_16712_b200.distributed import fit_lines_distributed, fit_subspace_distributed

        def e2e_step():
            if ncomp > 1:
                return fit_subspace_distributed(data, lams[0], ncomp)
            return fit_lines_distributed(data, lams)
    e2e_ms = []
    for k in range(args.warmup + args.steps):
        barrier()
        ms, res = _sync_time(stream, e2e_step)
        if k >= args.warmup:
            e2e_ms.append(ms)
    lines = list(res.components) if ncomp > 1 else res
    # optimality certificate of every column of the first winning line (device,
    # outside the timed region; oracle.py:141-174's dual conditions)
    cert = None
    if rank == 0 and ncomp == 1:
        from paper_2402_16712_b200.certify import certify_line
        c = certify_line(X, lines[0])
        cert = {"columns": int(np.isfinite(c.slack).sum()), "refuted": len(c.refuted), "lam": float(lines[0].lam)}
    e2e_val = solves_step * args.steps / (max_over_ranks(float(np.sum(e2e_ms))) / 1e3)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sps, per_fit, sample, kind = cpu_reference(X, lams, budget_s=args.cpu_budget)
        cpu = {"value": sps, "unit": "solves/s", "cores": os.cpu_count(), "kind": kind, "cpu_model": _cpu_model(),
               "sample": sample, "seconds_per_fit_extrapolated": per_fit}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator, seed 0)",
            "config": _config_dict(args, X, lams, world),
            "result": {"pivot": [l.preserved for l in lines][:4], "objective": [l.objective for l in lines][:4],
                       "nonzeros": [int(np.count_nonzero(l.v)) for l in lines][:4], "certificate": cert},
            "e2e": {"value": e2e_val, "unit": "solves/s", "ms_per_step": float(np.mean(e2e_ms)),
                    "h2d_bytes_per_step": int(X.nbytes),
                    "d2h_bytes_per_step": int(8 * m * len(lams) * ncomp + 8 * npiv * len(lams) * ncomp)},
            "gpu_launches": launches,
            "roofline": {"bound": "smem_atomic", "kernel": "k_bound (one FP32 bounding pass over every "
                                                          "(pivot, target, row) element)",
                         "achieved": kb_rate / 1e9, "peak": atoms_peak / 1e9,
                         "unit": "G shared-memory atomics/s (one per element)",
                         "frac": kb_rate / atoms_peak,
                         "traffic": _ncu_traffic(args.config, world),
                         "kernel_ms": kb_ms, "elements_per_launch": kb_elems,
                         "share_of_step": kb_ms * (1 if multi else len(lams)) * ncomp / (ms_total / args.steps),
                         "penalties_per_launch": len(ulams) if multi else 1,
                         "peak_source": "measured: l1b_atoms_probe (conflict-free red.shared.add.u32, "
                                        "8 in flight per thread)",
                         "fp32_view": {"ops_per_element": 5, "achieved_TOPs": 5 * kb_rate / 1e12,
                                       "peak_TOPs": _fp32_peak(dev) / 1e12},
                         "smem_wavefront_view": {
                             "note": "shared-memory pipe requests the design issues per element: per warp and row, "
                                     "8 problems x 32 lanes = 256 elements cost 8 histogram atomics + 1 tile load "
                                     "(2 wavefronts) + 3 broadcast record loads = 13 instructions; peak = one per "
                                     "SM-clock (the atomic probe / 32). ncu: profiles/r02/.",
                             "requests_per_element": 13.0 / 256.0,
                             "achieved_G_per_s": kb_rate * 13.0 / 256.0 / 1e9,
                             "peak_G_per_s": atoms_peak / 32.0 / 1e9,
                             "frac": kb_rate * 13.0 / 256.0 / (atoms_peak / 32.0)},
                         "step_view": {
                             "note": "whole pruned step against the exact algorithm's FP64 floor (SURVEY.md 8d: "
                                     "11 FP64 ops per ratio element, E = n*m*(m-1) per fit); > 1 means the step "
                                     "beats that floor by skipping provably losing pivots",
                             "elements_per_step": elems * ncomp,
                             "achieved_elements_per_s": elems * ncomp / (ms_total / args.steps / 1e3),
                             "exact_fp64_floor_elements_per_s": fp64_ops / 11.0,
                             "frac": elems * ncomp / (ms_total / args.steps / 1e3) / (fp64_ops / 11.0)},
                         "exact_fit_view": {
                             "kernel": "k_select+k_resolve+k_straggle (exact fit of every pivot)",
                             "achieved": achieved / 1e12, "peak": fp64_ops / 1e12,
                             "unit": "TOP/s (FP64 pipe ops)", "frac": achieved / fp64_ops,
                             "kernel_ms": sel_ms, "ops_per_element": 11, "elements_per_launch": elems,
                             "stragglers_per_launch": strag,
                             "peak_source": "measured: l1b_dfma_probe (DFMA/s, 1 op per DFMA)"}},
            "pruning": {"note": "fit_line needs only the argmin pivot: every (pivot, target) problem is bounded by "
                                "one FP32 pass (k_bound<1>), pivots whose lower bound exceeds the best upper "
                                "bound are provably not the winner; the survivors get three refining passes "
                                "(k_bound<3>) and the few left are fitted exactly by the warp-per-problem solver "
                                "started on the ranges the bounds left. Results are identical to fitting every "
                                "pivot (tests/test_gpu_parity.py::test_pruned_fit_equals_full_fit).",
                        "pivots_per_rank": npiv, "exactly_fitted_per_lambda": cand[:8],
                        "bound_pass_ms": bnd_ms,
                        "bound_pass_fp64_equiv_frac": 11.0 * npiv * (m - 1) * n / (bnd_ms / 1e3) / fp64_ops},
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _fp32_peak(dev) -> float:
    """FP32 pipe instructions/s: SMs x 128 lanes x the SM clock (nominal max)."""
    import torch
    props = torch.cuda.get_device_properties(dev)
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(dev.index or 0)
        mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
    except Exception:  # noqa: BLE001
        mhz = 1965
    return props.multi_processor_count * 128 * mhz * 1e6


def _ncu_traffic(config: str, world: int):
    """dram__bytes_read.sum + dram__bytes_write.sum of one k_bound launch
    from the committed ncu --set full capture (profiles/r02), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t.get(config) if world == 1 else None
    except Exception:  # noqa: BLE001
        return None


def _peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)["hbm_gbs"]
    except Exception:  # noqa: BLE001
        return 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of CPU baseline sampling")
    ap.add_argument("--ref-budget", type=float, default=60.0, help="seconds for the whole reference arm")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--port", action="store_true", help="reference arm: the oracle C port even where the "
                                                        "reference package is installed")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
