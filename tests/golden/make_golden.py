"""Generate the golden parity fixtures from the REFERENCE implementation.

Run in the build container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array written here comes out of the reference package ``l1line``
(``/root/reference/pkg/src/l1line``) through its public API: ``fit_line``
(fit.py:88-102), ``fit_for_pivot`` (fit.py:75-85), ``fit_subspace``
(subspace.py:54-76), ``gen_line_data`` / ``gen_outlier_data``
(datagen.py:36-82).  The GPU box has no /root/reference, so the tests read
these committed .npz files instead.  Inputs mirror the reference's own test
recipes: ``random_instance`` (pkg/tests/conftest.py:22-33), grid-quantised
copies, exact ties, exact zeros and -0.0 entries.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import l1line  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def _ref_pivots(X, lams):
    """Per-pivot reference results for every lambda: V [m][L][m], E/P/O [m][L]."""
    d = l1line.DataMatrix(X)
    m = X.shape[1]
    V = np.zeros((m, len(lams), m))
    E = np.zeros((m, len(lams)))
    P = np.zeros((m, len(lams)))
    O = np.zeros((m, len(lams)))
    for p in range(m):
        for k, lam in enumerate(lams):
            line = l1line.fit_for_pivot(d, p, lam)
            V[p, k], E[p, k], P[p, k], O[p, k] = line.v, line.error, line.penalty_norm, line.objective
    return V, E, P, O


def _ref_lines(X, lams):
    d = l1line.DataMatrix(X)
    out = {"piv": [], "v": [], "err": [], "pen": [], "obj": []}
    for lam in lams:
        line = l1line.fit_line(d, lam, threads=1)
        out["piv"].append(line.preserved)
        out["v"].append(line.v)
        out["err"].append(line.error)
        out["pen"].append(line.penalty_norm)
        out["obj"].append(line.objective)
    return {k: np.asarray(v) for k, v in out.items()}


def random_small():
    """Ragged set of small instances in the style of conftest.random_instance."""
    rng = np.random.default_rng(20240226)
    mats, lams_all, shapes = [], [], []
    pV, pE, pP, pO, lpiv, lv, lerr, lpen, lobj = [], [], [], [], [], [], [], [], []
    for t in range(160):
        n = int(rng.integers(1, 33))
        m = int(rng.integers(2, 9))
        X = rng.uniform(-10.0, 10.0, size=(n, m))
        kind = t % 6
        if kind == 1:
            X[rng.random(X.shape) < 0.25] = 0.0          # exact zeros (conftest zeros=True)
        elif kind == 2:
            X = np.round(X)                               # many exact ratio ties
        elif kind == 3:
            X[rng.random(X.shape) < 0.25] = -0.0          # signed zeros
            X[rng.random(X.shape) < 0.1] = 0.0
        elif kind == 4:
            X = np.round(X * 2**4) / 2**4                 # grid-quantised
            X[:, int(rng.integers(m))] = 0.0              # a zero column -> degenerate pivot
        elif kind == 5:
            X[:, -1] = X[:, 0]                            # identical columns -> objective ties
        tot = float(np.abs(X).sum())
        lams = [0.0, float(rng.uniform(0, 3)), float(rng.uniform(0, tot / 2 + 1)),
                float(rng.uniform(0, tot + 1))]
        V, E, P, O = _ref_pivots(X, lams)
        L = _ref_lines(X, lams)
        mats.append(X.ravel())
        shapes.append((n, m))
        lams_all.append(lams)
        pV.append(V.ravel()); pE.append(E.ravel()); pP.append(P.ravel()); pO.append(O.ravel())
        lpiv.append(L["piv"]); lv.append(L["v"].ravel()); lerr.append(L["err"])
        lpen.append(L["pen"]); lobj.append(L["obj"])
    np.savez_compressed(
        os.path.join(OUT, "random_small.npz"),
        shapes=np.asarray(shapes, dtype=np.int64), X=np.concatenate(mats),
        lams=np.asarray(lams_all), pV=np.concatenate(pV), pE=np.concatenate(pE),
        pP=np.concatenate(pP), pO=np.concatenate(pO), lpiv=np.asarray(lpiv, dtype=np.int64),
        lv=np.concatenate(lv), lerr=np.asarray(lerr), lpen=np.asarray(lpen), lobj=np.asarray(lobj))


def c1_and_grid():
    """Config C1 (BASELINE.json configs[0]) raw and grid-quantised, plus a medium grid case."""
    d, vtrue = l1line.gen_outlier_data(50, 200, 20, seed=0)
    X = d.values.copy()
    Xq = np.round(X * 2**20) / 2**20
    lams = [0.1, 0.0, 25.0, 500.0, 1500.0]
    out = {"X": X, "Xq": Xq, "vtrue": vtrue, "lams": np.asarray(lams)}
    for tag, M in (("raw", X), ("grid", Xq)):
        V, E, P, O = _ref_pivots(M, lams)
        L = _ref_lines(M, lams)
        out.update({f"{tag}_pV": V, f"{tag}_pE": E, f"{tag}_pP": P, f"{tag}_pO": O})
        out.update({f"{tag}_{k}": v for k, v in L.items()})
    np.savez_compressed(os.path.join(OUT, "c1.npz"), **out)

    d2, _ = l1line.gen_line_data(40, 300, seed=7, noise_scale=1.0)
    G = np.round(d2.values * 2**20) / 2**20
    lams2 = [0.0, 1.0, 50.0, 400.0]
    V, E, P, O = _ref_pivots(G, lams2)
    L = _ref_lines(G, lams2)
    np.savez_compressed(os.path.join(OUT, "grid_medium.npz"), X=G, lams=np.asarray(lams2),
                        pV=V, pE=E, pP=P, pO=O, **{f"l_{k}": v for k, v in L.items()})


def subspace_cases():
    toy = np.array([[4.0, -2.0, 3.0, -6.0], [-3.0, 4.0, 2.0, -1.0], [2.0, 3.0, -3.0, -2.0],
                    [-3.0, 4.0, 2.0, 3.0], [5.0, 3.0, 2.0, -1.0]])
    rng = np.random.default_rng(5)
    R = rng.uniform(-10, 10, size=(40, 6))
    G = np.round(l1line.gen_line_data(8, 120, seed=3, noise_scale=0.5)[0].values * 2**20) / 2**20
    out = {}
    for tag, X, lam, k in (("toy", toy, 1.0, 3), ("rand", R, 2.0, 3), ("grid", G, 1.0, 3)):
        fit = l1line.fit_subspace(l1line.DataMatrix(X), lam, k, threads=1)
        out[f"{tag}_X"] = X
        out[f"{tag}_lam"] = lam
        out[f"{tag}_k"] = k
        out[f"{tag}_degenerate"] = fit.degenerate
        out[f"{tag}_piv"] = np.asarray([c.preserved for c in fit.components])
        out[f"{tag}_v"] = np.asarray([c.v for c in fit.components])
        out[f"{tag}_obj"] = np.asarray([c.objective for c in fit.components])
        out[f"{tag}_err"] = np.asarray([c.error for c in fit.components])
    X1 = np.outer([1.0, 2.0, -1.0], [3.0, 0.0, 4.0])                   # rank one: stops early
    fit = l1line.fit_subspace(l1line.DataMatrix(X1), 0.0, 2)
    out["rank1_X"] = X1
    out["rank1_n"] = len(fit)
    out["rank1_degenerate"] = fit.degenerate
    np.savez_compressed(os.path.join(OUT, "subspace.npz"), **out)


def datagen_cases():
    out = {}
    for (m, n, seed, ns) in ((7, 11, 0, 1.0), (5, 9, 3, 0.0), (12, 30, 42, 2.5)):
        d, v = l1line.gen_line_data(m, n, seed=seed, noise_scale=ns)
        out[f"line_{m}_{n}_{seed}_X"] = d.values
        out[f"line_{m}_{n}_{seed}_v"] = v
    for (m, n, k, seed) in ((6, 13, 3, 1), (50, 200, 20, 0)):
        d, v = l1line.gen_outlier_data(m, n, k, seed=seed)
        out[f"outl_{m}_{n}_{k}_{seed}_X"] = d.values
        out[f"outl_{m}_{n}_{k}_{seed}_v"] = v
    d, v = l1line.gen_line_data(2000, 2000, seed=0, noise_scale=1.0)
    # C2 checksum (the full matrix is 32 MB): first/last rows and a strided sample.
    out["c2_head"] = d.values[:2].copy()
    out["c2_tail"] = d.values[-2:].copy()
    out["c2_stride"] = d.values[::97, ::89].copy()
    out["c2_v"] = v
    np.savez_compressed(os.path.join(OUT, "datagen.npz"), **out)


def _flat_breakpoints(pb):
    """pivot_breakpoints (path.py:76-102) as arrays: rows (target, weight, value) in
    the dict's target order, each target's entries in tuple order; lambda_max per target."""
    rows, lmax = [], []
    for target, entries in pb.entries.items():
        for bp, val in entries:
            rows.append((float(target), bp, val))
        lmax.append((float(target), pb.lambda_max[target]))
    return np.asarray(rows, dtype=np.float64).reshape(-1, 3), np.asarray(lmax, dtype=np.float64).reshape(-1, 2)


def breakpoint_cases():
    """Algorithm 2 (path.py:76-154): per-pivot breakpoint maps and the merged grid."""
    toy = np.array([[4.0, -2.0, 3.0, -6.0], [-3.0, 4.0, 2.0, -1.0], [2.0, 3.0, -3.0, -2.0],
                    [-3.0, 4.0, 2.0, 3.0], [5.0, 3.0, 2.0, -1.0]])
    rng = np.random.default_rng(77)
    cases = [("toy", toy)]
    for t in range(12):
        n, m = int(rng.integers(1, 40)), int(rng.integers(2, 8))
        X = rng.uniform(-10, 10, size=(n, m))
        if t % 4 == 1:
            X[rng.random(X.shape) < 0.3] = 0.0
        elif t % 4 == 2:
            X = np.round(X)
            X[rng.random(X.shape) < 0.2] = -0.0
        elif t % 4 == 3:
            X[:, int(rng.integers(m))] = 0.0
        cases.append((f"rand{t}", X))
    cases.append(("line", l1line.gen_line_data(12, 300, seed=5, noise_scale=1.0)[0].values))
    cases.append(("tall", np.round(l1line.gen_line_data(6, 3000, seed=9, noise_scale=0.5)[0].values * 2**10) / 2**10))
    out = {"names": np.asarray([c[0] for c in cases])}
    for name, X in cases:
        d = l1line.DataMatrix(X)
        out[f"{name}_X"] = X
        lambdas, sols = l1line.major_breakpoints(d, threads=1)
        out[f"{name}_grid"] = lambdas
        out[f"{name}_degenerate"] = np.asarray(sols.degenerate, dtype=np.int64)
        for p in range(X.shape[1]):
            if p in sols.pivots:
                rows, lmax = _flat_breakpoints(sols.pivots[p])
                out[f"{name}_p{p}_entries"] = rows
                out[f"{name}_p{p}_lmax"] = lmax
    np.savez_compressed(os.path.join(OUT, "breakpoints.npz"), **out)


def path_cases():
    """Algorithm 3 (path.py:166-283): the reference's solution_path on the
    breakpoint cases, segment by segment."""
    g = np.load(os.path.join(OUT, "breakpoints.npz"))
    out = {}
    for name in g["names"]:
        X = g[f"{name}_X"]
        path = l1line.solution_path(l1line.DataMatrix(X), threads=1)
        segs = path.segments
        out[f"{name}_lo"] = np.asarray([sg.lambda_lo for sg in segs])
        out[f"{name}_hi"] = np.asarray([sg.lambda_hi for sg in segs])
        out[f"{name}_zlo"] = np.asarray([sg.z_lo for sg in segs])
        out[f"{name}_zhi"] = np.asarray([sg.z_hi for sg in segs])
        out[f"{name}_piv"] = np.asarray([sg.line.preserved for sg in segs], dtype=np.int64)
        out[f"{name}_v"] = np.asarray([sg.line.v for sg in segs])
        out[f"{name}_err"] = np.asarray([sg.line.error for sg in segs])
        out[f"{name}_pen"] = np.asarray([sg.line.penalty_norm for sg in segs])
        out[f"{name}_obj"] = np.asarray([sg.line.objective for sg in segs])
    np.savez_compressed(os.path.join(OUT, "paths.npz"), names=g["names"], **out)


CSV_CASES = {
    "plain": "1.5,2,3\n4,5e-3,-6\n",
    "header": "a, b ,c\n1,2,3\n4,5,6\n",
    "crlf_blank": "1,2\r\n\r\n , \r\n3,4\r\n\r\n",
    "plus_space": " +1.25 ,\t-2.5\n3e2 , .5\n",
    "quoted": '"1.5",2\n3,"4e1"\n',
    "underscore": "1_000,2\n3,4\n",
    "ragged": "1,2,3\n4,5\n",
    "nonnumeric": "1,2\n3,abc\n",
    "empty_cell": "1,,3\n4,5,6\n",
    "nan": "1,2\nnan,4\n",
    "inf": "1,2\n3,-inf\n",
    "overflow": "1,2\n3,1e400\n",
    "underflow": "1e-400,2\n3,4.9e-324\n",
    "no_data": "\n\n",
    "header_only": "x,y\n",
    "header_mismatch": "x,y,z\n1,2\n",
    "one_col": "1\n2\n",
    "exp_forms": "1E5,2.E-3\n-0,0.0\n",
    "long_digits": "0.1000000000000000055511151231257827,3.141592653589793238462643383279\n2.718281828459045235360287,1\n",
    "unicode": "1,\u0663\n2,3\n",
    "plus_minus": "1,+-1\n2,3\n",
    "plus_plus": "1,2\n++3,4\n",
}


def tableau_cases():
    """pivot_tableau (ratios.py:109-135) of every pivot and dual_certificate
    (oracle.py:141-174) of every column's optimum -- and of two refuted values --
    at four penalties, on the toy, ragged random instances with exact zeros,
    -0.0 and ties, and a 300x12 grid-quantised line."""
    from l1line.fit import solve_column
    from l1line.oracle import OptimalityRefuted, dual_certificate
    from l1line.ratios import EmptyPivotError, build_column, pivot_tableau
    rng = np.random.default_rng(7)
    mats = {"toy": np.array([[4.0, -2.0, 3.0, -6.0], [-3.0, 4.0, 2.0, -1.0], [2.0, 3.0, -3.0, -2.0],
                             [-3.0, 4.0, 2.0, 3.0], [5.0, 3.0, 2.0, -1.0]])}
    for t in range(6):
        n, m = int(rng.integers(3, 40)), int(rng.integers(2, 7))
        X = np.round(rng.uniform(-5, 5, size=(n, m)) * 2) / 2
        X[rng.random(X.shape) < 0.2] = 0.0
        X[rng.random(X.shape) < 0.1] = -0.0
        if t == 5:
            X[:, 0] = 0.0
        mats[f"rand{t}"] = X
    d, _ = l1line.gen_line_data(12, 300, seed=4, noise_scale=1.0)
    mats["grid300"] = np.round(d.values * 2**10) / 2**10
    out = {"names": np.array(sorted(mats))}
    for name, X in mats.items():
        dm = l1line.DataMatrix(X)
        out[f"{name}_X"] = X
        n, m = X.shape
        T = float(np.abs(X).sum(axis=0).max())
        lams = [0.0, 0.5, 0.2 * T, 2.0 * T]
        out[f"{name}_lams"] = np.array(lams)
        cert = []  # rows: pivot, target, lam index, case (0 optimum, 1/2 perturbed), ok, gamma, pi...
        for p in range(m):
            try:
                tab = pivot_tableau(dm, p)
            except EmptyPivotError:
                out[f"{name}_p{p}_empty"] = np.array(1)
                continue
            for key in ("ratios", "weights", "source_rows", "prefix", "prefix_prev", "totals", "targets"):
                out[f"{name}_p{p}_{key}"] = getattr(tab, key)
            for j in range(m):
                if j == p or (name == "grid300" and p > 1):  # certificates of two pivots there (size)
                    continue
                col = build_column(dm, p, j)
                for li, lam in enumerate(lams):
                    v = solve_column(col, lam)
                    for case, val in enumerate((v, v + 0.25, float(col.ratios[len(col) // 2]))):
                        try:
                            c = dual_certificate(col, val, lam)
                            cert.append([p, j, li, case, val, 1, c.gamma] + list(c.pi))
                        except OptimalityRefuted:
                            cert.append([p, j, li, case, val, 0, 0.0] + [0.0] * len(col))
        w = max(len(r) for r in cert) if cert else 7
        out[f"{name}_cert"] = np.array([r + [0.0] * (w - len(r)) for r in cert]) if cert else np.zeros((0, 7))
    np.savez_compressed(os.path.join(OUT, "tableau.npz"), **out)


def csv_cases():
    """io.read_matrix / write_matrix (io.py:46-98) on edge-case files: the
    files under csv/ and the reference's outcome for each (values as hex, or
    the exception with its row and column)."""
    import json

    from l1line import io as rio
    out = os.path.join(OUT, "csv")
    os.makedirs(out, exist_ok=True)
    exp = {}
    for name, text in CSV_CASES.items():
        p = os.path.join(out, name + ".csv")
        with open(p, "w", newline="", encoding="utf-8") as f:
            f.write(text)
        for hh in (False, True):
            key = f"{name}|{int(hh)}"
            try:
                d = rio.read_matrix(p, has_header=hh)
                exp[key] = {"ok": True, "shape": list(d.values.shape),
                            "hex": [float(x).hex() for x in d.values.ravel()],
                            "names": list(d.column_names) if d.column_names else None}
            except rio.CsvParseError as e:
                exp[key] = {"ok": False, "type": "CsvParseError", "msg": str(e), "row": e.row, "col": e.column}
            except ValueError as e:
                exp[key] = {"ok": False, "type": "ValueError", "msg": str(e)}
    d, _ = l1line.gen_line_data(7, 5, seed=3, noise_scale=1.0)
    rio.write_matrix(d, os.path.join(out, "written.csv"), header=True)
    toy = l1line.DataMatrix(np.array([[4.0, -2.0, 3.0, -6.0], [-3.0, 4.0, 2.0, -1.0], [2.0, 3.0, -3.0, -2.0],
                                      [-3.0, 4.0, 2.0, 3.0], [5.0, 3.0, 2.0, -1.0]]))
    rio.write_path(l1line.solution_path(toy), os.path.join(out, "toy_path.json"))
    rio.write_sweep([{"lam": 0.0, "preserved": 3, "error": 34.5, "penalty_norm": 2.5, "objective": 34.5,
                      "l0_fraction": 0.25, "discordance": None},
                     {"lam": 1.5, "preserved": 0, "error": 40.1, "penalty_norm": 1.2, "objective": 41.9,
                      "l0_fraction": 0.5, "discordance": 0.125}], os.path.join(out, "sweep.csv"))
    np.save(os.path.join(out, "written_X.npy"), d.values)
    with open(os.path.join(out, "expected.json"), "w") as f:
        json.dump(exp, f, indent=0, sort_keys=True)


if __name__ == "__main__":
    want = set(sys.argv[1:])
    for f in (random_small, c1_and_grid, subspace_cases, datagen_cases, breakpoint_cases, path_cases, csv_cases,
              tableau_cases):
        if not want or f.__name__ in want:
            f()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
