/*
 * l1oracle.c -- CPU restatement of the l1line hot path (Algorithm 1).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path in paper_2402_16712_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never calls it.
 *
 * It restates, operation by operation, what the reference package computes
 * (paths relative to /root/reference/pkg/src/l1line):
 *
 *   ratios.py:109-135  pivot_tableau   rows with x_ip != 0, R = X[rows,t]/x_p
 *                                      (IEEE division), stable argsort per
 *                                      column (ties -> source row; -0.0 == +0.0),
 *                                      sequential f64 cumsum of |x_ip|.
 *   ratios.py:40-67    build_column    single-column twin of the above.
 *   fit.py:27-48,51-63 solve_column / _snap_all
 *                                      lower = T - 2P[k], upper = T - 2P[k-1]
 *                                      (upper_0 = T - 2*0.0), probe = +lam if
 *                                      r >= 0.0 else -lam, first k with
 *                                      lower < probe <= upper, else +0.0.
 *   fit.py:66-72       degenerate_line v = 0, error = sum|x|.
 *   fit.py:75-85       fit_for_pivot   v[p] = 1.0, v[targets] = snap.
 *   fit.py:88-102      fit_line        strict '<' argmin in pivot order.
 *   core.py:79-93      residual_error  np.abs(X - np.outer(X[:,p], v)).sum():
 *                                      elementwise fl(x_ij - fl(x_ip*v_j)),
 *                                      then NumPy's pairwise summation over the
 *                                      row-major flattened n*m temporary.
 *   core.py:126-133    FittedLine.build  pen = np.abs(v).sum() (pairwise over m),
 *                                      objective = err + lam*pen.
 *   parallel.py:36-43  map_indices     pivots on a thread pool, results in
 *                                      index order (OpenMP here).
 *
 * NumPy's float64 pairwise sum (numpy/_core/src/umath/loops_utils.h.src,
 * pairwise_sum_DOUBLE; NumPy 2.3.5 here, pinned only as numpy>=1.24 by
 * pkg/pyproject.toml:11-14): n < 8 -> sequential from 0.0; n <= 128 -> eight
 * strided accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus a
 * sequential tail; else split at n2 = n/2 - (n/2 % 8) and recurse.  A full
 * reduction of a C-contiguous 2-D array applies it to the flattened array
 * (checked against np.sum in tests/test_oracle.py).
 *
 * Compile with -ffp-contract=off: the reference never fuses multiply-adds.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define L1O_OK 0
#define L1O_EINVAL -1
#define L1O_ENOMEM -3
#define L1O_EMPTY_PIVOT 1 /* EmptyPivotError (ratios.py:27-28), internal */

/* ---------------------------------------------------------------- sums -- */

/* Pairwise sum of f(0..n-1) in NumPy's order; f is evaluated lazily so the
 * n*m residual temporary of core.py:93 never has to be materialised. */
typedef double (*l1o_elem_fn)(const void* ctx, int64_t idx);

static double pairwise_lazy(l1o_elem_fn f, const void* ctx, int64_t off, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; i++) res += f(ctx, off + i);
    return res;
  } else if (n <= 128) {
    double r[8];
    int64_t i;
    for (int k = 0; k < 8; k++) r[k] = f(ctx, off + k);
    for (i = 8; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; k++) r[k] += f(ctx, off + i + k);
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += f(ctx, off + i);
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_lazy(f, ctx, off, n2) + pairwise_lazy(f, ctx, off + n2, n - n2);
  }
}

static double elem_array(const void* ctx, int64_t idx) { return ((const double*)ctx)[idx]; }
static double elem_abs_array(const void* ctx, int64_t idx) { return fabs(((const double*)ctx)[idx]); }

double l1o_pairwise_sum(const double* a, int64_t n) {
  return pairwise_lazy(elem_array, a, 0, n);
}

typedef struct {
  const double* X;
  int64_t m;
  int64_t p;
  const double* v;
} resid_ctx;

static double elem_resid(const void* c, int64_t idx) {
  const resid_ctx* r = (const resid_ctx*)c;
  int64_t i = idx / r->m, j = idx - i * r->m;
  double prod = r->X[i * r->m + r->p] * r->v[j]; /* np.outer: x_ip * v_j */
  double d = r->X[i * r->m + j] - prod;          /* X - outer            */
  return fabs(d);                                /* np.abs               */
}

/* core.py:79-93 */
double l1o_residual_error(const double* X, int64_t n, int64_t m, const double* v, int64_t p) {
  resid_ctx c = {X, m, p, v};
  return pairwise_lazy(elem_resid, &c, 0, n * m);
}

/* core.py:131  float(np.abs(v).sum()) */
double l1o_abs_sum(const double* v, int64_t m) { return pairwise_lazy(elem_abs_array, v, 0, m); }

/* ---------------------------------------------------------- tableau -- */

typedef struct {
  double r;
  int64_t row;
} rr_t;

/* np.argsort(kind="stable") on float64: ascending, equal keys keep source
 * order.  -0.0 and +0.0 compare equal.  Inputs are finite so ratios are
 * finite or +-inf, never NaN. */
static int cmp_rr(const void* a, const void* b) {
  const rr_t* x = (const rr_t*)a;
  const rr_t* y = (const rr_t*)b;
  if (x->r < y->r) return -1;
  if (x->r > y->r) return 1;
  return (x->row > y->row) - (x->row < y->row);
}

/* ratios.py:40-67 build_column.  Outputs (len <= n): sorted ratios, weights,
 * source rows, inclusive prefix.  Returns L1O_EMPTY_PIVOT when column p has no
 * nonzero entry. */
int l1o_build_column(const double* X, int64_t n, int64_t m, int64_t p, int64_t j,
                     double* ratios, double* weights, int64_t* rows, double* prefix,
                     int64_t* len) {
  if (p < 0 || p >= m || j < 0 || j >= m || p == j) return L1O_EINVAL;
  rr_t* buf = (rr_t*)malloc(sizeof(rr_t) * (size_t)(n > 0 ? n : 1));
  if (!buf) return L1O_ENOMEM;
  int64_t c = 0;
  for (int64_t i = 0; i < n; i++) {
    double b = X[i * m + p];
    if (b != 0.0) {
      buf[c].r = X[i * m + j] / b;
      buf[c].row = i;
      c++;
    }
  }
  if (c == 0) {
    free(buf);
    *len = 0;
    return L1O_EMPTY_PIVOT;
  }
  qsort(buf, (size_t)c, sizeof(rr_t), cmp_rr);
  double acc = 0.0;
  for (int64_t k = 0; k < c; k++) {
    ratios[k] = buf[k].r;
    weights[k] = fabs(X[buf[k].row * m + p]);
    rows[k] = buf[k].row;
    acc = (k == 0) ? weights[k] : acc + weights[k]; /* np.cumsum, sequential */
    prefix[k] = acc;
  }
  *len = c;
  free(buf);
  return L1O_OK;
}

/* fit.py:27-48 solve_column / fit.py:51-63 _snap_all on one column. */
double l1o_solve_column(const double* ratios, const double* prefix, int64_t len, double lam) {
  double T = prefix[len - 1];
  for (int64_t k = 0; k < len; k++) {
    double lower = T - 2.0 * prefix[k];
    double upper = T - 2.0 * (k > 0 ? prefix[k - 1] : 0.0);
    double probe = (ratios[k] >= 0.0) ? lam : -lam;
    if (probe > lower && probe <= upper) return ratios[k];
  }
  return 0.0;
}

/* ------------------------------------------------------------ pivots -- */

/* fit.py:75-85 (+ fit.py:66-72 degenerate fallback) for nlam penalty
 * weights at once: the tableau (ratios.py:109-135) takes no lambda, so it is
 * built once and snapped per lambda, which is bit-identical to nlam separate
 * fit_for_pivot calls.  V is [nlam][m]; err/pen/obj are [nlam]. */
int l1o_fit_pivot_multi(const double* X, int64_t n, int64_t m, int64_t p, const double* lams,
                        int32_t nlam, double* V, double* err, double* pen, double* obj) {
  if (p < 0 || p >= m || n < 1 || m < 2 || nlam < 1) return L1O_EINVAL;
  for (int32_t l = 0; l < nlam; l++)
    if (!(lams[l] >= 0.0)) return L1O_EINVAL;
  int64_t nz = 0;
  for (int64_t i = 0; i < n; i++) nz += (X[i * m + p] != 0.0);
  if (nz == 0) { /* degenerate_line: v = 0, FittedLine.build */
    double* z = (double*)calloc((size_t)m, sizeof(double));
    if (!z) return L1O_ENOMEM;
    double e = l1o_residual_error(X, n, m, z, p);
    for (int32_t l = 0; l < nlam; l++) {
      memset(V + (size_t)l * m, 0, sizeof(double) * (size_t)m);
      err[l] = e;
      pen[l] = 0.0;
      obj[l] = e + lams[l] * 0.0;
    }
    free(z);
    return L1O_OK;
  }
  double* ratios = (double*)malloc(sizeof(double) * (size_t)n);
  double* weights = (double*)malloc(sizeof(double) * (size_t)n);
  double* prefix = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  if (!ratios || !weights || !prefix || !rows) {
    free(ratios); free(weights); free(prefix); free(rows);
    return L1O_ENOMEM;
  }
  for (int32_t l = 0; l < nlam; l++) {
    memset(V + (size_t)l * m, 0, sizeof(double) * (size_t)m);
    V[(size_t)l * m + p] = 1.0;
  }
  for (int64_t j = 0; j < m; j++) {
    if (j == p) continue;
    int64_t len = 0;
    l1o_build_column(X, n, m, p, j, ratios, weights, rows, prefix, &len);
    for (int32_t l = 0; l < nlam; l++)
      V[(size_t)l * m + j] = l1o_solve_column(ratios, prefix, len, lams[l]);
  }
  for (int32_t l = 0; l < nlam; l++) {
    const double* v = V + (size_t)l * m;
    err[l] = l1o_residual_error(X, n, m, v, p);
    pen[l] = l1o_abs_sum(v, m);
    obj[l] = err[l] + lams[l] * pen[l];
  }
  free(ratios); free(weights); free(prefix); free(rows);
  return L1O_OK;
}

int l1o_fit_for_pivot(const double* X, int64_t n, int64_t m, int64_t p, double lam, double* v,
                      double* err, double* pen, double* obj) {
  return l1o_fit_pivot_multi(X, n, m, p, &lam, 1, v, err, pen, obj);
}

/* Per-pivot results for pivots in [p_begin, p_end) (parallel.py:36-43 over
 * pivots).  V is [npiv][nlam][m] when non-NULL; ERR/PEN/OBJ are [npiv][nlam]. */
int l1o_fit_pivots(const double* X, int64_t n, int64_t m, const double* lams, int32_t nlam,
                   int64_t p_begin, int64_t p_end, int32_t threads, double* V, double* ERR,
                   double* PEN, double* OBJ) {
  if (p_begin < 0 || p_end > m || p_begin >= p_end || nlam < 1) return L1O_EINVAL;
  int status = L1O_OK;
#ifdef _OPENMP
  if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
#endif
  for (int64_t p = p_begin; p < p_end; p++) {
    int64_t k = p - p_begin;
    double* vbuf = V ? V + (size_t)k * nlam * m : (double*)malloc(sizeof(double) * (size_t)nlam * m);
    int rc = vbuf ? l1o_fit_pivot_multi(X, n, m, p, lams, nlam, vbuf, ERR + (size_t)k * nlam,
                                        PEN + (size_t)k * nlam, OBJ + (size_t)k * nlam)
                  : L1O_ENOMEM;
    if (!V) free(vbuf);
    if (rc != L1O_OK) {
#ifdef _OPENMP
#pragma omp critical
#endif
      status = rc;
    }
  }
  return status;
}

/* fit.py:88-102 for nlam weights: per lambda the strict '<' argmin over pivot
 * objectives in ascending pivot order.  Outputs [nlam] / [nlam][m]. */
int l1o_fit_line_multi(const double* X, int64_t n, int64_t m, const double* lams, int32_t nlam,
                       int32_t threads, double* v_out, int64_t* piv_out, double* err_out,
                       double* pen_out, double* obj_out) {
  if (n < 1 || m < 2 || nlam < 1) return L1O_EINVAL;
  size_t per = (size_t)m * nlam;
  double* V = (double*)malloc(sizeof(double) * per * (size_t)m);
  double* E = (double*)malloc(sizeof(double) * per);
  double* P = (double*)malloc(sizeof(double) * per);
  double* O = (double*)malloc(sizeof(double) * per);
  if (!V || !E || !P || !O) {
    free(V); free(E); free(P); free(O);
    return L1O_ENOMEM;
  }
  int rc = l1o_fit_pivots(X, n, m, lams, nlam, 0, m, threads, V, E, P, O);
  if (rc == L1O_OK) {
    for (int32_t l = 0; l < nlam; l++) {
      int64_t best = 0;
      for (int64_t p = 1; p < m; p++)
        if (O[(size_t)p * nlam + l] < O[(size_t)best * nlam + l]) best = p;
      piv_out[l] = best;
      err_out[l] = E[(size_t)best * nlam + l];
      pen_out[l] = P[(size_t)best * nlam + l];
      obj_out[l] = O[(size_t)best * nlam + l];
      memcpy(v_out + (size_t)l * m, V + ((size_t)best * nlam + l) * m, sizeof(double) * (size_t)m);
    }
  }
  free(V); free(E); free(P); free(O);
  return rc;
}

int l1o_fit_line(const double* X, int64_t n, int64_t m, double lam, int32_t threads, double* v,
                 int64_t* piv, double* err, double* pen, double* obj) {
  return l1o_fit_line_multi(X, n, m, &lam, 1, threads, v, piv, err, pen, obj);
}

int l1o_version(void) { return 1; }
