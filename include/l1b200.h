/*
 * l1b200.h -- C ABI of the B200-native sparse l1 line-fit hot path.
 *
 * The reference (l1line, /root/reference/pkg/src/l1line) is pure Python on
 * NumPy and has no FFI of its own; each entry point below replaces the
 * Python function named beside it, with the same argument meaning.  The
 * Python mirror of the reference API (paper_2402_16712_b200/api.py) binds
 * these through ctypes; INTEGRATION.md shows the binding a maintainer would
 * add to l1line itself.
 *
 * Conventions
 *   - Every pointer named d_* is DEVICE memory; h_* is host memory.
 *   - X is the data matrix exactly as DataMatrix.values holds it
 *     (core.py:45-68): row-major, n rows x m columns, float64, ld = m.
 *   - All work is enqueued on `stream` (a cudaStream_t passed as void*);
 *     no call synchronises unless its comment says so.  The library owns no
 *     device memory: callers pass a workspace of l1b_workspace_bytes().
 *   - Status codes: 0 = OK, negative = error (see l1b_status_string).  No C++
 *     exception ever crosses this boundary.
 */
#ifndef L1B200_H
#define L1B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define L1B_OK 0
#define L1B_EINVAL -1   /* bad shape / index / lambda -> ValueError or IndexError */
#define L1B_ECUDA -2    /* CUDA launch or runtime failure                          */
#define L1B_ENOMEM -3   /* workspace too small                                     */
#define L1B_EINTERNAL -4
#define L1B_EFALLBACK -5  /* l1b_csv_read: the file needs the reference's general CSV rules    */

/* Human-readable text for a status code. */
const char* l1b_status_string(int status);

/* ABI version (bumped on any signature change). */
int l1b_version(void);

/* Bytes of device workspace needed by l1b_prepare + l1b_fit_pivots for an
 * n x m matrix, nlam penalty weights and npiv pivots in the shard. */
size_t l1b_workspace_bytes(int64_t n, int64_t m, int32_t nlam, int64_t npiv);

/* K0: per-column statistics and the pivot-major tableau records.
 * Replaces the lambda-independent half of ratios.py:109-135 (pivot_tableau:
 * nonzero rows, weights |x_ip|) for every pivot at once, plus the column
 * sums sum_i |x_ij| that core.py:93 (residual_error) needs for dead columns
 * and degenerate pivots (fit.py:66-72).  Must run before l1b_fit_pivots on
 * the same workspace whenever X changes. */
int l1b_prepare(const double* d_X, int64_t n, int64_t m, void* d_ws, size_t ws_bytes,
                void* stream);

/* K1 + K2: Algorithm 1 for the pivots {p_begin + k*p_stride : 0 <= k < npiv}
 * and nlam penalty weights h_lams[0..nlam).
 * Replaces fit.py:75-85 (fit_for_pivot) for each pivot and the per-pivot
 * half of fit.py:88-102 (fit_line) -- everything except the final argmin,
 * which l1b_argmin performs.  Outputs (device, lambda-major):
 *   d_V   [nlam][npiv][m]  direction per pivot (v[p] = 1, or all 0 for a
 *                          zero pivot column); may be NULL if not wanted
 *   d_err [nlam][npiv]     sum_ij |x_ij - v_j x_ip|       (core.py:93)
 *   d_pen [nlam][npiv]     sum_j |v_j|                    (core.py:131)
 *   d_obj [nlam][npiv]     err + lam * pen                (core.py:133)
 * Rejects lambda < 0 or NaN (fit.py:20-24); +inf is accepted. */
int l1b_fit_pivots(const double* d_X, int64_t n, int64_t m, const double* h_lams, int32_t nlam,
                   int64_t p_begin, int64_t p_stride, int64_t npiv, double* d_V, double* d_err,
                   double* d_pen, double* d_obj, void* d_ws, size_t ws_bytes, void* stream);

/* l1b_fit_pivots for an arbitrary pivot list h_pivots[0..npiv) (host
 * memory): outputs are indexed by list position.  Used to fit exactly only
 * the pivots l1b_bound_pivots could not rule out. */
int l1b_fit_pivot_list(const double* d_X, int64_t n, int64_t m, const double* h_lams, int32_t nlam,
                       const int64_t* h_pivots, int64_t npiv, double* d_V, double* d_err, double* d_pen,
                       double* d_obj, void* d_ws, size_t ws_bytes, void* stream);

/* Pivot pruning for fit_line (fit.py:88-102 needs only the argmin): for
 * the pivots p_begin + k*p_stride and one lam, one FP32 pass per (pivot,
 * target) problem yields rigorous bounds d_lb[k] <= z_p <= d_ub[k] on the
 * pivot objective z_p (error + lam * penalty, core.py:126-133), float error
 * included as explicit margins.  A pivot with lb > min(ub) cannot be the
 * winner.  Inputs outside the FP32 window get lb = -inf, ub = +inf. */
int l1b_bound_pivots(const double* d_X, int64_t n, int64_t m, double lam, int64_t p_begin, int64_t p_stride,
                     int64_t npiv, double* d_lb, double* d_ub, void* d_ws, size_t ws_bytes, void* stream);

/* The same per-pivot bounds from fit_line's own first pass (the pass
 * l1b_fit_line runs before its cascade): per-pivot sums only -- no per-column
 * bounds or seeds are left in the workspace, so the pass writes 8 bytes per
 * problem (its next range) instead of 48.  steer = 0: one pass over every
 * row; steer = s > 1: a pass over every s-th 64-row chunk first narrows the
 * brackets (tall data, l1b_set_steer). */
int l1b_bound_pivot_sums(const double* d_X, int64_t n, int64_t m, double lam, int64_t p_begin, int64_t p_stride,
                         int64_t npiv, int32_t steer, double* d_lb, double* d_ub, void* d_ws, size_t ws_bytes,
                         void* stream);

/* Algorithm 2 (path.py:76-102) for one pivot: for every target column
 * c (targets j != pivot in ascending order) the tableau's column in stable
 * (ratio, row) order (ratios.py:109-135): d_ratios[c*ld + k] = r_k,
 * d_start[c*ld + k] = sgn(r_k)((T - P_k) - P_{k-1}) - w_k and
 * d_right[c*ld + k] = start + 2 w_k, k < *h_nrows (the pivot's nonzero
 * rows), bit-identical to the reference's NumPy arithmetic.  With all three
 * outputs NULL it only reports *h_nrows (0: zero pivot column, the
 * reference's EmptyPivotError).  Needs l1b_prepare.  Up to 16384 nonzero
 * rows a column is sorted in shared memory; beyond, the three output arrays
 * double as scratch for chunk sorts and global merges (same results). */
int l1b_pivot_breakpoints(const double* d_X, int64_t n, int64_t m, int64_t pivot, int64_t* h_nrows,
                          double* d_ratios, double* d_start, double* d_right, int64_t ld, void* d_ws,
                          size_t ws_bytes, void* stream);

/* pivot_tableau / build_column (ratios.py:40-67, 109-135) on the device:
 * for target column `target` (or, target < 0, every target j != pivot in
 * ascending order, output column c), the column in stable (ratio, row)
 * order: d_ratios[c*ld + k] = fl(x_ij / x_ip), d_weights = |x_ip|,
 * d_prefix = np.cumsum's sequential inclusive prefix, d_rows = source row,
 * k < *h_nrows (the pivot's nonzero rows), bit-identical to the reference.
 * Outputs NULL: size query only (*h_nrows = 0 is the EmptyPivotError case).
 * Replaces the NumPy sort of ratios.py:55,121. */
int l1b_pivot_tableau(const double* d_X, int64_t n, int64_t m, int64_t pivot, int64_t target, int64_t* h_nrows,
                      double* d_ratios, double* d_weights, double* d_prefix, int64_t* d_rows, int64_t ld,
                      void* d_ws, size_t ws_bytes, void* stream);

/* brute_force_column (oracle.py:39-58) for every target column of one pivot
 * (targets j != pivot ascending): the objective at every kink candidate
 * {0} u {x_ij / x_ip}, summed over rows in order; d_t[c] the smallest
 * minimiser (+0.0 for zero), d_f[c] its objective.  O(n^2) per column --
 * an independent check, not a fast path.  d_X device row-major n x m. */
int l1b_brute_force_columns(const double* d_X, int64_t n, int64_t m, int64_t pivot, double lam, double* d_t,
                            double* d_f, void* stream);

/* Optimality certificate of every column of one line (oracle.py:141-174's
 * dual conditions, checked through the subdifferential with exact weight
 * sums): d_slack[j] >= 0 iff v_j (device d_v[m]) minimises pivot `pivot`'s
 * column-j objective at lam; +inf for j == pivot and for a zero pivot column.
 * In weight units (compare with a tolerance for raw, non-grid inputs). */
int l1b_certify_columns(const double* d_X, int64_t n, int64_t m, int64_t pivot, const double* d_v, double lam,
                        double* d_slack, void* d_ws, size_t ws_bytes, void* stream);

/* l1b_bound_pivots for nlam penalties (strictly ascending, host memory) in
 * ONE pass: the histogram range covers the crossings of the smallest and
 * largest penalty (and 0 where the largest may kill the column), and every
 * penalty gets its own bounds from the same histogram and residual.
 * d_lb / d_ub are [nlam][npiv] (device).  d_ranges (device, may be NULL):
 * [nlam][npiv][m] float pairs, each (penalty, pivot, target)'s next range,
 * for l1b_bound_entries to continue from.  The batched lambda sweep (C3). */
int l1b_bound_pivots_multi(const double* d_X, int64_t n, int64_t m, const double* h_lams, int32_t nlam,
                           int64_t p_begin, int64_t p_stride, int64_t npiv, double* d_lb, double* d_ub,
                           void* d_ranges, void* d_ws, size_t ws_bytes, void* stream);

/* l1b_bound_pivots for a pivot list (host memory) with 1 to 3 passes per
 * problem: every further pass re-histograms the range where the previous
 * one proved the optimum lies (62 sub-bins; or extends the range when the
 * optimum lay outside it), which tightens the bounds by orders of magnitude
 * per pass -- used on the pivots the one-pass bounds could not rule out. */
int l1b_bound_pivot_list(const double* d_X, int64_t n, int64_t m, double lam, const int64_t* h_pivots,
                         int64_t npiv, int32_t passes, double* d_lb, double* d_ub, void* d_ws, size_t ws_bytes,
                         void* stream);

/* Reduction half of fit.py:98-102: per lambda, the strict '<' argmin of
 * d_obj[l][0..npiv) in ascending pivot order (ties -> smallest pivot).
 * Writes d_best_k[l] (index into the shard) and d_best_obj[l]. */
int l1b_argmin(const double* d_obj, int32_t nlam, int64_t npiv, int64_t* d_best_k,
               double* d_best_obj, void* stream);

/* core.py:79-93 with NumPy's exact pairwise summation order over the
 * row-major flattened n*m residual |x_ij - fl(x_ip * v_j)|, so the returned
 * error is bit-identical to residual_error() in the reference.  Used to
 * re-score the winning pivot(s).  d_out is one double. */
int l1b_residual_exact(const double* d_X, int64_t n, int64_t m, const double* d_v, int64_t p,
                       double* d_out, void* d_ws, size_t ws_bytes, void* stream);

/* l1b_residual_exact for `count` candidate lines at once: direction k is
 * d_V + k*ldv (device), its pivot h_pivots[k]; d_out[k] (device) receives
 * its exact residual error (NumPy's summation order, bit-identical). */
int l1b_residual_exact_batch(const double* d_X, int64_t n, int64_t m, const double* d_V, int64_t ldv,
                             const int64_t* h_pivots, int64_t count, double* d_out, void* d_ws, size_t ws_bytes,
                             void* stream);

/* subspace.py:22-36 deflate: X <- X - (X w) w^T with w = v / ||v||_2, in
 * place.  d_tmp must hold n + 1 doubles. */
int l1b_deflate(double* d_X, int64_t n, int64_t m, const double* d_v, double* d_tmp, void* stream);

/* max_ij |x_ij| into d_out[0] (the early-stop test of subspace.py:67,71). */
int l1b_absmax(const double* d_X, int64_t n, int64_t m, double* d_out, void* stream);

/* Host memcpy for the staging of an upload (no reference counterpart: the
 * reference never leaves the host): dst <- src, `bytes` bytes, split over
 * `threads` threads of a persistent pool (<= 0: 8), written with streaming
 * stores so the pinned destination is not left dirty in the CPU caches when
 * the copy engine reads it (hostcopy.inc). */
int l1b_host_copy(void* dst, const void* src, size_t bytes, int32_t threads);

/* Host -> device upload of `bytes` from pageable h_src through two pinned
 * staging buffers of stage_bytes each (l1b_host_copy into one while the copy
 * engine reads the other), all on `stream`; returns once the last transfer is
 * queued (the staging buffers must not be reused before the stream passes it). */
int l1b_upload(void* d_dst, const void* h_src, size_t bytes, void* h_stage0, void* h_stage1, size_t stage_bytes,
               int32_t threads, void* stream);

/* The same max_ij |x_ij| of the matrix the workspace was last prepared for
 * (l1b_prepare computes it with the column statistics): one 8-byte copy into
 * d_out[0] on the stream, no pass over X. */
int l1b_prepared_absmax(const void* d_ws, int64_t n, int64_t m, size_t ws_bytes, double* d_out, void* stream);

/* Self-test of the bit-exact division used by K1 (no reference counterpart;
 * it backs the parity claim for ratios.py:119 R = X[rows,t] / x_p): n_pairs
 * random (a, b) in the SAFE exponent window, counting results that differ
 * from IEEE __ddiv_rn into *d_mismatches (device uint64). */
int l1b_selftest_divide(uint64_t seed, int64_t n_pairs, uint64_t* d_mismatches, void* stream);

/* Diagnostics of the last l1b_fit_pivots on this workspace (no reference
 * counterpart): h_out[0], h_out[1] = number of (pivot, target) problems the
 * main selection kernel handed to the exact straggler solver for the last
 * two penalty weights (even / odd index).  Synchronises the stream. */
int l1b_fit_stats(int64_t n, int64_t m, int64_t npiv, const void* d_ws, size_t ws_bytes,
                  uint64_t* h_out, void* stream);

/* Profiling aid (no reference counterpart): when d_buf is non-NULL, every
 * later k_select launch writes per-CTA %globaltimer stamps at its phase
 * boundaries (sample, F passes, pass B, resolve) into d_buf[cta * 8 + k];
 * d_buf must hold 8 * (number of CTAs) uint64.  NULL switches it off. */
int l1b_set_probe(uint64_t* d_buf);

/* Diagnostics (no reference counterpart): copies up to max_records of the
 * last l1b_fit_pivots' straggler queue (40-byte records: int32 pivot index
 * in the shard, int32 target, uint64 key interval lo, hi, double unused,
 * double G) to host memory; returns the number copied or a status < 0.
 * Synchronises the stream. */
int l1b_straggler_records(int64_t n, int64_t m, int64_t npiv, const void* d_ws, size_t ws_bytes, void* h_out,
                          int64_t max_records, void* stream);

/* One more bounding pass for a pivot list that the previous l1b_bound_*
 * call on this workspace covered: pivot k was entry h_from[k] of that call's
 * list of from_npiv pivots, and its pass starts from the range that call
 * left for each (pivot, target) problem.  A cascade (all pivots, then the
 * survivors, then theirs) costs one pass per level per surviving pivot. */
int l1b_bound_pivot_list_continue(const double* d_X, int64_t n, int64_t m, double lam, const int64_t* h_pivots,
                                  int64_t npiv, const int64_t* h_from, int64_t from_npiv, double* d_lb,
                                  double* d_ub, void* d_ws, size_t ws_bytes, void* stream);

/* Optional hook of a sharded fit: maps this shard's best upper bound to the
 * best over all shards (an all-reduce MIN); called once per pruned fit. */
typedef double (*l1b_ub_exchange_fn)(double top, void* ctx);

/* fit_line (fit.py:88-102) over one pivot shard (p_begin + k p_stride,
 * k < npiv) in one call: bounds every pivot, refines the survivors, fits the
 * rest exactly (seeded) and re-scores the near-minimal ones in NumPy's order;
 * prune = 1 / 0 / -1 (auto: m > 32 and m^2 n >= 2^24).  Outputs the winning
 * pivot, its direction (device d_v[m]) and its error, penalty norm and
 * objective exactly as the reference computes them; *h_candidates (may be
 * NULL) gets the number of pivots fitted exactly.  With ub_exchange (may be
 * NULL) the shard prunes against the global best and may keep no pivot:
 * then *h_pivot = -1.  Synchronises the stream. */
int l1b_fit_line(const double* d_X, int64_t n, int64_t m, double lam, int64_t p_begin, int64_t p_stride,
                 int64_t npiv, int32_t prune, l1b_ub_exchange_fn ub_exchange, void* exchange_ctx, int64_t* h_pivot,
                 double* d_v, double* h_err, double* h_pen, double* h_obj, int64_t* h_candidates, void* d_ws,
                 size_t ws_bytes, void* stream);

/* Vector form of the exchange hook (a penalty sweep): replaces tops[0..count)
 * -- this shard's best upper bound per penalty -- by the best over all shards. */
typedef void (*l1b_ub_exchange_vec_fn)(double* tops, int32_t count, void* ctx);

/* fit_lines for one pivot shard in one call: every penalty of h_lams (>= 2
 * distinct finite values; any order, repeats allowed) bounded by one
 * multi-penalty pass, the survivors of all penalties refined and fitted as one
 * entry list per level, the near-minimal candidates re-scored in NumPy's order.
 * Per input penalty j: h_pivot[j] (-1 when another shard provably wins),
 * d_v[j*m .. j*m+m), h_err[j], h_pen[j], h_obj[j].  d_bounds: device scratch of
 * 2 * L * npiv doubles (L distinct penalties); d_ranges (may be NULL): device
 * scratch of ranges_bytes >= 8 L npiv m for the per-penalty next ranges (the
 * first refinement level continues from them).  Synchronises the stream. */
int l1b_fit_lines(const double* d_X, int64_t n, int64_t m, const double* h_lams, int32_t nlam, int64_t p_begin,
                  int64_t p_stride, int64_t npiv, l1b_ub_exchange_vec_fn ub_exchange, void* exchange_ctx,
                  double* d_bounds, void* d_ranges, size_t ranges_bytes, int64_t* h_pivot, double* d_v,
                  double* h_err, double* h_pen, double* h_obj, int64_t* h_candidates, void* d_ws, size_t ws_bytes,
                  void* stream);

/* Entry lists (a penalty sweep's survivors, batched): count (pivot, penalty)
 * entries h_pivots[k], h_lams[k] in one launch.  l1b_bound_entries is one
 * bounding pass per entry -- from row samples at the entry's penalty, or,
 * with h_from, continuing from entry h_from[k] of the previous bound call's
 * list of from_count entries (or, with d_from_ranges, from row h_from[k] of
 * l1b_bound_pivots_multi's d_ranges); l1b_fit_entries_seeded is the seeded exact fit
 * of entries (h_seed[k]: entry of the last bound call).  Same outputs as the
 * single-penalty calls, per entry. */
int l1b_bound_entries(const double* d_X, int64_t n, int64_t m, const double* h_lams, const int64_t* h_pivots,
                      int64_t count, const int64_t* h_from, int64_t from_count, const void* d_from_ranges,
                      double* d_lb, double* d_ub, void* d_ws, size_t ws_bytes, void* stream);
int l1b_fit_entries_seeded(const double* d_X, int64_t n, int64_t m, const double* h_lams, const int64_t* h_pivots,
                           int64_t count, const int64_t* h_seed, int64_t seed_count, double* d_V, double* d_err,
                           double* d_pen, double* d_obj, void* d_ws, size_t ws_bytes, void* stream);

/* Exact fit (as l1b_fit_pivot_list, one lambda) of a short pivot list that
 * a preceding l1b_bound_pivot_list call on this workspace bounded: pivot k
 * is entry h_seed[k] of that call's list of seed_npiv pivots (-1: no seed).
 * Every (pivot, target) problem goes to the warp-per-problem exact solver,
 * started on the range the bound passes left for its optimum (typically a
 * handful of rows, so one collecting pass), instead of the batched
 * k_select path whose per-CTA row loop is latency-bound for few pivots.
 * Results are identical to l1b_fit_pivot_list. */
int l1b_fit_pivot_list_seeded(const double* d_X, int64_t n, int64_t m, double lam, const int64_t* h_pivots,
                              int64_t npiv, const int64_t* h_seed, int64_t seed_npiv, double* d_V, double* d_err,
                              double* d_pen, double* d_obj, void* d_ws, size_t ws_bytes, void* stream);

/* Per-column bounds lb_pj <= f_j* <= ub_pj ([npiv][m], pivot order) of the
 * last l1b_bound_* call on this workspace, which bounded npiv pivots; copied
 * to host memory (test and diagnostic accessor).  Synchronises the stream. */
int l1b_bound_columns(int64_t n, int64_t m, int64_t npiv, const void* d_ws, size_t ws_bytes, double* h_lb,
                      double* h_ub, void* stream);

/* Device time (CUDA events on the launching stream) of the last k_bound
 * launch made by l1b_bound_pivots / l1b_bound_pivot_list; waits for it.
 * Benchmark evidence for the roofline (no reference counterpart). */
int l1b_last_bound_ms(float* ms);

/* Shared-memory atomic throughput probe: blocks x threads threads issue
 * 8 * iters conflict-free 32-bit shared-memory adds each (the operation
 * k_bound's histograms are built from); bench.py times it for the peak. */
int l1b_atoms_probe(int64_t iters, int32_t blocks, int32_t threads, uint32_t* d_out, void* stream);

/* Cumulative count of kernels this library has enqueued in the process
 * (benchmark evidence for "gpu_launches"; no reference counterpart). */
uint64_t l1b_kernel_launches(void);

/* FP64 pipe probe: `blocks` x `threads` threads each run 8 independent DFMA
 * chains of `iters` steps (8 * iters FMAs per thread).  bench.py times it
 * with CUDA events to measure the FP64 peak the roofline is quoted against.
 * d_out: one device double (written only to keep the chains alive). */
int l1b_dfma_probe(int64_t iters, int32_t blocks, int32_t threads, double* d_out, void* stream);

/* read_matrix (io.py:46-85) for plain numeric CSV files, natively and in
 * parallel (threads <= 0: all cores): *out_values (row-major n x m,
 * malloc'd; free with l1b_csv_free) holds exactly the doubles float()
 * parses.  Returns L1B_EFALLBACK for quotes, underscores, non-ASCII bytes,
 * lone CRs, and for every malformed file (ragged rows, non-numeric or
 * non-finite cells, no data): the caller then applies the reference's rules
 * (and its exact error messages).  With has_header, *out_header (malloc'd,
 * may be NULL) is the header line. */
int l1b_csv_read(const char* path, int32_t has_header, int32_t threads, double** out_values, int64_t* out_n,
                 int64_t* out_m, char** out_header);
void l1b_csv_free(void* p);

/* Algorithm 3 (path.py:166-277, merge_path) on the host, bit-identical to
 * the reference: X host row-major n x m; the grid lambdas[K]; usable pivots
 * piv[np_] and degenerate pivots deg[nd], both ascending; breakpoint events
 * (pivot ev_p, target ev_t, value ev_v) grouped by snapped grid index
 * (ev_off[K+1]) in the reference's insertion order.  Writes up to cap path
 * segments (o_lo, o_hi, o_piv, o_v [cap][m], o_err, o_pen, o_obj, o_zlo,
 * o_zhi) and *count; L1B_ENOMEM (with *count set) when cap is short. */
int l1b_merge_path(const double* X, int64_t n, int64_t m, const double* lambdas, int64_t K, const int64_t* piv,
                   int64_t np_, const int64_t* deg, int64_t nd, const int64_t* ev_off, const int64_t* ev_p,
                   const int64_t* ev_t, const double* ev_v, int64_t cap, double* o_lo, double* o_hi,
                   int64_t* o_piv, double* o_v, double* o_err, double* o_pen, double* o_obj, double* o_zlo,
                   double* o_zhi, int64_t* count);

/* Algorithm 3 with its data-parallel parts on the device (csrc/merge_dev.cuh),
 * the same arguments and bit-identical results as l1b_merge_path but X on the
 * device (d_X, after l1b_prepare on d_ws): every event's column error, every
 * pivot's running (sum colerr, sum |v|), every grid interval's crossing
 * analysis and probe minima run as kernels; the host keeps the sequential
 * segment walk; the segment lines' residuals are batched on the device.
 * Scratch is stream-ordered (cudaMallocAsync on `stream`).  The *count
 * segments come back in one malloc'ed block *o_seg of [count][8 + m]
 * doubles (lo, hi, pivot, err, pen, obj, z_lo, z_hi, v[m]); free it with
 * l1b_csv_free. */
/* Steering of l1b_fit_line's first bound pass on workspace d_ws: -1
 * automatic (a 1-in-8 row-chunk steering pass for n >= 32768), 0 off, s > 1 a
 * steering pass over every s-th 64-row chunk.  fit_subspace turns it off for
 * the first component (one pass prunes it) and back to automatic for the
 * deflated ones (whose pivots sit within ~1e-4 of each other). */
int l1b_set_steer(const void* d_ws, int32_t mode);

/* path.py:157-163 for E breakpoint events at once: out_order[E] = the events
 * grouped by their snapped grid index (ascending; insertion order within a
 * group), out_off[K+1] = group offsets.  Host arrays.  L1B_EINTERNAL when a
 * breakpoint is not within tol of the grid (the reference's AssertionError). */
int l1b_snap_events(const double* lambdas, int64_t K, const double* bp, int64_t E, double tol, int64_t* out_order,
                    int64_t* out_off);

int l1b_merge_path_device(const double* d_X, int64_t n, int64_t m, const double* lambdas, int64_t K,
                          const int64_t* piv, int64_t np_, const int64_t* deg, int64_t nd, const int64_t* ev_off,
                          const int64_t* ev_p, const int64_t* ev_t, const double* ev_v, double** o_seg,
                          int64_t* count, void* d_ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* L1B200_H */
