// driver.cuh -- fit_line for one pivot shard in one C call (included at the
// end of l1b200.cu).
//
// The pruned cascade of engine.DeviceFit.shard_winners, host logic in C++
// so a step makes no Python round trips: bound every pivot (k_bound) ->
// keep lb <= min ub (1 + 1e-9) -> up to three continuing passes on the
// survivors while more than two remain -> seeded exact fit of the rest ->
// re-score the near-minimal candidates in NumPy's order (exact residual on
// the device, the penalty norm with NumPy's pairwise sum on the host) ->
// the first strict minimum in pivot order (fit.py:98-102).

namespace {

constexpr double kRescoreRtol = 1e-8;   // engine.RESCORE_RTOL
constexpr double kRescoreAtol = 1e-13;  // engine.RESCORE_ATOL (times n m max|x|)
constexpr double kPruneRtol = 1e-9;     // engine.PRUNE_RTOL
constexpr int kRefineMin = 2, kRefinePasses = 3;
constexpr int64_t kSteerRows = 32768;  // rows from which the first pass is steered by a row sample
constexpr int kSteerStride = 8;        // the steering sample: every 8th 64-row chunk

// NumPy's pairwise_sum_DOUBLE for a contiguous array (loops_utils.h.src):
// n < 8 sequential, n <= 128 eight strided accumulators, else split at n/2
// rounded down to a multiple of 8.
double np_pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int q = 0; q < 8; ++q) r[q] = a[q];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int q = 0; q < 8; ++q) r[q] += a[i + q];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise(a, n2) + np_pairwise(a + n2, n - n2);
}

}  // namespace

extern "C" {

int l1b_fit_line(const double* d_X, int64_t n, int64_t m, double lam, int64_t p_begin, int64_t p_stride,
                 int64_t npiv, int32_t prune, l1b_ub_exchange_fn ub_exchange, void* exchange_ctx, int64_t* h_pivot,
                 double* d_v, double* h_err, double* h_pen, double* h_obj, int64_t* h_candidates, void* d_ws,
                 size_t ws_bytes, void* stream) {
  if (!d_X || !h_pivot || !d_v || !h_err || !h_pen || !h_obj || n < 1 || m < 2 || npiv < 1 || !(lam >= 0.0))
    return L1B_EINVAL;
  if (p_stride < 1 || p_begin < 0 || p_begin + (npiv - 1) * p_stride >= m) return L1B_EINVAL;
  Workspace w;
  const int64_t cap = ws_capacity(n, m, ws_bytes);
  if (cap < npiv) return L1B_ENOMEM;
  carve(&w, d_ws, n, m, cap);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t ce;
  auto sync = [&]() { return cudaStreamSynchronize(s) == cudaSuccess; };
  // device scratch: lb, ub [npiv] and err/pen/obj [npiv] (the driver's own region)
  double* d_lb = w.drv;
  double* d_ub = w.drv + cap;
  double* d_err = w.drv + 2 * cap;
  double* d_pen = w.drv + 3 * cap;
  double* d_obj = w.drv + 4 * cap;
  // n m max|x|: the re-score window's absolute floor (K0 left max |x| in the
  // workspace; read with the first results, so nothing waits before the
  // first pass is queued)
  int st = L1B_OK;
  double amax = 0.0, abs_scale = 0.0;  // abs_scale set once the copy has synchronised
  auto read_amax = [&]() {
    return cudaMemcpyAsync(&amax, w.flags + 6, sizeof(double), cudaMemcpyDeviceToHost, s) == cudaSuccess;
  };
  auto thr = [&](double top) {
    return std::isfinite(top) ? top + kPruneRtol * fabs(top) + kRescoreAtol * abs_scale : INFINITY;
  };
  std::vector<int64_t> piv(npiv);
  for (int64_t k = 0; k < npiv; ++k) piv[k] = p_begin + k * p_stride;
  const bool do_prune = prune > 0 || (prune < 0 && m > 32 && (double)m * m * n >= 16777216.0);
  std::vector<int64_t> cand_piv, seed;
  int64_t seed_n = 0;
  std::vector<double> lb(npiv), ub(npiv);
  int64_t nfit;
  if (do_prune) {
    // lean: per-pivot bound sums and next ranges only (the continuing passes
    // over the survivors write their seeds and column bounds)
    // tall columns: a steering pass over a row sample narrows the first full
    // pass's brackets (deflated components of tall data prune only then)
    int steer = n >= kSteerRows ? kSteerStride : 0;
    {
      std::lock_guard<std::mutex> g(g_win_mu);
      const auto it = g_steer.find(d_ws);
      if (it != g_steer.end() && it->second >= 0) steer = it->second;  // l1b_set_steer
    }
    if (const char* e = getenv("L1B200_STEER")) steer = atoi(e);  // tuning knob: chunk stride, 0 = off
    st = fit_impl(d_X, n, m, &lam, 1, p_begin, p_stride, nullptr, npiv, true, nullptr, nullptr, nullptr, nullptr,
                  d_lb, d_ub, d_ws, ws_bytes, stream, 1, nullptr, 0, nullptr, nullptr, nullptr, /*lean=*/true, steer);
    if (st != L1B_OK) return st;
    if (!read_amax() ||
        cudaMemcpyAsync(lb.data(), d_lb, sizeof(double) * npiv, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(ub.data(), d_ub, sizeof(double) * npiv, cudaMemcpyDeviceToHost, s) != cudaSuccess || !sync())
      return L1B_ECUDA;
    abs_scale = amax * (double)n * (double)m;
    double top = INFINITY;
    for (double u : ub) top = std::min(top, u);  // NaN never wins std::min here
    if (ub_exchange) top = ub_exchange(top, exchange_ctx);  // the best upper bound over every shard
    std::vector<int64_t> keep;
    for (int64_t k = 0; k < npiv; ++k)
      if (!(lb[k] > thr(top))) keep.push_back(k);  // NaN-safe: keep unless provably worse
    seed = keep;
    seed_n = npiv;
    std::vector<int64_t> list(keep.size());
    for (size_t i = 0; i < keep.size(); ++i) list[i] = piv[keep[i]];
    // at least one continuing pass: the lean pass left no exact-solver seeds
    bool seeded_ranges = false;
    for (int level = 0; level < kRefinePasses && !list.empty() && (!seeded_ranges || (int64_t)list.size() > kRefineMin);
         ++level) {
      seeded_ranges = true;
      const int64_t c = (int64_t)list.size();
      st = fit_impl(d_X, n, m, &lam, 1, 0, 1, list.data(), c, true, nullptr, nullptr, nullptr, nullptr, d_lb, d_ub,
                    d_ws, ws_bytes, stream, 1, seed.data(), seed_n);
      if (st != L1B_OK) return st;
      lb.resize(c);
      ub.resize(c);
      if (cudaMemcpyAsync(lb.data(), d_lb, sizeof(double) * c, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
          cudaMemcpyAsync(ub.data(), d_ub, sizeof(double) * c, cudaMemcpyDeviceToHost, s) != cudaSuccess || !sync())
        return L1B_ECUDA;
      for (int64_t k = 0; k < c; ++k) top = std::min(top, ub[k]);
      std::vector<int64_t> sel, nl;
      for (int64_t k = 0; k < c; ++k)
        if (!(lb[k] > thr(top))) {
          sel.push_back(k);
          nl.push_back(list[k]);
        }
      seed = sel;
      seed_n = c;
      list = nl;
    }
    cand_piv = list;
    nfit = (int64_t)cand_piv.size();
    if (nfit == 0) {  // another shard holds a pivot provably better than all of ours
      *h_pivot = -1;
      if (h_candidates) *h_candidates = 0;
      return L1B_OK;
    }
    st = fit_impl(d_X, n, m, &lam, 1, 0, 1, cand_piv.data(), nfit, false, nullptr, d_err, d_pen, d_obj, nullptr,
                  nullptr, d_ws, ws_bytes, stream, 1, seed.data(), seed_n);
  } else {
    cand_piv = piv;
    nfit = npiv;
    st = fit_impl(d_X, n, m, &lam, 1, p_begin, p_stride, nullptr, npiv, false, nullptr, d_err, d_pen, d_obj,
                  nullptr, nullptr, d_ws, ws_bytes, stream);
  }
  if (st != L1B_OK) return st;
  if (h_candidates) *h_candidates = nfit;
  std::vector<double> obj(nfit);
  if ((!do_prune && !read_amax()) ||
      cudaMemcpyAsync(obj.data(), d_obj, sizeof(double) * nfit, cudaMemcpyDeviceToHost, s) != cudaSuccess || !sync())
    return L1B_ECUDA;
  abs_scale = amax * (double)n * (double)m;
  // near-minimal candidates (engine._candidates), ascending pivot order
  double best = INFINITY;
  for (double o : obj) {
    if (std::isnan(o)) return L1B_EINVAL;  // lam = inf with an all-zero pivot column (core.py:120-124)
    best = std::min(best, o);
  }
  std::vector<int64_t> ck;
  for (int64_t k = 0; k < nfit; ++k) {
    if (std::isinf(best) ? obj[k] == best : obj[k] <= best + kRescoreRtol * fabs(best) + kRescoreAtol * abs_scale + 1e-300)
      ck.push_back(k);
    if (std::isinf(best) && !ck.empty()) break;
  }
  // candidates' directions: rows of the fit's value array, moved aside (the
  // batched residual uses that array as scratch)
  const int64_t C = (int64_t)ck.size();
  for (int64_t i = 0; i < C; ++i) {
    ce = cudaMemcpyAsync(w.ework + i * m, w.vwork + ck[i] * m, sizeof(double) * m, cudaMemcpyDeviceToDevice, s);
    if (ce != cudaSuccess) return L1B_ECUDA;
  }
  std::vector<int64_t> cp(C);
  for (int64_t i = 0; i < C; ++i) cp[i] = cand_piv[ck[i]];
  st = l1b_residual_exact_batch(d_X, n, m, w.ework, m, cp.data(), C, d_err, d_ws, ws_bytes, stream);
  if (st != L1B_OK) return st;
  std::vector<double> errs(C), vh((size_t)C * m);
  if (cudaMemcpyAsync(errs.data(), d_err, sizeof(double) * C, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(vh.data(), w.ework, sizeof(double) * C * m, cudaMemcpyDeviceToHost, s) != cudaSuccess || !sync())
    return L1B_ECUDA;
  int64_t win = -1;
  double wz = 0.0, we = 0.0, wp = 0.0;
  std::vector<double> av(m);
  for (int64_t i = 0; i < C; ++i) {
    for (int64_t j = 0; j < m; ++j) av[j] = fabs(vh[(size_t)i * m + j]);
    const double pn = np_pairwise(av.data(), m);
    const double z = errs[i] + lam * pn;
    if (win < 0 || z < wz) {
      win = i;
      wz = z;
      we = errs[i];
      wp = pn;
    }
  }
  *h_pivot = cp[win];
  *h_err = we;
  *h_pen = wp;
  *h_obj = wz;
  ce = cudaMemcpyAsync(d_v, w.ework + win * m, sizeof(double) * m, cudaMemcpyDeviceToDevice, s);
  if (ce != cudaSuccess || !sync()) return L1B_ECUDA;
  return L1B_OK;
}

}  // extern "C"
