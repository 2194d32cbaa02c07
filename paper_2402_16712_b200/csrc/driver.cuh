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


// A penalty sweep (fit_lines) for one pivot shard in one call: the cascade of
// engine.DeviceFit._sweep_winners in C++ (one multi-penalty bound pass, every
// penalty's survivors refined and fitted as one entry list per level, the
// near-minimal candidates re-scored in NumPy's order), so a step makes no
// Python round trips between its synchronisations.
int l1b_fit_lines(const double* d_X, int64_t n, int64_t m, const double* h_lams, int32_t nlam, int64_t p_begin,
                  int64_t p_stride, int64_t npiv, l1b_ub_exchange_vec_fn ub_exchange, void* exchange_ctx,
                  double* d_bounds, void* d_ranges, size_t ranges_bytes, int64_t* h_pivot, double* d_v,
                  double* h_err, double* h_pen, double* h_obj, int64_t* h_candidates, void* d_ws, size_t ws_bytes,
                  void* stream) {
  if (!d_X || !h_lams || !d_bounds || !h_pivot || !d_v || !h_err || !h_pen || !h_obj || n < 1 || m < 2 ||
      nlam < 1 || npiv < 1)
    return L1B_EINVAL;
  if (p_stride < 1 || p_begin < 0 || p_begin + (npiv - 1) * p_stride >= m) return L1B_EINVAL;
  std::vector<double> uniq(h_lams, h_lams + nlam);
  for (double x : uniq)
    if (!(x >= 0.0) || !std::isfinite(x)) return L1B_EINVAL;
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  const int32_t L = (int32_t)uniq.size();
  if (L < 2) return L1B_EINVAL;  // one penalty: l1b_fit_line
  Workspace w;
  const int64_t cap = ws_capacity(n, m, ws_bytes);
  if (cap < npiv) return L1B_ENOMEM;
  carve(&w, d_ws, n, m, cap);
  cudaStream_t s = (cudaStream_t)stream;
  auto sync = [&]() { return cudaStreamSynchronize(s) == cudaSuccess; };
  double* d_lb = w.drv;
  double* d_ub = w.drv + cap;
  double* d_err = w.drv + 2 * cap;
  double* d_pen = w.drv + 3 * cap;
  double* d_obj = w.drv + 4 * cap;
  // one bounding pass for every penalty; its per-penalty next ranges let the
  // first refinement level continue instead of re-sampling
  const bool keep = d_ranges && ranges_bytes >= (size_t)L * (size_t)npiv * (size_t)m * sizeof(float2);
  int st = l1b_bound_pivots_multi(d_X, n, m, uniq.data(), L, p_begin, p_stride, npiv, d_bounds,
                                  d_bounds + (size_t)L * npiv, keep ? d_ranges : nullptr, d_ws, ws_bytes, stream);
  if (st != L1B_OK) return st;
  std::vector<double> lbm((size_t)L * npiv), ubm((size_t)L * npiv);
  double amax = 0.0;
  if (cudaMemcpyAsync(&amax, w.flags + 6, sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(lbm.data(), d_bounds, sizeof(double) * lbm.size(), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaMemcpyAsync(ubm.data(), d_bounds + (size_t)L * npiv, sizeof(double) * ubm.size(), cudaMemcpyDeviceToHost,
                      s) != cudaSuccess || !sync())
    return L1B_ECUDA;
  const double abs_scale = amax * (double)n * (double)m;
  auto thr = [&](double top) {
    return std::isfinite(top) ? top + kPruneRtol * fabs(top) + kRescoreAtol * abs_scale : INFINITY;
  };
  std::vector<double> tops(L, INFINITY);
  for (int32_t i = 0; i < L; ++i)
    for (int64_t k = 0; k < npiv; ++k) tops[i] = std::min(tops[i], ubm[(size_t)i * npiv + k]);
  if (ub_exchange) ub_exchange(tops.data(), L, exchange_ctx);  // every penalty's best over all shards
  std::vector<std::vector<int64_t>> ent(L);
  for (int32_t i = 0; i < L; ++i)
    for (int64_t k = 0; k < npiv; ++k)
      if (!(lbm[(size_t)i * npiv + k] > thr(tops[i]))) ent[i].push_back(k);  // NaN-safe: keep unless worse
  // entry lists are bounded by the workspace's pivot capacity
  std::vector<std::vector<int32_t>> batches;
  {
    std::vector<int32_t> cur;
    int64_t size = 0;
    for (int32_t i = 0; i < L; ++i) {
      const int64_t c = (int64_t)ent[i].size();
      if (!cur.empty() && size + c > cap) {
        batches.push_back(cur);
        cur.clear();
        size = 0;
      }
      cur.push_back(i);
      size += c;
    }
    if (!cur.empty()) batches.push_back(cur);
  }
  std::vector<int64_t> wpiv(L, -1);
  std::vector<double> werr(L, 0.0), wpen(L, 0.0), wobj(L, 0.0);
  std::vector<std::vector<double>> wv(L);
  int64_t ncand = 0;
  for (const auto& bl : batches) {
    std::vector<int32_t> li;
    std::vector<int64_t> kk, seed;
    for (int32_t i : bl)
      for (int64_t k : ent[i]) {
        li.push_back(i);
        kk.push_back(k);
      }
    int64_t seed_n = 0;
    const void* src = nullptr;
    if (keep) {  // level 0 continues from the multi pass's per-penalty ranges
      seed.resize(li.size());
      for (size_t e = 0; e < li.size(); ++e) seed[e] = (int64_t)li[e] * npiv + kk[e];
      seed_n = (int64_t)L * npiv;
      src = d_ranges;
    }
    std::vector<double> lam_e, lb2, ub2;
    std::vector<int64_t> piv_e;
    auto entries = [&]() {
      lam_e.resize(li.size());
      piv_e.resize(li.size());
      for (size_t e = 0; e < li.size(); ++e) {
        lam_e[e] = uniq[li[e]];
        piv_e[e] = p_begin + kk[e] * p_stride;
      }
    };
    for (int level = 0; level <= kRefinePasses; ++level) {
      if (kk.empty()) break;
      if (level > 0) {
        std::vector<int64_t> counts(L, 0);
        for (int32_t i : li) ++counts[i];
        if (std::all_of(counts.begin(), counts.end(), [](int64_t c) { return c <= kRefineMin; })) break;
      }
      entries();
      const int64_t K = (int64_t)li.size();
      st = l1b_bound_entries(d_X, n, m, lam_e.data(), piv_e.data(), K, seed.empty() ? nullptr : seed.data(),
                             seed_n, src, d_lb, d_ub, d_ws, ws_bytes, stream);
      if (st != L1B_OK) return st;
      src = nullptr;
      lb2.resize(K);
      ub2.resize(K);
      if (cudaMemcpyAsync(lb2.data(), d_lb, sizeof(double) * K, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
          cudaMemcpyAsync(ub2.data(), d_ub, sizeof(double) * K, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
          !sync())
        return L1B_ECUDA;
      for (int64_t e = 0; e < K; ++e) tops[li[e]] = std::min(tops[li[e]], ub2[e]);
      std::vector<int32_t> nli;
      std::vector<int64_t> nkk, sel;
      for (int64_t e = 0; e < K; ++e)
        if (!(lb2[e] > thr(tops[li[e]]))) {
          nli.push_back(li[e]);
          nkk.push_back(kk[e]);
          sel.push_back(e);
        }
      li.swap(nli);
      kk.swap(nkk);
      seed.swap(sel);
      seed_n = K;
    }
    ncand += (int64_t)kk.size();
    if (kk.empty()) continue;
    entries();
    const int64_t K = (int64_t)li.size();
    st = l1b_fit_entries_seeded(d_X, n, m, lam_e.data(), piv_e.data(), K, seed.data(), seed_n, nullptr, d_err, d_pen,
                                d_obj, d_ws, ws_bytes, stream);
    if (st != L1B_OK) return st;
    std::vector<double> obj(K);
    if (cudaMemcpyAsync(obj.data(), d_obj, sizeof(double) * K, cudaMemcpyDeviceToHost, s) != cudaSuccess || !sync())
      return L1B_ECUDA;
    // near-minimal candidates of every penalty (engine._candidates), ascending pivot order
    std::vector<int64_t> ce_idx;  // entry index of each candidate
    std::vector<int32_t> ce_lam;  // its penalty
    for (int32_t i : bl) {
      double best = INFINITY;
      bool any = false;
      for (int64_t e = 0; e < K; ++e)
        if (li[e] == i) {
          if (std::isnan(obj[e])) return L1B_EINVAL;
          best = std::min(best, obj[e]);
          any = true;
        }
      if (!any) continue;
      for (int64_t e = 0; e < K; ++e) {
        if (li[e] != i) continue;
        const bool near = std::isinf(best) ? obj[e] == best
                                           : obj[e] <= best + kRescoreRtol * fabs(best) + kRescoreAtol * abs_scale +
                                                           1e-300;
        if (near) {
          ce_idx.push_back(e);
          ce_lam.push_back(i);
          if (std::isinf(best)) break;
        }
      }
    }
    const int64_t C = (int64_t)ce_idx.size();
    for (int64_t c = 0; c < C; ++c)
      if (cudaMemcpyAsync(w.ework + c * m, w.vwork + ce_idx[c] * m, sizeof(double) * m, cudaMemcpyDeviceToDevice,
                          s) != cudaSuccess)
        return L1B_ECUDA;
    std::vector<int64_t> cp(C);
    for (int64_t c = 0; c < C; ++c) cp[c] = piv_e[ce_idx[c]];
    st = l1b_residual_exact_batch(d_X, n, m, w.ework, m, cp.data(), C, d_err, d_ws, ws_bytes, stream);
    if (st != L1B_OK) return st;
    std::vector<double> errs(C), vh((size_t)C * m), av(m);
    if (cudaMemcpyAsync(errs.data(), d_err, sizeof(double) * C, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaMemcpyAsync(vh.data(), w.ework, sizeof(double) * C * m, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        !sync())
      return L1B_ECUDA;
    for (int64_t c = 0; c < C; ++c) {  // first strict minimum per penalty, in pivot order (fit.py:98-102)
      const int32_t i = ce_lam[c];
      for (int64_t j = 0; j < m; ++j) av[j] = fabs(vh[(size_t)c * m + j]);
      const double pn = np_pairwise(av.data(), m);
      const double z = errs[c] + uniq[i] * pn;
      if (wpiv[i] < 0 || z < wobj[i]) {
        wpiv[i] = cp[c];
        werr[i] = errs[c];
        wpen[i] = pn;
        wobj[i] = z;
        wv[i].assign(vh.begin() + (size_t)c * m, vh.begin() + (size_t)(c + 1) * m);
      }
    }
  }
  if (h_candidates) *h_candidates = ncand;
  for (int32_t j = 0; j < nlam; ++j) {
    const int32_t i = (int32_t)(std::lower_bound(uniq.begin(), uniq.end(), h_lams[j]) - uniq.begin());
    h_pivot[j] = wpiv[i];
    h_err[j] = werr[i];
    h_pen[j] = wpen[i];
    h_obj[j] = wobj[i];
    if (wpiv[i] >= 0 &&
        cudaMemcpyAsync(d_v + (size_t)j * m, wv[i].data(), sizeof(double) * m, cudaMemcpyHostToDevice, s) !=
            cudaSuccess)
      return L1B_ECUDA;
  }
  return sync() ? L1B_OK : L1B_ECUDA;
}
}  // extern "C"
