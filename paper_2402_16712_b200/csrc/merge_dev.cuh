// merge_dev.cuh -- Algorithm 3 (the envelope merge, path.py:166-277) with its
// data-parallel parts on the device (included by l1b200.cu).
//
// The reference walks the K grid intervals in order; per interval it (1)
// applies that weight's breakpoint events -- v_p[t] = val and the column
// error np.abs(X[:, t] - val X[:, p]).sum() --, (2) forms every pivot's line
// z = sum(colerr) + lam_k sum(|v|), (3) runs the O(P^2) crossing analysis,
// (4) picks the minimum line at each sub-interval's probe, (5) opens a
// segment (FittedLine.build: an n x m residual) when the winner changes.
// Here:
//   k_mrg_event_err   (1b) every event's column error at once (NumPy's
//                     pairwise order over n), independent of the walk;
//   k_mrg_pivot_walk  (1a+2) per pivot, its events in grid order over a
//                     shared-memory copy of its colerr / v, recording
//                     (k, sum(colerr), sum(|v|)) -- NumPy's pairwise sums
//                     over m -- at every interval that changes it;
//   k_mrg_intervals   (2-4) a CTA per block of consecutive intervals, pivot
//                     cursors advancing through those change lists: the
//                     candidates' lines, the crossing analysis (thread per
//                     candidate, loop over competitors), the starts sorted
//                     and deduplicated, the probe minimum of every
//                     sub-interval (first strict minimum in pivot order);
// and the host walks the per-interval winners in order, opening segments
// exactly where the reference does (5), their residuals batched on the
// device (l1b_residual_exact_batch).  Every float is produced by the same
// IEEE operations in the same order as the reference (no contraction), so
// segments, lines and objectives are bit-identical.

namespace {

constexpr int kMrgThreads = 256;
constexpr int kMrgBlock = 64;  // consecutive intervals per k_mrg_intervals CTA

// NumPy's pairwise_sum over f(off .. off+cnt-1) (loops_utils.h.src), iterative
// over the recursion's leaves: cnt < 8 sequential; <= 128 eight strided
// accumulators; else split at n/2 rounded down to a multiple of 8 -- the same
// additions in the same order as the recursive form.
template <typename F>
__device__ double np_pairwise_dev(F f, int64_t off, int64_t cnt) {
  // explicit stack of (off, cnt, state) with partial results
  int64_t so[40], sc[40];
  double sr[40];
  int sst[40];
  int top = 0;
  so[0] = off;
  sc[0] = cnt;
  sst[0] = 0;
  double ret = 0.0;
  while (top >= 0) {
    const int64_t o = so[top], c = sc[top];
    if (c <= 128) {
      double r;
      if (c < 8) {
        r = 0.0;
        for (int64_t i = 0; i < c; ++i) r = __dadd_rn(r, f(o + i));
      } else {
        double a[8];
        for (int q = 0; q < 8; ++q) a[q] = f(o + q);
        int64_t i;
        for (i = 8; i < c - (c % 8); i += 8)
          for (int q = 0; q < 8; ++q) a[q] = __dadd_rn(a[q], f(o + i + q));
        r = __dadd_rn(__dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3])),
                      __dadd_rn(__dadd_rn(a[4], a[5]), __dadd_rn(a[6], a[7])));
        for (; i < c; ++i) r = __dadd_rn(r, f(o + i));
      }
      ret = r;
      --top;
      // deliver to the parent
      while (top >= 0) {
        if (sst[top] == 1) {  // left half done: store, descend right
          sr[top] = ret;
          sst[top] = 2;
          int64_t n2 = sc[top] / 2;
          n2 -= n2 % 8;
          ++top;
          so[top] = so[top - 1] + n2;
          sc[top] = sc[top - 1] - n2;
          sst[top] = 0;
          break;
        }
        // right half done
        ret = __dadd_rn(sr[top], ret);
        --top;
      }
      continue;
    }
    // split: descend left
    int64_t n2 = c / 2;
    n2 -= n2 % 8;
    sst[top] = 1;
    ++top;
    so[top] = o;
    sc[top] = n2;
    sst[top] = 0;
  }
  return ret;
}

// (1b) err[e] = sum_i |x_{i,t} - val x_{i,p}| in NumPy's pairwise order over
// the contiguous temporary of n (core.py:93 on one column).  Xc column-major.
// Threads take the events in (pivot, target) order (pord), so a warp's lanes
// read the same two columns in lockstep: every load is a broadcast.
__global__ void k_mrg_event_err(const double* __restrict__ Xc, int64_t n, int64_t E,
                                const int64_t* __restrict__ pord, const int64_t* __restrict__ ep,
                                const int64_t* __restrict__ et, const double* __restrict__ ev,
                                double* __restrict__ err) {
  const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= E) return;
  const int64_t e = pord[x];
  const double* xt = Xc + et[e] * n;
  const double* xp = Xc + ep[e] * n;
  const double val = ev[e];
  err[e] = np_pairwise_dev([&](int64_t i) { return fabs(__dsub_rn(xt[i], __dmul_rn(val, xp[i]))); }, 0, n);
}

// (1a+2) Pivot slot s (a CTA; thread 0 walks): events ord[pe_off[s] ..
// pe_off[s+1]) in grid order.  State (colerr, v) in shared memory when m fits,
// else in the global scratch gst + s * 2m.  Change record c of slot s:
// ch_k / ch_E / ch_S [ch_off[s] + c]; record 0 is the initial state (k = -1).
__global__ void k_mrg_pivot_walk(int64_t m, const int64_t* __restrict__ piv, const double* __restrict__ colsums,
                                 const int64_t* __restrict__ pe_off, const int64_t* __restrict__ ord,
                                 const int64_t* __restrict__ ek, const int64_t* __restrict__ et,
                                 const double* __restrict__ ev, const double* __restrict__ eerr,
                                 const int64_t* __restrict__ ch_off, int64_t* __restrict__ ch_k,
                                 double* __restrict__ ch_E, double* __restrict__ ch_S, double* __restrict__ gst,
                                 int use_smem) {
  extern __shared__ double mst[];
  const int64_t s = blockIdx.x;
  const int64_t p = piv[s];
  double* ce = use_smem ? mst : gst + s * 2 * m;
  double* v = ce + m;
  for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
    ce[j] = j == p ? 0.0 : colsums[j];
    v[j] = j == p ? 1.0 : 0.0;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  auto sums = [&](int64_t at) {
    ch_E[at] = np_pairwise_dev([&](int64_t j) { return ce[j]; }, 0, m);
    ch_S[at] = np_pairwise_dev([&](int64_t j) { return fabs(v[j]); }, 0, m);
  };
  int64_t c = ch_off[s];
  ch_k[c] = -1;
  sums(c);
  ++c;
  for (int64_t i = pe_off[s]; i < pe_off[s + 1];) {
    const int64_t k = ek[ord[i]];
    for (; i < pe_off[s + 1] && ek[ord[i]] == k; ++i) {
      const int64_t e = ord[i];
      v[et[e]] = ev[e];
      ce[et[e]] = eerr[e];
    }
    ch_k[c] = k;
    sums(c);
    ++c;
  }
}

// (2-4) Intervals [k0, k0 + kMrgBlock) per CTA.  Candidates in pivot order:
// the usable pivots' slots and the degenerate pivots merged (cp[] pivot
// index, cs[] slot or -1).  Output: the winner at lam_k (sub-interval 0) in
// win0[k]; further sub-intervals (a, p*) appended to ovf (k, i, a, p) with an
// atomic counter (rare).
__global__ void __launch_bounds__(kMrgThreads) k_mrg_intervals(
    int64_t K, const double* __restrict__ lambdas, int64_t NC, const int64_t* __restrict__ cp,
    const int64_t* __restrict__ cs, const int64_t* __restrict__ ch_off, const int64_t* __restrict__ ch_k,
    const double* __restrict__ ch_E, const double* __restrict__ ch_S, double degen_error, int64_t* __restrict__ win0,
    int64_t* __restrict__ ovf_k, int64_t* __restrict__ ovf_i, double* __restrict__ ovf_a,
    int64_t* __restrict__ ovf_p, unsigned long long* __restrict__ ovf_n, int64_t ovf_cap) {
  extern __shared__ __align__(8) unsigned char msm[];
  double* z = (double*)msm;            // [NC]
  double* sl = z + NC;                 // [NC]
  double* st = sl + NC;                // [NC] starts
  int64_t* cur = (int64_t*)(st + NC);  // [NC] change cursors
  double* bnd = (double*)(cur + NC);   // [NC + 1] sub-interval bounds
  __shared__ int nst;
  __shared__ int nb;
  __shared__ unsigned long long bestkey[kMrgThreads / 32];
  __shared__ double bestz[kMrgThreads / 32];
  const int tid = threadIdx.x;
  const int64_t k0 = (int64_t)blockIdx.x * kMrgBlock, k1 = min(K, k0 + kMrgBlock);
  // cursors: the last change with k <= k0 (binary search), then stepped
  for (int64_t c = tid; c < NC; c += blockDim.x) {
    if (cs[c] < 0) {
      cur[c] = -1;
      continue;
    }
    int64_t a = ch_off[cs[c]], b = ch_off[cs[c] + 1] - 1;  // ch_k[a] = -1 <= k0
    while (a < b) {
      const int64_t mid = (a + b + 1) >> 1;
      if (ch_k[mid] <= k0) a = mid;
      else b = mid - 1;
    }
    cur[c] = a;
  }
  __syncthreads();
  for (int64_t k = k0; k < k1; ++k) {
    const double lam_k = lambdas[k];
    const double lam_next = k + 1 < K ? lambdas[k + 1] : INFINITY;
    for (int64_t c = tid; c < NC; c += blockDim.x) {
      if (cs[c] < 0) {
        z[c] = degen_error;
        sl[c] = 0.0;
        continue;
      }
      int64_t a = cur[c];
      const int64_t end = ch_off[cs[c] + 1];
      while (a + 1 < end && ch_k[a + 1] <= k) ++a;
      cur[c] = a;
      const double S = ch_S[a];
      z[c] = __dadd_rn(ch_E[a], __dmul_rn(lam_k, S));
      sl[c] = S;
    }
    if (tid == 0) nst = 0;
    __syncthreads();
    // crossing analysis (path.py:223-240)
    for (int64_t c = tid; c < NC; c += blockDim.x) {
      const double zp = z[c], sp = sl[c];
      // four competitors per step with their own running extrema (max / min
      // are exact, so splitting the reduction changes nothing)
      double blo4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY}, bhi4[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
      bool dom = false;
      for (int64_t q0 = 0; q0 < NC && !dom; q0 += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t q = q0 + u;
          if (q >= NC || q == c) continue;
          const double zq = z[q], sq = sl[q];
          const double ds = __dsub_rn(sq, sp);
          if (fabs(ds) <= 1e-9 * fmax(fmax(1.0, sp), sq)) {
            dom |= zp > zq;
          } else if (sq > sp) {
            blo4[u] = fmax(blo4[u], __ddiv_rn(__dsub_rn(zp, zq), ds));
          } else {
            bhi4[u] = fmin(bhi4[u], __ddiv_rn(__dsub_rn(zq, zp), __dsub_rn(sp, sq)));
          }
        }
      }
      const double blo = fmax(fmax(blo4[0], blo4[1]), fmax(blo4[2], blo4[3]));
      const double bhi = fmin(fmin(bhi4[0], bhi4[1]), fmin(bhi4[2], bhi4[3]));
      // starts within DEDUP_TOL of lam_k (the elif branch's lam_k itself, always)
      // or of lam_next never survive the dedup walk below -- the sorted walk
      // drops them whatever else is kept -- so only the others are collected
      if (!dom && 0.0 < blo && blo < bhi) {
        const double b0 = __dadd_rn(lam_k, blo);
        if (b0 <= lam_next && __dsub_rn(b0, lam_k) > 1e-9 && __dsub_rn(lam_next, b0) > 1e-9) st[atomicAdd(&nst, 1)] = b0;
      }
    }
    __syncthreads();
    if (tid == 0) {  // sorted(starts), then the dedup walk (path.py:242-245)
      const int ns = nst;
      for (int i = 1; i < ns; ++i) {  // insertion sort (few starts per interval)
        const double x = st[i];
        int j = i - 1;
        while (j >= 0 && st[j] > x) {
          st[j + 1] = st[j];
          --j;
        }
        st[j + 1] = x;
      }
      int b = 1;
      bnd[0] = lam_k;
      for (int i = 0; i < ns; ++i)
        if (__dsub_rn(st[i], bnd[b - 1]) > 1e-9 && __dsub_rn(lam_next, st[i]) > 1e-9) bnd[b++] = st[i];
      nb = b;
    }
    __syncthreads();
    // the minimum line at each sub-interval's probe: first strict minimum in
    // candidate (pivot) order -> key (z, c) lexicographic
    for (int i = 0; i < nb; ++i) {
      const double a = bnd[i];
      const double b = i + 1 < nb ? bnd[i + 1] : lam_next;
      const double probe = isinf(b) ? __dadd_rn(a, 1.0) : __dmul_rn(0.5, __dadd_rn(a, b));
      const double dp = __dsub_rn(probe, lam_k);
      double bz = INFINITY;
      long long bc = -1;
      for (int64_t c = tid; c < NC; c += blockDim.x) {
        const double zc = __dadd_rn(z[c], __dmul_rn(dp, sl[c]));
        if (bc < 0 || zc < bz) {
          bz = zc;
          bc = c;
        }
      }
      // warp then block reduction, ties -> smaller candidate index
      for (int o = 16; o; o >>= 1) {
        const double oz = __shfl_xor_sync(0xffffffffu, bz, o);
        const long long oc = __shfl_xor_sync(0xffffffffu, bc, o);
        if (oc >= 0 && (bc < 0 || oz < bz || (oz == bz && oc < bc))) {
          bz = oz;
          bc = oc;
        }
      }
      if ((tid & 31) == 0) {
        bestz[tid >> 5] = bz;
        bestkey[tid >> 5] = (unsigned long long)bc;
      }
      __syncthreads();
      if (tid == 0) {
        double z0 = INFINITY;
        long long c0 = -1;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
          const long long oc = (long long)bestkey[w];
          const double oz = bestz[w];
          if (oc >= 0 && (c0 < 0 || oz < z0 || (oz == z0 && oc < c0))) {
            z0 = oz;
            c0 = oc;
          }
        }
        if (i == 0) {
          win0[k] = c0;
        } else {
          const unsigned long long at = atomicAdd(ovf_n, 1ull);
          if ((int64_t)at < ovf_cap) {
            ovf_k[at] = k;
            ovf_i[at] = i;
            ovf_a[at] = a;
            ovf_p[at] = c0;
          }
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace

namespace {

// np.abs(X).sum(axis=0) of a C-contiguous X: rows accumulated in order.
__global__ void k_mrg_colsums(const double* __restrict__ X, int64_t n, int64_t m, double* __restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double a = 0.0;
  for (int64_t i = 0; i < n; ++i) a = __dadd_rn(a, fabs(X[i * m + j]));
  out[j] = a;
}

template <typename T>
struct DevBuf {  // stream-ordered scratch owned by one l1b_merge_path_device call
  T* p = nullptr;
  cudaStream_t s;
  explicit DevBuf(cudaStream_t st) : s(st) {}
  cudaError_t alloc(size_t n) { return cudaMallocAsync((void**)&p, sizeof(T) * (n ? n : 1), s); }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

}  // namespace

extern "C" {

int l1b_merge_path_device(const double* d_X, int64_t n, int64_t m, const double* lambdas, int64_t K,
                          const int64_t* piv, int64_t np_, const int64_t* deg, int64_t nd, const int64_t* ev_off,
                          const int64_t* ev_p, const int64_t* ev_t, const double* ev_v, double** o_seg,
                          int64_t* count, void* d_ws, size_t ws_bytes, void* stream) {
  if (!d_X || !lambdas || K < 1 || n < 1 || m < 2 || !count || !o_seg || np_ + nd < 1) return L1B_EINVAL;
  *o_seg = nullptr;
  const bool timing = getenv("L1B200_MERGE_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!timing) return;
    cudaStreamSynchronize((cudaStream_t)stream);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "merge_path_device %-28s %9.3f ms\n", what,
            std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  Workspace w;
  const int64_t wcap = ws_capacity(n, m, ws_bytes);
  if (wcap < 1) return L1B_ENOMEM;
  carve(&w, d_ws, n, m, wcap);
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t E = ev_off[K];
  std::vector<int64_t> slot_of(m, -1);
  for (int64_t k = 0; k < np_; ++k) slot_of[piv[k]] = k;
  for (int64_t e = 0; e < E; ++e)
    if (ev_p[e] < 0 || ev_p[e] >= m || slot_of[ev_p[e]] < 0 || ev_t[e] < 0 || ev_t[e] >= m) return L1B_EINVAL;
  // event grid index; events of each slot in grid order (a stable counting sort)
  std::vector<int64_t> ek(E), pe_off(np_ + 1, 0), ord(E), ch_off(np_ + 1, 0);
  for (int64_t k = 0; k < K; ++k)
    for (int64_t e = ev_off[k]; e < ev_off[k + 1]; ++e) ek[e] = k;
  for (int64_t e = 0; e < E; ++e) ++pe_off[slot_of[ev_p[e]] + 1];
  for (int64_t q = 0; q < np_; ++q) pe_off[q + 1] += pe_off[q];
  {
    std::vector<int64_t> at(pe_off.begin(), pe_off.end() - 1);
    std::vector<int64_t> lastk(np_, -1);
    for (int64_t e = 0; e < E; ++e) {
      const int64_t q = slot_of[ev_p[e]];
      ord[at[q]++] = e;
      if (ek[e] != lastk[q]) {
        lastk[q] = ek[e];
        ++ch_off[q + 1];
      }
    }
  }
  for (int64_t q = 0; q < np_; ++q) ch_off[q + 1] += ch_off[q] + 1;  // + the initial state
  // events in (pivot slot, target) order for the column-error kernel
  std::vector<int64_t> pord(E);
  {
    std::vector<int64_t> cnt((size_t)np_ * m + 1, 0);
    for (int64_t e = 0; e < E; ++e) ++cnt[(size_t)slot_of[ev_p[e]] * m + ev_t[e] + 1];
    for (size_t b = 1; b < cnt.size(); ++b) cnt[b] += cnt[b - 1];
    for (int64_t e = 0; e < E; ++e) pord[cnt[(size_t)slot_of[ev_p[e]] * m + ev_t[e]]++] = e;
  }
  const int64_t NCH = ch_off[np_];
  // candidates in pivot order (path.py:215-218)
  std::vector<int64_t> cp, cs;
  {
    int64_t a = 0, b = 0;
    while (a < np_ || b < nd) {
      if (b >= nd || (a < np_ && piv[a] < deg[b])) {
        cp.push_back(piv[a]);
        cs.push_back(a++);
      } else {
        cp.push_back(deg[b++]);
        cs.push_back(-1);
      }
    }
  }
  const int64_t NC = (int64_t)cp.size();
  mark("host prep");
  DevBuf<int64_t> d_ep(s), d_et(s), d_ek(s), d_ord(s), d_pord(s), d_peoff(s), d_choff(s), d_chk(s), d_piv(s), d_cp(s), d_cs(s),
      d_win(s), d_ok(s), d_oi(s), d_op(s);
  DevBuf<double> d_ev(s), d_err(s), d_chE(s), d_chS(s), d_col(s), d_lam(s), d_gst(s), d_oa(s), d_V(s), d_segerr(s);
  DevBuf<unsigned long long> d_on(s);
  const int64_t ovf_cap = std::max<int64_t>(1024, K / 4);
  cudaError_t ce = cudaSuccess;
  auto chk = [&](cudaError_t e) {
    if (ce == cudaSuccess) ce = e;
  };
  chk(d_ep.alloc(E));
  chk(d_et.alloc(E));
  chk(d_ek.alloc(E));
  chk(d_ev.alloc(E));
  chk(d_err.alloc(E));
  chk(d_ord.alloc(E));
  chk(d_pord.alloc(E));
  chk(d_peoff.alloc(np_ + 1));
  chk(d_choff.alloc(np_ + 1));
  chk(d_chk.alloc(NCH));
  chk(d_chE.alloc(NCH));
  chk(d_chS.alloc(NCH));
  chk(d_piv.alloc(np_));
  chk(d_col.alloc(m));
  chk(d_lam.alloc(K));
  chk(d_cp.alloc(NC));
  chk(d_cs.alloc(NC));
  chk(d_win.alloc(K));
  chk(d_ok.alloc(ovf_cap));
  chk(d_oi.alloc(ovf_cap));
  chk(d_oa.alloc(ovf_cap));
  chk(d_op.alloc(ovf_cap));
  chk(d_on.alloc(1));
  if (ce != cudaSuccess) return L1B_ENOMEM;
  auto up = [&](void* dst, const void* src, size_t bytes) {
    if (bytes) chk(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
  };
  up(d_ep.p, ev_p, 8 * E);
  up(d_et.p, ev_t, 8 * E);
  up(d_ev.p, ev_v, 8 * E);
  up(d_ek.p, ek.data(), 8 * E);
  up(d_ord.p, ord.data(), 8 * E);
  up(d_pord.p, pord.data(), 8 * E);
  up(d_peoff.p, pe_off.data(), 8 * (np_ + 1));
  up(d_choff.p, ch_off.data(), 8 * (np_ + 1));
  up(d_piv.p, piv, 8 * np_);
  up(d_lam.p, lambdas, 8 * K);
  up(d_cp.p, cp.data(), 8 * NC);
  up(d_cs.p, cs.data(), 8 * NC);
  chk(cudaMemsetAsync(d_on.p, 0, 8, s));
  if (ce != cudaSuccess) return L1B_ECUDA;
  mark("uploads");
  count_launch(4);
  k_mrg_colsums<<<(unsigned)((m + 127) / 128), 128, 0, s>>>(d_X, n, m, d_col.p);
  if (E)
    k_mrg_event_err<<<(unsigned)((E + 127) / 128), 128, 0, s>>>(w.xc, n, E, d_pord.p, d_ep.p, d_et.p, d_ev.p, d_err.p);
  const bool use_smem = 2 * m * 8 <= 96 * 1024;
  if (!use_smem) {
    chk(d_gst.alloc((size_t)2 * m * np_));
  } else {
    chk(cudaFuncSetAttribute(k_mrg_pivot_walk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(2 * m * 8)));
  }
  if (np_)
    k_mrg_pivot_walk<<<(unsigned)np_, 128, use_smem ? 2 * m * 8 : 0, s>>>(
        m, d_piv.p, d_col.p, d_peoff.p, d_ord.p, d_ek.p, d_et.p, d_ev.p, d_err.p, d_choff.p, d_chk.p, d_chE.p,
        d_chS.p, d_gst.p, use_smem ? 1 : 0);
  mark("event errors + pivot walks");
  // degen_error = np.abs(X).sum() (path.py:190): residual_error with v = 0
  double degen_error = 0.0;
  if (nd) {
    DevBuf<double> d_zero(s), d_de(s);
    chk(d_zero.alloc(m));
    chk(d_de.alloc(1));
    chk(cudaMemsetAsync(d_zero.p, 0, 8 * m, s));
    if (ce != cudaSuccess) return L1B_ECUDA;
    const int64_t p0 = 0;
    int st = l1b_residual_exact_batch(d_X, n, m, d_zero.p, m, &p0, 1, d_de.p, d_ws, ws_bytes, stream);
    if (st != L1B_OK) return st;
    chk(cudaMemcpyAsync(&degen_error, d_de.p, 8, cudaMemcpyDeviceToHost, s));
    chk(cudaStreamSynchronize(s));
  }
  const size_t sm = (size_t)NC * (3 * sizeof(double) + sizeof(int64_t)) + (size_t)(NC + 1) * sizeof(double);
  chk(cudaFuncSetAttribute(k_mrg_intervals, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  if (ce != cudaSuccess) return L1B_ECUDA;
  k_mrg_intervals<<<(unsigned)((K + kMrgBlock - 1) / kMrgBlock), kMrgThreads, sm, s>>>(
      K, d_lam.p, NC, d_cp.p, d_cs.p, d_choff.p, d_chk.p, d_chE.p, d_chS.p, degen_error, d_win.p, d_ok.p, d_oi.p,
      d_oa.p, d_op.p, d_on.p, ovf_cap);
  chk(cudaGetLastError());
  mark("intervals");
  std::vector<int64_t> win(K);
  unsigned long long novf = 0;
  chk(cudaMemcpyAsync(win.data(), d_win.p, 8 * K, cudaMemcpyDeviceToHost, s));
  chk(cudaMemcpyAsync(&novf, d_on.p, 8, cudaMemcpyDeviceToHost, s));
  chk(cudaStreamSynchronize(s));
  if (ce != cudaSuccess) return L1B_ECUDA;
  if ((int64_t)novf > ovf_cap) return L1B_EINTERNAL;  // more sub-intervals than the overflow list holds
  std::vector<int64_t> ok(novf), oi(novf), op(novf);
  std::vector<double> oa(novf);
  if (novf) {
    chk(cudaMemcpyAsync(ok.data(), d_ok.p, 8 * novf, cudaMemcpyDeviceToHost, s));
    chk(cudaMemcpyAsync(oi.data(), d_oi.p, 8 * novf, cudaMemcpyDeviceToHost, s));
    chk(cudaMemcpyAsync(oa.data(), d_oa.p, 8 * novf, cudaMemcpyDeviceToHost, s));
    chk(cudaMemcpyAsync(op.data(), d_op.p, 8 * novf, cudaMemcpyDeviceToHost, s));
    chk(cudaStreamSynchronize(s));
    if (ce != cudaSuccess) return L1B_ECUDA;
  }
  std::vector<int64_t> oidx(novf);
  for (size_t i = 0; i < novf; ++i) oidx[i] = (int64_t)i;
  std::sort(oidx.begin(), oidx.end(), [&](int64_t a, int64_t b) { return ok[a] != ok[b] ? ok[a] < ok[b] : oi[a] < oi[b]; });
  // (5) the sequential walk: segments open where the winner's line changes
  std::vector<std::vector<double>> V(np_, std::vector<double>(m, 0.0));
  std::vector<int64_t> ver(np_, 0);
  for (int64_t q = 0; q < np_; ++q) V[q][piv[q]] = 1.0;
  std::vector<double> zero(m, 0.0);
  struct Seg {
    double lo, hi;
    int64_t pivot, slot, ver;
    std::vector<double> v;
  };
  std::vector<Seg> segs;
  bool open = false;
  size_t oc = 0;
  auto consider = [&](double a, int64_t c) {
    const int64_t p = cp[c], q = cs[c];
    const std::vector<double>& vs = q >= 0 ? V[q] : zero;
    if (open) {
      Seg& o = segs.back();
      if (o.pivot == p && (q < 0 || o.ver == ver[q] || o.v == vs)) return;
      o.hi = a;
    }
    segs.push_back({a, INFINITY, p, q, q >= 0 ? ver[q] : 0, vs});
    open = true;
  };
  for (int64_t k = 0; k < K; ++k) {
    for (int64_t e = ev_off[k]; e < ev_off[k + 1]; ++e) {
      const int64_t q = slot_of[ev_p[e]];
      V[q][ev_t[e]] = ev_v[e];
      ver[q] = k + 1;
    }
    consider(lambdas[k], win[k]);
    for (; oc < novf && ok[oidx[oc]] == k; ++oc) consider(oa[oidx[oc]], op[oidx[oc]]);
  }
  mark("downloads + host walk");
  const int64_t S = (int64_t)segs.size();
  *count = S;
  // the segments: one malloc'ed block [S][8 + m] (lo, hi, pivot, err, pen,
  // obj, z_lo, z_hi, v[m]), freed by the caller with l1b_csv_free
  const int64_t rec = 8 + m;
  double* out = (double*)malloc(sizeof(double) * (size_t)std::max<int64_t>(1, S) * rec);
  if (!out) return L1B_ENOMEM;
  // FittedLine.build of every segment line: residuals batched on the device
  std::vector<double> Vh((size_t)S * m);
  std::vector<int64_t> sp(S);
  for (int64_t i = 0; i < S; ++i) {
    std::memcpy(Vh.data() + (size_t)i * m, segs[i].v.data(), 8 * m);
    sp[i] = segs[i].pivot;
  }
  std::vector<double> errs(S);
  chk(d_V.alloc((size_t)S * m));
  chk(d_segerr.alloc(S));
  if (ce == cudaSuccess) up(d_V.p, Vh.data(), 8 * (size_t)S * m);
  int st = ce == cudaSuccess ? l1b_residual_exact_batch(d_X, n, m, d_V.p, m, sp.data(), S, d_segerr.p, d_ws, ws_bytes,
                                                          stream)
                             : L1B_ECUDA;
  if (st == L1B_OK) {
    chk(cudaMemcpyAsync(errs.data(), d_segerr.p, 8 * S, cudaMemcpyDeviceToHost, s));
    chk(cudaStreamSynchronize(s));
    if (ce != cudaSuccess) st = L1B_ECUDA;
  }
  if (st != L1B_OK) {
    free(out);
    return st;
  }
  mark("segment residuals");
  for (int64_t i = 0; i < S; ++i) {
    const Seg& g = segs[i];
    const double err = errs[i];
    const double pen = np_pairwise_f([&](int64_t j) { return fabs(g.v[j]); }, 0, m);
    const double obj = err + g.lo * pen;
    double* r = out + (size_t)i * rec;
    r[0] = g.lo;
    r[1] = g.hi;
    r[2] = (double)g.pivot;
    r[3] = err;
    r[4] = pen;
    r[5] = obj;
    r[6] = obj;
    r[7] = std::isinf(g.hi) ? (pen > 0.0 ? INFINITY : err) : err + g.hi * pen;
    std::memcpy(r + 8, g.v.data(), 8 * m);
  }
  *o_seg = out;
  mark("outputs");
  return L1B_OK;
}

}  // extern "C"

extern "C" {

// path.py:157-163 for every event at once, grouped for the merge: event e's
// breakpoint bp[e] snaps to the grid index k of lambdas[K] (ascending) with
// |lambdas[k] - bp| <= tol (the left searchsorted position, else the one
// before); out_order lists the events grouped by k, insertion order kept
// within a group, and out_off[K+1] the groups' offsets.  Host code: an LSD
// radix sort of the breakpoints, one merge sweep against the grid, a stable
// counting sort by k (numpy's searchsorted on unsorted queries + argsort
// took 15 s for 22 M events).  L1B_EINTERNAL if a breakpoint is off the grid.
int l1b_snap_events(const double* lambdas, int64_t K, const double* bp, int64_t E, double tol, int64_t* out_order,
                    int64_t* out_off) {
  if (!lambdas || K < 1 || (E > 0 && (!bp || !out_order)) || !out_off) return L1B_EINVAL;
  std::vector<uint64_t> key(E);
  std::vector<int64_t> idx(E), tmp_i(E);
  std::vector<uint64_t> tmp_k(E);
  const int NT = (int)std::max<int64_t>(1, std::min<int64_t>(std::thread::hardware_concurrency(), E / 65536));
  auto par = [&](auto&& fn) {  // fn(t, lo, hi) over NT contiguous slices of [0, E)
    std::vector<std::thread> th;
    for (int t = 0; t < NT; ++t) th.emplace_back([&, t] { fn(t, E * t / NT, E * (t + 1) / NT); });
    for (auto& x : th) x.join();
  };
  par([&](int, int64_t lo, int64_t hi) {
    for (int64_t e = lo; e < hi; ++e) {
      uint64_t b;
      const double x = bp[e] == 0.0 ? 0.0 : bp[e];  // -0.0 sorts with +0.0
      std::memcpy(&b, &x, 8);
      key[e] = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // order-preserving image of the double
      idx[e] = e;
    }
  });
  // LSD radix sort, 16-bit digits, stable; each pass: per-slice digit counts,
  // an exclusive scan over (digit, slice), parallel scatter
  std::vector<int64_t> cnt((size_t)NT * 65536);
  for (int pass = 0; pass < 4; ++pass) {
    const int sh = 16 * pass;
    std::fill(cnt.begin(), cnt.end(), 0);
    par([&](int t, int64_t lo, int64_t hi) {
      int64_t* c = cnt.data() + (size_t)t * 65536;
      for (int64_t e = lo; e < hi; ++e) ++c[(key[e] >> sh) & 0xffff];
    });
    int64_t run = 0;
    for (int d = 0; d < 65536; ++d)
      for (int t = 0; t < NT; ++t) {
        const int64_t v = cnt[(size_t)t * 65536 + d];
        cnt[(size_t)t * 65536 + d] = run;
        run += v;
      }
    par([&](int t, int64_t lo, int64_t hi) {
      int64_t* c = cnt.data() + (size_t)t * 65536;
      for (int64_t e = lo; e < hi; ++e) {
        const int64_t at = c[(key[e] >> sh) & 0xffff]++;
        tmp_k[at] = key[e];
        tmp_i[at] = idx[e];
      }
    });
    key.swap(tmp_k);
    idx.swap(tmp_i);
  }
  std::vector<int64_t> kk(E);
  int64_t i = 0;
  for (int64_t r = 0; r < E; ++r) {
    const int64_t e = idx[r];
    const double b = bp[e];
    while (i < K && lambdas[i] < b) ++i;  // np.searchsorted(..., side="left")
    int64_t k;
    if (i < K && fabs(lambdas[i] - b) <= tol) k = i;
    else if (i > 0 && fabs(lambdas[i - 1] - b) <= tol) k = i - 1;
    else return L1B_EINTERNAL;
    kk[e] = k;
  }
  std::fill(out_off, out_off + K + 1, 0);
  for (int64_t e = 0; e < E; ++e) ++out_off[kk[e] + 1];
  for (int64_t k = 0; k < K; ++k) out_off[k + 1] += out_off[k];
  std::vector<int64_t> at(out_off, out_off + K);
  for (int64_t e = 0; e < E; ++e) out_order[at[kk[e]]++] = e;
  return L1B_OK;
}

}  // extern "C"
