// path.cuh -- Algorithm 2 (per-pivot breakpoints) on the device (included
// by l1b200.cu after select.cuh).
//
// pivot_breakpoints (path.py:76-102) needs, for one pivot p and every target
// j != p, the column of the sorted tableau (ratios.py:109-135): the ratios
// x_ij / x_ip of the rows with x_ip != 0 in stable (ratio, row) order, their
// weights |x_ip|, the sequential prefix sums P_k (np.cumsum), and
//   center_k = (T - P_k) - P_{k-1},  start_k = sgn(r_k) center_k - w_k,
//   right_k  = start_k + 2 w_k        (sgn(r) = +1 iff r >= 0.0).
// k_breakpoints does one target column per CTA: exact ratios (the hoisted
// division, bit-identical to IEEE division) keyed by (key64, row), a bitonic
// sort of the column in shared memory, then the prefix walk in order by one
// thread (sequential, so the sums round exactly as np.cumsum's do).  The host
// keeps the live runs (right > 0) and builds the entry tuples.

constexpr int kBpThreads = 1024;
constexpr int64_t kBpMaxRows = 16384;  // nonzero rows of the pivot a CTA can sort in shared memory

// TAB: the tableau column itself (pivot_tableau, ratios.py:109-135) instead
// of the runs: rs = sorted ratios, st = weights, rt = inclusive prefix
// (np.cumsum), rows = source rows.  Columns c0 + blockIdx.x of the pivot's
// targets (j != p), written at output column blockIdx.x.
__device__ __forceinline__ void bp_emit(bool tab, double ratio, double w, double Pk, double T, double Pp, int r,
                                        int64_t o, double* rs, double* st, double* rt, int64_t* rows) {
  if (tab) {
    rs[o] = ratio;
    st[o] = w;
    rt[o] = Pk;
    rows[o] = r;
  } else {
    const double center = __dsub_rn(__dsub_rn(T, Pk), Pp);
    const double s = __dsub_rn(ratio >= 0.0 ? center : -center, w);
    rs[o] = ratio;
    rt[o] = __dadd_rn(s, __dmul_rn(2.0, w));
    st[o] = s;  // last: the tall walk's rows share st's storage (see k_bp_tall_walk)
  }
}

template <bool SAFE>
__global__ void __launch_bounds__(kBpThreads) k_breakpoints(SelParams P, int64_t p, int64_t np2, int64_t ld,
                                                            double* __restrict__ rs, double* __restrict__ st,
                                                            double* __restrict__ rt, int64_t c0, int tab,
                                                            int64_t* __restrict__ rows_out) {
  extern __shared__ __align__(16) unsigned char psm[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(psm);
  int* row = reinterpret_cast<int*>(psm + np2 * sizeof(unsigned long long));
  __shared__ int cnt_s;
  const int tid = threadIdx.x;
  const int64_t n = P.n;
  const int64_t c = blockIdx.x;           // output column
  const int64_t cj = c0 + c;              // target column index among j != p
  const int64_t j = cj < p ? cj : cj + 1;
  const double* xc = P.Xc + j * n;
  const double* pb = P.pb + p * P.np;
  const double* py = P.py + p * P.np;
  if (tid == 0) cnt_s = 0;
  __syncthreads();
  // compact the rows with x_ip != 0 in row order (ratios.py:115): a block-wide
  // ordered compaction, 1024 rows at a time
  __shared__ int wsum[kBpThreads / 32];
  int base = 0;
  for (int64_t i0 = 0; i0 < n; i0 += kBpThreads) {
    const int64_t i = i0 + tid;
    const bool nz = i < n && pb[i] != 0.0;
    const unsigned bal = __ballot_sync(0xffffffffu, nz);
    const int w = tid >> 5, l = tid & 31;
    if (l == 0) wsum[w] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
    for (int k = 0; k < kBpThreads / 32; ++k) {
      off += k < w ? wsum[k] : 0;
      tot += wsum[k];
    }
    if (nz) {
      const int pos = base + off + __popc(bal & ((1u << l) - 1));
      key[pos] = key64(sratio<SAFE>(P, xc[i], pb[i], py[i]));
      row[pos] = (int)i;
    }
    base += tot;
    __syncthreads();
  }
  const int cnt = base;
  for (int64_t e = cnt + tid; e < np2; e += kBpThreads) {
    key[e] = ~0ULL;
    row[e] = 0x7fffffff;
  }
  __syncthreads();
  // stable order = ascending (key, row) (np.argsort(kind="stable"), +-0 tied)
  for (int64_t kq = 2; kq <= np2; kq <<= 1) {
    for (int64_t jq = kq >> 1; jq > 0; jq >>= 1) {
      for (int64_t e = tid; e < np2; e += kBpThreads) {
        const int64_t l = e ^ jq;
        if (l > e) {
          const unsigned long long ka = key[e], kb = key[l];
          const int ra = row[e], rb = row[l];
          const bool gt = ka > kb || (ka == kb && ra > rb);
          if (gt == ((e & kq) == 0)) {
            key[e] = kb;
            key[l] = ka;
            row[e] = rb;
            row[l] = ra;
          }
        }
      }
      __syncthreads();
    }
  }
  // the tableau's column totals first (T = P_last, ratios.py:124,134)
  __shared__ double Tsh;
  if (tid == 0) {
    double P = 0.0;
    for (int k = 0; k < cnt; ++k) P = __dadd_rn(P, fabs(pb[row[k]]));
    Tsh = P;
  }
  __syncthreads();
  // the per-position runs (path.py:86-89), in sorted order
  if (tid == 0) {
    const double T = Tsh;
    double Pp = 0.0;  // prefix_prev
    for (int k = 0; k < cnt; ++k) {
      const int r = row[k];
      const double w = fabs(pb[r]);
      const double Pk = __dadd_rn(Pp, w);
      double ratio = sratio<SAFE>(P, xc[r], pb[r], py[r]);
      if (ratio == 0.0) ratio = __ddiv_rn(xc[r], pb[r]);  // the zero's sign (the hoisted path may drop it)
      bp_emit(tab, ratio, w, Pk, T, Pp, r, c * ld + k, rs, st, rt, rows_out);
      Pp = Pk;
    }
  }
}

// ---- pivots with more than kBpMaxRows nonzero rows (tall data, C4) ----
//
// The same column, sorted in global memory with the caller's output arrays
// as scratch (column c: keys in rs, rows as int32 in the second half of st,
// a ping-pong key buffer in rt and row buffer in st's first half):
// k_bp_tall_keys compacts the rows and sorts chunks of kBpMaxRows in shared
// memory, k_bp_merge merges sorted runs pairwise (merge path: every thread
// finds its output segment's split by binary search and merges it
// sequentially), k_bp_tall_walk is the prefix walk of k_breakpoints in
// sorted order.  Ties in the key are broken by row, as the stable argsort.

__device__ __forceinline__ bool bp_less(unsigned long long ka, int ra, unsigned long long kb, int rb) {
  return ka < kb || (ka == kb && ra < rb);
}

template <bool SAFE>
__global__ void __launch_bounds__(kBpThreads) k_bp_tall_keys(SelParams P, int64_t p, int64_t ld,
                                                             double* __restrict__ rs, double* __restrict__ st,
                                                             int64_t c0) {
  extern __shared__ __align__(16) unsigned char psm[];
  unsigned long long* key = reinterpret_cast<unsigned long long*>(psm);
  int* row = reinterpret_cast<int*>(psm + kBpMaxRows * sizeof(unsigned long long));
  __shared__ int wsum[kBpThreads / 32];
  const int tid = threadIdx.x;
  const int64_t n = P.n;
  const int64_t c = blockIdx.x, cj = c0 + c;
  const int64_t j = cj < p ? cj : cj + 1;
  const double* xc = P.Xc + j * n;
  const double* pb = P.pb + p * P.np;
  const double* py = P.py + p * P.np;
  unsigned long long* gk = reinterpret_cast<unsigned long long*>(rs + c * ld);
  int* gr = reinterpret_cast<int*>(st + c * ld) + ld;  // rows, buffer A
  int base = 0;
  for (int64_t i0 = 0; i0 < n; i0 += kBpThreads) {  // ordered compaction (ratios.py:115)
    const int64_t i = i0 + tid;
    const bool nz = i < n && pb[i] != 0.0;
    const unsigned bal = __ballot_sync(0xffffffffu, nz);
    const int w = tid >> 5, l = tid & 31;
    if (l == 0) wsum[w] = __popc(bal);
    __syncthreads();
    int off = 0, tot = 0;
    for (int k = 0; k < kBpThreads / 32; ++k) {
      off += k < w ? wsum[k] : 0;
      tot += wsum[k];
    }
    if (nz) {
      const int pos = base + off + __popc(bal & ((1u << l) - 1));
      gk[pos] = key64(sratio<SAFE>(P, xc[i], pb[i], py[i]));
      gr[pos] = (int)i;
    }
    base += tot;
    __syncthreads();
  }
  const int cnt = base;
  // sort every chunk of kBpMaxRows in shared memory (bitonic, padded)
  for (int c0 = 0; c0 < cnt; c0 += (int)kBpMaxRows) {
    const int len = min((int)kBpMaxRows, cnt - c0);
    for (int e = tid; e < (int)kBpMaxRows; e += kBpThreads) {
      key[e] = e < len ? __ldcg(gk + c0 + e) : ~0ULL;
      row[e] = e < len ? __ldcg(gr + c0 + e) : 0x7fffffff;
    }
    __syncthreads();
    for (int kq = 2; kq <= (int)kBpMaxRows; kq <<= 1) {
      for (int jq = kq >> 1; jq > 0; jq >>= 1) {
        for (int e = tid; e < (int)kBpMaxRows; e += kBpThreads) {
          const int l = e ^ jq;
          if (l > e) {
            const unsigned long long ka = key[e], kb = key[l];
            const int ra = row[e], rb = row[l];
            if (bp_less(kb, rb, ka, ra) == ((e & kq) == 0)) {
              key[e] = kb;
              key[l] = ka;
              row[e] = rb;
              row[l] = ra;
            }
          }
        }
        __syncthreads();
      }
    }
    for (int e = tid; e < len; e += kBpThreads) {
      gk[c0 + e] = key[e];
      gr[c0 + e] = row[e];
    }
    __syncthreads();
  }
}

// Merge the sorted runs of width W pairwise (run 2a with run 2a + 1) from
// buffer `from` (0 = A: keys rs, rows st[ld..]; 1 = B: keys rt, rows st[0..]).
__global__ void __launch_bounds__(kBpThreads) k_bp_merge(int64_t cnt, int64_t ld, int64_t W, int from,
                                                         double* __restrict__ rs, double* __restrict__ st,
                                                         double* __restrict__ rt) {
  const int64_t c = blockIdx.x;
  int* rows = reinterpret_cast<int*>(st + c * ld);
  const unsigned long long* sk = reinterpret_cast<const unsigned long long*>((from ? rt : rs) + c * ld);
  unsigned long long* dk = reinterpret_cast<unsigned long long*>((from ? rs : rt) + c * ld);
  const int* sr = rows + (from ? 0 : ld);
  int* dr = rows + (from ? ld : 0);
  for (int64_t a0 = 0; a0 < cnt; a0 += 2 * W) {
    const int64_t na = min(W, cnt - a0), nb = max((int64_t)0, min(W, cnt - a0 - W));
    const unsigned long long* ka = sk + a0;
    const unsigned long long* kb = sk + a0 + na;
    const int* ra = sr + a0;
    const int* rb = sr + a0 + na;
    const int64_t tot = na + nb;
    const int64_t d0 = tot * threadIdx.x / kBpThreads, d1 = tot * (threadIdx.x + 1) / kBpThreads;
    // co-rank: the number of A elements among the first d outputs
    auto corank = [&](int64_t d) {
      int64_t lo = max((int64_t)0, d - nb), hi = min(d, na);
      while (lo < hi) {
        const int64_t i = (lo + hi) >> 1;  // A[i] vs B[d - i - 1]
        if (bp_less(ka[i], ra[i], kb[d - i - 1], rb[d - i - 1])) lo = i + 1;
        else hi = i;
      }
      return lo;
    };
    int64_t i = corank(d0), k = d0 - i;
    for (int64_t d = d0; d < d1; ++d) {
      const bool takeA = k >= nb || (i < na && bp_less(ka[i], ra[i], kb[k], rb[k]));
      if (takeA) {
        dk[a0 + d] = ka[i];
        dr[a0 + d] = ra[i];
        ++i;
      } else {
        dk[a0 + d] = kb[k];
        dr[a0 + d] = rb[k];
        ++k;
      }
    }
  }
}

// k_breakpoints' prefix walk over the rows sorted in buffer A (one thread per
// column; the outputs overwrite the scratch behind the read position: st[k]
// covers rows int32 2k, 2k + 1 < ld + k of buffer A).
template <bool SAFE>
__global__ void k_bp_tall_walk(SelParams P, int64_t p, int64_t cnt, int64_t ld, int64_t ncol,
                               double* __restrict__ rs, double* __restrict__ st, double* __restrict__ rt,
                               int64_t c0, int tab, int64_t* __restrict__ rows_out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const int64_t n = P.n;
  const int64_t cj = c0 + c;
  const int64_t j = cj < p ? cj : cj + 1;
  const double* xc = P.Xc + j * n;
  const double* pb = P.pb + p * P.np;
  const double* py = P.py + p * P.np;
  const int* row = reinterpret_cast<const int*>(st + c * ld) + ld;
  double T = 0.0;
  for (int64_t k = 0; k < cnt; ++k) T = __dadd_rn(T, fabs(pb[row[k]]));
  double Pp = 0.0;
  for (int64_t k = 0; k < cnt; ++k) {
    const int r = row[k];
    const double w = fabs(pb[r]);
    const double Pk = __dadd_rn(Pp, w);
    double ratio = sratio<SAFE>(P, xc[r], pb[r], py[r]);
    if (ratio == 0.0) ratio = __ddiv_rn(xc[r], pb[r]);  // the zero's sign (the hoisted path may drop it)
    bp_emit(tab, ratio, w, Pk, T, Pp, r, c * ld + k, rs, st, rt, rows_out);  // st[k] after row[k] was read
    Pp = Pk;
  }
}

// ------------------------------------------- optimality certificates --
//
// The dual certificate of oracle.py:141-174 for every column of one line at
// once: v_j minimises f_j(t) = sum_i w_i |r_i - t| + lam |t| iff 0 lies in
// the subdifferential, i.e. with exact weight sums below / above / at v_j
// (fixed-point weights wq, exact in any order) and L = lam 2^s_p:
//   v > 0: |D + L| <= A,  v < 0: |D - L| <= A,  v = 0: |D| <= A + L,
// D = W(r < v) - W(r > v), A = W(r = v).  The slack (A - |...|, or
// A + L - |D|) in weight units is >= 0 exactly when a feasible,
// complementary multiplier vector exists (the reference builds it).  Warp
// per target column; exact ratios compared through their 64-bit keys.
template <bool SAFE>
__global__ void k_certify(SelParams P, int64_t p, const double* __restrict__ v, double lam,
                          double* __restrict__ slack) {
  const int warp = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  const int64_t n = P.n, m = P.m, j = warp;
  if (j >= m) return;
  if (j == p || P.nnz[p] == 0) {
    if (lane == 0) slack[j] = INFINITY;
    return;
  }
  const double* xc = P.Xc + j * n;
  const double* pb = P.pb + p * P.np;
  const double* py = P.py + p * P.np;
  const double* pw = P.pw + p * P.np;
  const double vj = v[j];
  const unsigned long long kv = key64(vj);
  double below = 0.0, above = 0.0, at = 0.0;
  for (int64_t i = lane; i < n; i += 32) {
    const double w = pw[i];
    if (w == 0.0) continue;  // x_ip = 0: not in the column (ratios.py:115)
    const unsigned long long k = key64(sratio<SAFE>(P, xc[i], pb[i], py[i]));
    below += k < kv ? w : 0.0;
    above += k > kv ? w : 0.0;
    at += k == kv ? w : 0.0;
  }
  below = warp_sum(below);
  above = warp_sum(above);
  at = warp_sum(at);
  if (lane == 0) {
    const double L = ldexp(lam, P.spow[p]), D = below - above;
    double s;
    if (kv == kZeroKey) s = at + L - fabs(D);
    else if (vj > 0.0) s = at - fabs(D + L);
    else s = at - fabs(D - L);
    slack[j] = ldexp(s, -P.spow[p]);
  }
}

// ------------------------------------------------------ brute force --
//
// brute_force_column (oracle.py:39-58) for every target column of one pivot:
// f(t) = sum_i |x_ij - t x_ip| + lam |t| evaluated at every candidate t in
// {0} u {x_ij / x_ip : x_ip != 0} (the kinks of the convex objective), the
// smallest t among the minima.  One CTA per target column, one candidate per
// thread at a time, each f(t) summed over the rows in order (the reference's
// axis-0 reduction: the same doubles).  O(n^2) per column: an independent
// check of the sort-free solver, not a fast path.
__global__ void __launch_bounds__(256) k_brute_force(const double* __restrict__ X, int64_t n, int64_t m, int64_t p,
                                                     double lam, double* __restrict__ t_out,
                                                     double* __restrict__ f_out) {
  const int64_t c = blockIdx.x;  // target column index among j != p
  const int64_t j = c < p ? c : c + 1;
  __shared__ double sf[256], st[256];
  double bf = INFINITY, bt = 0.0;
  for (int64_t k = (int64_t)threadIdx.x - 1; k < n; k += blockDim.x) {  // k = -1: the candidate 0
    double t;
    if (k < 0) {
      t = 0.0;
    } else {
      const double b = X[k * m + p];
      if (b == 0.0) continue;
      t = __ddiv_rn(X[k * m + j], b);
    }
    double f = 0.0;
    for (int64_t i = 0; i < n; ++i) f = __dadd_rn(f, fabs(__dsub_rn(X[i * m + j], __dmul_rn(X[i * m + p], t))));
    f = __dadd_rn(f, __dmul_rn(lam, fabs(t)));
    if (f < bf || (f == bf && t < bt)) {
      bf = f;
      bt = t;
    }
  }
  sf[threadIdx.x] = bf;
  st[threadIdx.x] = bt;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) {
      const double f2 = sf[threadIdx.x + o], t2 = st[threadIdx.x + o];
      if (f2 < sf[threadIdx.x] || (f2 == sf[threadIdx.x] && t2 < st[threadIdx.x])) {
        sf[threadIdx.x] = f2;
        st[threadIdx.x] = t2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    t_out[c] = st[0] == 0.0 ? 0.0 : st[0];  // a zero candidate is +0.0
    f_out[c] = sf[0];
  }
}
