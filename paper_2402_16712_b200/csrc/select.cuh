// select.cuh -- K1: the per-(pivot, target) lambda-shifted weighted median
// and column residual (included by l1b200.cu; see its header for the map to
// the reference).
//
// Semantics reproduced (reference ratios.py:109-135 + fit.py:51-63, restated
// sort-free in SURVEY.md Appendix A.2):
//   rows with x_ip == 0 are dropped; r_i = fl(x_ij / x_ip), w_i = |x_ip|;
//   order = stable ascending by r (ties, incl. -0 == +0, by row);
//   with exact fixed-point weights wq, Tq = sum wq, Wneg = sum_{r<0} wq,
//   D = Tq - 2 Wneg and L = lam * 2^s:
//     D < -L           -> negative region, G = (Tq + floor L) / 2
//     D >= ceil(L)     -> non-negative region, G = (Tq - ceil L) / 2
//     otherwise        -> dead column, v_j = +0.0
//   v_j = r of the first element (in that order) whose inclusive prefix
//   weight exceeds G (its exact bits; a zero picks the sign of its own row).
//
// Kernel structure (one thread = one problem, warp = pivot x 32 targets,
// CTA = 8 pivots sharing each staged tile of X):
//   sample   32 rows, float ratios, sorted in registers -> value bracket
//   pass A   FP32 only: r ~ a32 * y32, 32-bin fp32 histogram in VALUE space
//            over the bracket (tails in the edge bins) -> candidate window
//   pass B   exact: fl(a / b), exact int64 weight below the window, exact
//            Wneg -> G, rows inside the window collected -> resolve
//   pass E   residual sum_i |x_ij - v_j x_ip| in row order
// Every CTA runs exactly these passes.  A problem whose window missed the
// crossing or overflowed kCapB is queued with its exact key interval for
// k_straggle (warp per problem), so no CTA waits on its slowest problem.

constexpr int kNBA = 32;         // pass-A histogram bins (2 edge + 30 interior)
constexpr int kCapB = 64;        // rows collected per problem in pass B
constexpr int kDelta = 6;        // +- sample ranks around the estimated crossing
constexpr float kMargin = 0.03f; // window margin, in bins, against float error

struct SelParams {
  const double* X;       // row-major n x m
  const float* Xf;       // float copy (pass A)
  const PivRec* piv;     // [m][n]
  const long long* tq;
  const int* spow;
  const long long* nnz;
  const double* colsum;
  int64_t n, m;
  int64_t p_begin, p_stride, npiv;
  double lam;
  double* V;             // [npiv][m]
  double* E;             // [npiv][m]
  Straggler* strag;      // queue
  unsigned long long* nstrag;
  int* status;
};

// Exact region test: returns false for a dead column, else sets G.
__device__ __forceinline__ bool region_G(long long Tq, long long wneg, double Lsc, long long* G) {
  const double cap = 4.0e18;
  double lf = floor(Lsc), lc = ceil(Lsc);
  long long Lf = lf > cap ? (long long)cap : (long long)lf;
  long long Lc = lc > cap ? (long long)cap : (long long)lc;
  long long D = Tq - 2 * wneg, thr;
  if (D < -Lf) thr = -Lf;
  else if (D >= Lc) thr = Lc;
  else return false;
  *G = (Tq - thr) >> 1;  // Tq - thr >= 0
  return true;
}

template <typename RowT>
__device__ void resolve_rows(const SelParams& P, const RowT* cbuf, int tid, int cnt, long long cum,
                             long long G, int64_t p, int64_t j, double* vout, bool* ok) {
  // Walk the window's distinct values ascending (the stable argsort order of
  // ratios.py:121); within the +-0 group, rows in row order.
  unsigned long long lk[kCapB];
  long long lw[kCapB];
  for (int c = 0; c < cnt; ++c) {
    int row = (int)cbuf[c * kBS + tid];
    PivRec rec = P.piv[p * P.n + row];
    lk[c] = key64(ratio_fast(P.X[(int64_t)row * P.m + j], rec.b, rec.y));
    lw[c] = rec.wq;
  }
  unsigned long long last = 0;
  bool first = true;
  for (int guard = 0; guard <= cnt; ++guard) {
    unsigned long long kmin = ~0ULL;
    bool found = false;
    for (int c = 0; c < cnt; ++c)
      if ((first || lk[c] > last) && lk[c] <= kmin) { kmin = lk[c]; found = true; }
    if (!found) break;
    long long ws = 0;
    for (int c = 0; c < cnt; ++c) ws += (lk[c] == kmin) ? lw[c] : 0;
    if (cum + ws > G) {
      if (kmin == kZeroKey) {
        for (int c = 0; c < cnt; ++c) {
          if (lk[c] != kZeroKey) continue;
          cum += lw[c];
          if (cum > G) {
            int row = (int)cbuf[c * kBS + tid];
            *vout = __ddiv_rn(P.X[(int64_t)row * P.m + j], P.piv[p * P.n + row].b);
            *ok = true;
            return;
          }
        }
      } else {
        *vout = key64_inv(kmin);
        *ok = true;
        return;
      }
    }
    cum += ws;
    last = kmin;
    first = false;
  }
  *ok = false;
}

template <typename RowT>
__global__ void __launch_bounds__(kBS, 2) k_select(SelParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  double* tileA = (double*)smem;                                  // [2][kRows][32]
  float* tileF = (float*)(tileA + 2 * kRows * 32);                // [2][kRows][32]
  PivRec* tileP = (PivRec*)(tileF + 2 * kRows * 32);              // [2][kWarps][kRows]
  float* hist = (float*)(tileP + 2 * kWarps * kRows);             // [kNBA][kBS]
  RowT* cbuf = (RowT*)(hist + kNBA * kBS);                        // [kCapB][kBS]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n = P.n, m = P.m;
  const int64_t kk = (int64_t)blockIdx.y * kWarps + warp;
  const bool piv_ok = kk < P.npiv;
  const int64_t p = piv_ok ? P.p_begin + kk * P.p_stride : 0;
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  const int64_t j = j0 + lane;
  const bool degenerate = piv_ok && P.nnz[p] == 0;
  const bool active = piv_ok && !degenerate && j < m && j != p;
  const int64_t jc = j < m ? j : m - 1;

  long long Tq = 0;
  double Lsc = 0.0;
  if (piv_ok && !degenerate) {
    Tq = P.tq[p];
    Lsc = ldexp(P.lam, P.spow[p]);
  }
  const float lam32 = (float)P.lam;

  // ---- sample: float ratios of 32 strided rows, sorted -> value bracket ----
  float sA = 0.f, oA = 0.f;  // pass-A bin map: bin = RN(clamp(r * sA + oA))
  float lo = 0.f, hi = 0.f;
  if (active) {
    float sr[kSample], sw[kSample];
#pragma unroll
    for (int s = 0; s < kSample; ++s) {
      int64_t r = ((2 * s + 1) * n) / (2 * kSample);
      PivRec rec = P.piv[p * n + r];
      sr[s] = P.Xf[r * m + jc] * rec.y32;
      sw[s] = rec.w32;
    }
#pragma unroll
    for (int k = 2; k <= kSample; k <<= 1) {
#pragma unroll
      for (int jj = k >> 1; jj > 0; jj >>= 1) {
#pragma unroll
        for (int i = 0; i < kSample; ++i) {
          int l = i ^ jj;
          if (l > i) {
            bool up = (i & k) == 0;
            bool sw_ = up ? (sr[i] > sr[l]) : (sr[i] < sr[l]);
            float ta = sr[i], tb = sr[l], wa = sw[i], wb = sw[l];
            sr[i] = sw_ ? tb : ta;
            sr[l] = sw_ ? ta : tb;
            sw[i] = sw_ ? wb : wa;
            sw[l] = sw_ ? wa : wb;
          }
        }
      }
    }
    float ws = 0.f, wn = 0.f;
#pragma unroll
    for (int s = 0; s < kSample; ++s) {
      ws += sw[s];
      wn += sr[s] < 0.f ? sw[s] : 0.f;
    }
    float rho = Tq > 0 ? (float)(Lsc / (double)Tq) : 0.f;
    float d = ws > 0.f ? 1.f - 2.f * wn / ws : 1.f;
    float f = d < -rho ? 0.5f * (1.f + rho) : (d >= rho ? 0.5f * (1.f - rho) : 0.5f);
    float t = f * ws, c = 0.f;
    int sstar = kSample - 1;
    bool got = false;
#pragma unroll
    for (int s = 0; s < kSample; ++s) {
      c += sw[s];
      if (!got && c > t) { sstar = s; got = true; }
    }
    int lo_i = max(sstar - kDelta, 0), hi_i = min(sstar + kDelta, kSample - 1);
#pragma unroll
    for (int s = 0; s < kSample; ++s) {
      if (s == lo_i) lo = sr[s];
      if (s == hi_i) hi = sr[s];
    }
    float span = hi - lo;
    if (!(span > 0.f)) span = fmaxf(fabsf(lo), 1e-30f) * 1e-3f;  // degenerate sample: tiny bracket
    sA = (float)(kNBA - 2) / span;
    oA = 0.5f - lo * sA;  // r in [lo + (b-1) w, lo + b w) -> bin b
  }

  const int64_t nch = (n + kRows - 1) / kRows;
  auto stage = [&](int64_t c, int buf, bool wantA, bool wantF) {
    if (wantA) {
      double* ta = tileA + buf * kRows * 32;
      for (int t = tid; t < kRows * 32; t += kBS) {
        int r = t >> 5, l = t & 31;
        int64_t i = c * kRows + r, jj = j0 + l;
        bool ok = i < n && jj < m;
        cp_async8(ta + t, ok ? (const void*)(P.X + i * m + jj) : (const void*)P.X, ok ? 8 : 0);
      }
    }
    if (wantF) {
      float* tf = tileF + buf * kRows * 32;
      for (int t = tid; t < kRows * 32; t += kBS) {
        int r = t >> 5, l = t & 31;
        int64_t i = c * kRows + r, jj = j0 + l;
        bool ok = i < n && jj < m;
        cp_async4(tf + t, ok ? (const void*)(P.Xf + i * m + jj) : (const void*)P.Xf, ok ? 4 : 0);
      }
    }
    PivRec* tp = tileP + (buf * kWarps + warp) * kRows;
    for (int t = lane; t < 2 * kRows; t += 32) {
      int r = t >> 1, h = t & 1;
      int64_t i = c * kRows + r;
      bool ok = piv_ok && i < n;
      const char* src = ok ? (const char*)(P.piv + p * n + i) + 16 * h : (const char*)P.piv;
      cp_async16((char*)(tp + r) + 16 * h, src, ok ? 16 : 0);
    }
    cp_commit();
  };
  // Runs `body(r, i, buf)` over all rows with double-buffered staging.
  auto sweep = [&](bool wantA, bool wantF, bool busy, auto&& body) {
    stage(0, 0, wantA, wantF);
    for (int64_t c = 0; c < nch; ++c) {
      if (c + 1 < nch) stage(c + 1, (int)((c + 1) & 1), wantA, wantF);
      else cp_commit();
      cp_wait1();
      __syncthreads();
      if (busy) {
        const int buf = (int)(c & 1);
        const int rmax = (int)min((int64_t)kRows, n - c * kRows);
        body(buf, rmax, c * kRows);
      }
      __syncthreads();
    }
    cp_wait0();
  };

  // ---- pass A: approximate value-space histogram (FP32) ------------------
#pragma unroll
  for (int b = 0; b < kNBA; ++b) hist[b * kBS + tid] = 0.f;
  float wn32 = 0.f;
  const bool warp_active = __any_sync(0xffffffffu, active);
  sweep(false, true, warp_active, [&](int buf, int rmax, int64_t i0) {
    const float* tf = tileF + buf * kRows * 32;
    const PivRec* tp = tileP + (buf * kWarps + warp) * kRows;
#pragma unroll 4
    for (int r = 0; r < rmax; ++r) {
      const float2 yw = *reinterpret_cast<const float2*>(&tp[r].y32);
      const float q = tf[r * 32 + lane] * yw.x;
      float t = fminf(fmaxf(fmaf(q, sA, oA), 0.f), (float)(kNBA - 1));
      int b = __float_as_int(t + 8388608.f) - 0x4B000000;  // RN(t), monotone in q
      hist[b * kBS + tid] += yw.y;
      wn32 += q < 0.f ? yw.y : 0.f;
    }
  });

  // window from pass A: the bin holding the approximate crossing
  unsigned long long KL = 0, KH = ~0ULL;
  if (active) {
    float T32 = 0.f;
#pragma unroll
    for (int b = 0; b < kNBA; ++b) T32 += hist[b * kBS + tid];
    float D = T32 - 2.f * wn32;
    float thr = D < -lam32 ? -lam32 : (D >= lam32 ? lam32 : 0.f);
    float G32 = 0.5f * (T32 - thr);
    float cum = 0.f;
    int bw = kNBA - 1;
    bool got = false;
#pragma unroll
    for (int b = 0; b < kNBA; ++b) {
      cum += hist[b * kBS + tid];
      if (!got && cum > G32) { bw = b; got = true; }
    }
    // interior bin b covers r in [lo + (b-1) w, lo + b w), w = 1 / sA
    const double w = 1.0 / (double)sA;
    if (bw > 0) KL = key64((double)lo + ((double)bw - 1.0 - kMargin) * w);
    if (bw < kNBA - 1) KH = key64((double)lo + ((double)bw + kMargin) * w);
  }

  // ---- pass B: exact ratios, exact weights, collect the window ------------
  long long wb = 0, win = 0, wneg = 0;
  int cnt = 0;
  sweep(true, false, warp_active, [&](int buf, int rmax, int64_t i0) {
    const double* ta = tileA + buf * kRows * 32;
    const PivRec* tp = tileP + (buf * kWarps + warp) * kRows;
#pragma unroll 2
    for (int r = 0; r < rmax; ++r) {
      const PivRec rec = tp[r];
      const double q = ratio_fast(ta[r * 32 + lane], rec.b, rec.y);
      const unsigned long long k = key64(q);
      const long long wq = rec.wq;
      wneg += (k < kZeroKey) ? wq : 0;
      if (k < KL) {
        wb += wq;
      } else if (k < KH) {
        win += wq;
        if (cnt < kCapB) cbuf[cnt * kBS + tid] = (RowT)(i0 + r);
        ++cnt;
      }
    }
  });

  double v = 0.0;
  bool done = !active;
  if (active) {
    long long G = 0;
    if (!region_G(Tq, wneg, Lsc, &G)) {
      v = 0.0;  // dead column (fit.py:60-63 returns +0.0)
      done = true;
    } else if (wb <= G && G < wb + win && cnt <= kCapB) {
      resolve_rows<RowT>(P, cbuf, tid, cnt, wb, G, p, jc, &v, &done);
    }
    if (!done) {
      Straggler s;
      s.kk = (int)kk;
      s.j = (int)j;
      s.G = G;
      if (G < wb) { s.lo = 0; s.hi = KL - 1; s.wb = 0; }
      else if (G >= wb + win) { s.lo = KH; s.hi = ~0ULL; s.wb = wb + win; }
      else { s.lo = KL; s.hi = KH - 1; s.wb = wb; }
      unsigned long long slot = atomicAdd(P.nstrag, 1ULL);
      P.strag[slot] = s;
    }
  }

  // ---- pass E: residual in row order --------------------------------------
  double e = 0.0;
  const bool warp_err = __any_sync(0xffffffffu, active && done);
  sweep(true, false, warp_err, [&](int buf, int rmax, int64_t i0) {
    const double* ta = tileA + buf * kRows * 32;
    const PivRec* tp = tileP + (buf * kWarps + warp) * kRows;
#pragma unroll 4
    for (int r = 0; r < rmax; ++r) e += fabs(__dsub_rn(ta[r * 32 + lane], __dmul_rn(tp[r].b, v)));
  });

  if (piv_ok && j < m) {
    if (degenerate) {
      P.V[kk * m + j] = 0.0;
      P.E[kk * m + j] = P.colsum[j];
    } else if (j == p) {
      P.V[kk * m + j] = 1.0;
      P.E[kk * m + j] = 0.0;
    } else if (done) {
      P.V[kk * m + j] = v;
      P.E[kk * m + j] = e;
    }
  }
}

// Route every problem of a shard to the straggler queue (inputs outside the
// fast path's exponent window use k_straggle for everything).
__global__ void k_queue_all(SelParams P) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= P.npiv * P.m) return;
  int64_t kk = idx / P.m, j = idx - kk * P.m;
  int64_t p = P.p_begin + kk * P.p_stride;
  if (P.nnz[p] == 0) {
    P.V[kk * P.m + j] = 0.0;
    P.E[kk * P.m + j] = P.colsum[j];
    return;
  }
  if (j == p) {
    P.V[kk * P.m + j] = 1.0;
    P.E[kk * P.m + j] = 0.0;
    return;
  }
  Straggler s;
  s.kk = (int)kk;
  s.j = (int)j;
  s.G = -1;  // unknown: k_straggle computes Wneg and G first
  s.lo = 0;
  s.hi = ~0ULL;
  s.wb = 0;
  unsigned long long slot = atomicAdd(P.nstrag, 1ULL);
  P.strag[slot] = s;
}

// ----------------------------------------------------------- stragglers --
//
// One warp per queued problem, exact throughout.  The record carries a key
// interval [lo, hi] known to contain the crossing and the exact weight below
// it.  Each round either collects every element of the interval (<= kSCap)
// into shared memory, bitonic-sorts them by (key, row) and walks the prefix,
// or histograms the interval into 256 key buckets (shared int64 atomics) and
// narrows to the crossing bucket.  Ratios are the fast exact path when SAFE,
// IEEE __ddiv_rn otherwise.

constexpr int kSWarps = 4;
constexpr int kSCap = 1024;
constexpr int kSBins = 256;

struct SEnt {
  unsigned long long k;
  long long w;
  int row;
  int pad;
};

template <bool SAFE>
__device__ __forceinline__ double sratio(const SelParams& P, int64_t i, int64_t j, const PivRec& rec) {
  double a = P.X[i * P.m + j];
  if (SAFE) return ratio_fast(a, rec.b, rec.y);
  return rec.b != 0.0 ? __ddiv_rn(a, rec.b) : __longlong_as_double(0x7ff8000000000000LL);
}

__device__ __forceinline__ long long warp_sum_ll(long long x) {
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

constexpr size_t kStraggleSmem = (size_t)kSWarps * (kSCap * sizeof(SEnt) + kSBins * sizeof(unsigned long long));

template <bool SAFE>
__global__ void __launch_bounds__(kSWarps * 32) k_straggle(SelParams P) {
  extern __shared__ __align__(16) unsigned char ssm[];
  SEnt(*ent)[kSCap] = reinterpret_cast<SEnt(*)[kSCap]>(ssm);
  unsigned long long(*bins)[kSBins] =
      reinterpret_cast<unsigned long long(*)[kSBins]>(ssm + (size_t)kSWarps * kSCap * sizeof(SEnt));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned long long total = *P.nstrag;
  const int64_t n = P.n, m = P.m;
  for (unsigned long long t = (unsigned long long)blockIdx.x * kSWarps + warp; t < total;
       t += (unsigned long long)gridDim.x * kSWarps) {
    Straggler s = P.strag[t];
    const int64_t kk = s.kk, j = s.j, p = P.p_begin + kk * P.p_stride;
    const PivRec* pr = P.piv + p * n;
    const long long Tq = P.tq[p];
    const double Lsc = ldexp(P.lam, P.spow[p]);
    long long G = s.G, wb = s.wb;
    unsigned long long lo = s.lo, hi = s.hi;
    bool dead = false;
    if (G < 0) {  // exact Wneg and key range first
      long long wneg = 0;
      unsigned long long kmin = ~0ULL, kmax = 0;
      for (int64_t i = lane; i < n; i += 32) {
        PivRec rec = pr[i];
        if (rec.wq == 0) continue;
        double q = sratio<SAFE>(P, i, j, rec);
        unsigned long long k = key64(q);
        if (q < 0.0) wneg += rec.wq;
        kmin = min(kmin, k);
        kmax = max(kmax, k);
      }
      wneg = warp_sum_ll(wneg);
      for (int o = 16; o; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
      }
      dead = !region_G(Tq, wneg, Lsc, &G);
      lo = kmin;
      hi = kmax;
      wb = 0;
    }
    double v = 0.0;
    bool ok = dead;
    for (int round = 0; round < 40 && !ok; ++round) {
      // collect the interval if it fits, counting it either way
      int base = 0;
      long long wsum = 0;
      for (int64_t i0 = 0; i0 < n; i0 += 32) {
        int64_t i = i0 + lane;
        bool in = false;
        unsigned long long k = 0;
        long long w = 0;
        if (i < n) {
          PivRec rec = pr[i];
          if (rec.wq != 0) {
            k = key64(sratio<SAFE>(P, i, j, rec));
            in = k >= lo && k <= hi;
            w = rec.wq;
          }
        }
        unsigned mask = __ballot_sync(0xffffffffu, in);
        int pos = base + __popc(mask & ((1u << lane) - 1));
        if (in) {
          wsum += w;
          if (pos < kSCap) ent[warp][pos] = SEnt{k, w, (int)i, 0};
        }
        base += __popc(mask);
      }
      __syncwarp();
      if (base <= kSCap) {
        // bitonic sort by (key, row) over the next power of two
        int np2 = 1;
        while (np2 < base) np2 <<= 1;
        for (int e = base + lane; e < np2; e += 32) ent[warp][e] = SEnt{~0ULL, 0, 0x7fffffff, 0};
        __syncwarp();
        for (int kq = 2; kq <= np2; kq <<= 1) {
          for (int jq = kq >> 1; jq > 0; jq >>= 1) {
            for (int e = lane; e < np2; e += 32) {
              int l = e ^ jq;
              if (l > e) {
                SEnt a = ent[warp][e], b = ent[warp][l];
                bool gt = a.k > b.k || (a.k == b.k && a.row > b.row);
                bool up = (e & kq) == 0;
                if (gt == up) { ent[warp][e] = b; ent[warp][l] = a; }
              }
            }
            __syncwarp();
          }
        }
        // first element whose inclusive prefix exceeds G
        long long cum = wb;
        int hit = -1;
        for (int e0 = 0; e0 < base && hit < 0; e0 += 32) {
          int e = e0 + lane;
          long long w = e < base ? ent[warp][e].w : 0;
          long long x = w;
          for (int o = 1; o < 32; o <<= 1) {
            long long y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          bool cross = e < base && cum + x > G;
          unsigned cm = __ballot_sync(0xffffffffu, cross);
          if (cm) hit = e0 + __ffs(cm) - 1;
          cum += __shfl_sync(0xffffffffu, x, 31);
        }
        if (hit >= 0) {
          SEnt h = ent[warp][hit];
          v = h.k == kZeroKey ? __ddiv_rn(P.X[(int64_t)h.row * m + j], pr[h.row].b) : key64_inv(h.k);
          ok = true;
        }
        __syncwarp();
        if (!ok) break;  // cannot happen: the interval holds the crossing
      } else {
        // narrow: 256 key buckets over [lo, hi]
        int sh = ceil_log2_u64(hi - lo + 1) - 8;
        if (hi - lo == ~0ULL) sh = 56;
        sh = sh > 0 ? sh : 0;
        for (int b = lane; b < kSBins; b += 32) bins[warp][b] = 0;
        __syncwarp();
        for (int64_t i = lane; i < n; i += 32) {
          PivRec rec = pr[i];
          if (rec.wq == 0) continue;
          unsigned long long k = key64(sratio<SAFE>(P, i, j, rec));
          if (k >= lo && k <= hi) atomicAdd(&bins[warp][(k - lo) >> sh], (unsigned long long)rec.wq);
        }
        __syncwarp();
        long long cum = wb;
        int bsel = kSBins - 1;
        for (int b = 0; b < kSBins; ++b) {
          long long hb = (long long)bins[warp][b];
          if (cum + hb > G) { bsel = b; break; }
          cum += hb;
        }
        unsigned long long nlo = lo + ((unsigned long long)bsel << sh);
        unsigned long long nhi = nlo + ((sh >= 64) ? ~0ULL : ((1ULL << sh) - 1));
        if (nhi > hi || nhi < nlo) nhi = hi;
        lo = nlo;
        hi = nhi;
        wb = cum;
        __syncwarp();
      }
    }
    if (!ok) {
      if (lane == 0) atomicExch(P.status, L1B_EINTERNAL);
      v = 0.0;
    }
    // residual, lane-strided then a fixed butterfly
    double e = 0.0;
    for (int64_t i = lane; i < n; i += 32)
      e += fabs(__dsub_rn(P.X[i * m + j], __dmul_rn(pr[i].b, v)));
    for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    if (lane == 0) {
      P.V[kk * m + j] = v;
      P.E[kk * m + j] = e;
    }
    __syncwarp();
  }
}
