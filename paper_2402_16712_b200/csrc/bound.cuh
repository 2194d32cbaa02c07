// bound.cuh -- pivot pruning for fit_line (included by l1b200.cu after
// select.cuh).
//
// fit_line (fit.py:88-102) needs only the winning pivot, and most pivots'
// objectives sit far above it.  k_bound runs ONE FP32 pass per (pivot p,
// target j) problem and bounds the column optimum
//     f_j* = min_v e_j(v) + lam |v|,   e_j(v) = sum_i |x_ij - v x_ip|
// from below and above:
//   * the pass histograms the ratios r_i = x_ij / x_ip over the sample bracket
//     (64 slots: below / 62 bins / above, as k_select's first pass; weights
//     are 32-bit fixed point, wq / 2^21, so the sums are exact and the only
//     weight error is the rounding of each weight) and sums e_j at the sample
//     centre c;
//   * f_j is convex with subgradient g(v) = W(r < v) - W(r > v) + lam sgn(v),
//     so the histogram bounds g on every bin, f at the bin edges follows from
//     f(c) by integrating those bounds, and the optimum lies between the last
//     edge with g <= 0 and the first with g >= 0 (tangent lower bound there);
//   * v = 0 is always feasible with f(0) = sum_i |x_ij| exactly, which also
//     pins dead columns.
// Every float error (histogram sums, residual terms) enters as an explicit
// margin, so lb <= f_j* <= ub rigorously; per pivot z_p = lam + sum_j f_j*
// (v_p = 1).  A pivot whose lower bound exceeds the smallest upper bound
// cannot win; the host fits only the others exactly (l1b_fit_pivot_list).
//
// Layout: a CTA is 4 pivots x 64 targets and each thread owns FOUR problems
// (the 2 pivots of its warp's pair x 2 targets): one x_ij load serves two
// problems, one 16-byte broadcast of a row pair's (y, x, wq) records serves
// 128 elements, and the four histogram chains interleave (k_bound below).

constexpr int kBPairs = 2;                 // pivot pairs per k_bound CTA
constexpr int kBPiv = 2 * kBPairs;         // pivots per CTA (k_group_bound's plane groups)
constexpr int kBQuarters = 4;              // row quarters per pair
constexpr int kBWarps = kBPairs * kBQuarters;
constexpr int kBThreads = kBWarps * 32;
constexpr int kBSlots = kBPairs * 64;      // histogram columns: (pair, target of 64)
#ifndef KB_ROWS
#define KB_ROWS 64
#endif
#ifndef KB_GUNROLL
#define KB_GUNROLL 4  // 4-row groups of a chunk unrolled per warp (a 64-row chunk has 4)
#endif
#ifndef KB_STAGES
#define KB_STAGES 2
#endif
constexpr int kBRows = KB_ROWS;            // rows per staged chunk
constexpr int kBTile = kBRows * 32 * 4;    // one x_ij float tile [row][32 targets]; a stage holds two
constexpr int kBPlane = kBRows * kBPiv * 12;  // k_group_bound records: 12 B per (row, pivot)
constexpr int kBStage = 2 * kBTile + kBPlane;
constexpr int kBStages = KB_STAGES;
constexpr int kBGUnroll = KB_GUNROLL;
constexpr int kBHist = 2 * kNB * kBSlots * 4;  // [pivot of the pair][bin][slot], exact 32-bit sums
static_assert(kBPiv == kGroupBoundPiv, "k_bound reads k_group_bound's plane groups");
static_assert(kBRows % (4 * kBQuarters) == 0, "a chunk is whole 4-row groups per quarter");
static_assert(kBStages * kBStage >= kBQuarters * 4 * kBPairs * 32 * 8, "stage buffers hold the residual shares");
constexpr size_t kBoundSmem = (size_t)kBStages * kBStage + kBHist;
// bracket half-width in sample ranks: narrow for the one-pass bound (tight
// bins), wider when later passes refine it (fewer optima outside)
#ifndef KB_DELTA1
#define KB_DELTA1 8
#endif
#ifndef KB_DELTAN
#define KB_DELTAN 10
#endif
constexpr int kBDelta1 = KB_DELTA1, kBDeltaN = KB_DELTAN;

// Bounds of one column optimum from its histogram h[slot * hs] (exact sums
// of 32-bit weights of q each) over the bracket [lo, hi) (62 interior bins),
// e_j(c) = ec, the exact pivot weight T and the column's sum_i |x_ij| (f(0)).
// The histogram column as inclusive prefix sums Cu_k, in place, and the
// checkpoints SC_{8i} of SC_k = sum_{q<k} Cu_q (exact integers).
struct Prefix {
  unsigned* h;
  int hs;
  unsigned long long sc8[8];
  __device__ __forceinline__ void build() {
    unsigned cu = 0;
    unsigned long long sc = 0;
#pragma unroll
    for (int k = 0; k < kNB; ++k) {
      if ((k & 7) == 0) sc8[k >> 3] = sc;
      cu += h[k * hs];
      h[k * hs] = cu;
      sc += cu;
    }
  }
  __device__ __forceinline__ unsigned cu(int k) const { return h[k * hs]; }
  __device__ __forceinline__ unsigned long long sc(int k) const {
    unsigned long long s = sc8[k >> 3];
    for (int q = k & ~7; q < k; ++q) s += h[q * hs];
    return s;
  }
};

__device__ __forceinline__ void column_bounds(const Prefix& H, double q, double lo, double hi, double c,
                                              double ec, double T, double lam, double colsum, int64_t n,
                                              float smin, float smax, double* lbo, double* ubo, double2* range,
                                              float2* next) {
  const double w = (hi - lo) / (double)kNI;
  // margins: the 32-bit weights are within q/2 of |x_ip| each (so any
  // cumulative weight within n q / 2), the residual terms within 2^-22 of
  // |a| + |c b|, and their per-chunk float sums
  const double dC = 0.5000001 * (double)n * q;
  // every row's float ratio (and the float bin edges) sit within pert / w_i
  // of its binned position, so f moves by at most pert when the rows are
  // moved into their bins; the bounds below hold for that moved problem
  const double pert = 0x1p-22 * colsum + T * (0x1p-21 * (fabs(lo) + fabs(hi)) + 0x1p-20 * w);
  // (a chunk sums 16 pairwise 4-row sums: relative error <= 18 u)
  const double eps = 0x1p-22 * (colsum + fabs(c) * T) + 20.0 * 0x1p-24 * ec + pert;
  const double fc = ec + lam * fabs(c);
  // edges e_k = lo + k w (k = 0..62); C_k = q Cu_k = weight with r < e_k
  // (slots 0..k).  The subgradient bounds at edge k are
  //   glo(k) = 2 (C_k - dC) - T + lam sp(k) <= g(e_k+),  sp(k) = e_k >= 0 ? 1 : -1,
  //   ghi(k) = 2 (C_k + dC) - T + lam sm(k) >= g(e_k-),  sm(k) = e_k >  0 ? 1 : -1,
  // on bin [e_k, e_k+1] g lies in [glo(k), ghi(k+1)], and their integrals
  //   Ilo(k) = sum_{q<k} w glo(q),  Ihi(k) = sum_{q<k} w ghi(q+1)
  // need only the exact integer prefix sums Cu_k, SC_k = sum_{q<k} Cu_q and
  // the edge-sign counts, so the walk over the edges is integer-only.
  auto edge = [&](int k) { return lo + (double)k * w; };
  int z0 = min(kNB - 1, max(0, (int)ceil(-lo / w)));  // edges e_0 .. e_z0-1 are < 0
  while (z0 > 0 && edge(z0 - 1) >= 0.0) --z0;
  while (z0 < kNB - 1 && edge(z0) < 0.0) ++z0;
  int z1 = z0;  // edges e_0 .. e_z1-1 are <= 0
  while (z1 < kNB - 1 && edge(z1) <= 0.0) ++z1;
  const int kc = min(kNI - 1, max(0, (int)floor((c - lo) / w)));
  // integer thresholds, rounded so that passing them implies the double test:
  // ghi(k) <= 0 <=> Cu_k <= (T - 2 dC - lam sm) / 2q;  glo(k) >= 0 <=> Cu_k >= (T + 2 dC - lam sp) / 2q
  const double iq2 = 0.5 / q;
  auto thr_le = [&](double x) -> long long {
    x = x * iq2 * (1.0 - 0x1p-44) - 0x1p-8;
    return x < 0.0 ? -1LL : (x >= 0x1p62 ? (1LL << 62) : (long long)floor(x));
  };
  auto thr_ge = [&](double x) -> long long {
    x = x * iq2 * (1.0 + 0x1p-44) + 0x1p-8;
    return x <= 0.0 ? 0LL : (x >= 0x1p62 ? (1LL << 62) : (long long)ceil(x));
  };
  const long long tLm = thr_le(T - 2.0 * dC + lam), tLp = thr_le(T - 2.0 * dC - lam);  // sm = -1 / +1
  const long long tRm = thr_ge(T + 2.0 * dC + lam), tRp = thr_ge(T + 2.0 * dC - lam);  // sp = -1 / +1
  // kL = last edge with ghi <= 0, kR = first with glo >= 0: Cu_k grows and
  // the thresholds only drop at the sign change, so both tests are monotone
  // in k and two binary searches over the prefix sums find them
  const bool hasL_m = tLm >= 0, hasL_p = tLp >= 0;
  const unsigned uLm = (unsigned)min(max(tLm, 0LL), 0xffffffffLL), uLp = (unsigned)min(max(tLp, 0LL), 0xffffffffLL);
  const unsigned uRm = (unsigned)min(tRm, 0xffffffffLL), uRp = (unsigned)min(tRp, 0xffffffffLL);
  const bool hasR_m = tRm <= 0xffffffffLL, hasR_p = tRp <= 0xffffffffLL;
  auto pL = [&](int k) {
    const unsigned cu = H.cu(k);
    return k >= z1 ? (hasL_p & (cu <= uLp)) : (hasL_m & (cu <= uLm));
  };
  auto pR = [&](int k) {
    const unsigned cu = H.cu(k);
    return k >= z0 ? (hasR_p & (cu >= uRp)) : (hasR_m & (cu >= uRm));
  };
  int kL, kR;
  {
    int a = -1, b = kNI + 1;  // pL(a) holds, pL(b) fails
    while (b - a > 1) {
      const int mid = (a + b) >> 1;
      if (pL(mid)) a = mid;
      else b = mid;
    }
    kL = a;
    a = -1;
    b = kNI + 1;  // pR(a) fails, pR(b) holds
    while (b - a > 1) {
      const int mid = (a + b) >> 1;
      if (pR(mid)) b = mid;
      else a = mid;
    }
    kR = b;  // kNI + 1 = kNB - 1: not in the bracket
  }
  const long long CuL = kL >= 0 ? (long long)H.cu(kL) : 0, SCL = kL >= 0 ? (long long)H.sc(kL) : 0;
  const long long CuR = kR <= kNI ? (long long)H.cu(kR) : 0, SCR = kR <= kNI ? (long long)H.sc(kR) : 0;
  const long long CuC = H.cu(kc), SCC = (long long)H.sc(kc), CuC1 = H.cu(kc + 1), Cu0 = H.cu(0);
  const long long Cu62 = H.cu(kNI), SC62 = (long long)H.sc(kNI);
  const double q2 = 2.0 * q;
  auto glo = [&](int k, long long Cu) { return q2 * (double)Cu - 2.0 * dC - T + (k >= z0 ? lam : -lam); };
  auto ghi = [&](int k, long long Cu) { return q2 * (double)Cu + 2.0 * dC - T + (k >= z1 ? lam : -lam); };
  auto Ilo = [&](int k, long long SC) {  // SP(k) = sum_{q<k} sp(q) = k - 2 min(k, z0)
    return w * (q2 * (double)SC - (double)k * (2.0 * dC + T) + lam * (double)(k - 2 * min(k, z0)));
  };
  auto Ihi = [&](int k, long long SC, long long Cu) {  // SM1(k) = sum_{q=1..k} sm(q)
    const int le = max(0, min(k, z1 - 1));
    return w * (q2 * (double)(SC + Cu - Cu0) + (double)k * (2.0 * dC - T) + lam * (double)(k - 2 * le));
  };
  const double IloC = Ilo(kc, SCC), IhiC = Ihi(kc, SCC, CuC);
  const double gloC = glo(kc, CuC), ghiC = ghi(kc + 1, CuC1), gloL = kL >= 0 ? glo(kL, CuL) : 0.0;
  const double CL = q * (double)CuL, CR = kR <= kNI ? q * (double)CuR : T;
  // f at e_kc from f(c), then at any edge k from e_kc
  const double dc = c - edge(kc);
  const double fkc_lo = fc - dc * ghiC, fkc_hi = fc - dc * gloC;
  auto f_lo = [&](int k, long long SC, long long Cu) {
    return k >= kc ? fkc_lo + (Ilo(k, SC) - IloC) : fkc_lo - (IhiC - Ihi(k, SC, Cu));
  };
  auto f_hi = [&](int k, long long SC, long long Cu) {
    return k >= kc ? fkc_hi + (Ihi(k, SC, Cu) - IhiC) : fkc_hi - (IloC - Ilo(k, SC));
  };
  // f(0) = sum_i |x_ij|: the dead value; colsum carries the rounding of an
  // n-term f64 sum (any order): within (n + 128) 2^-53 of it
  const double f0e = (double)(n + 128) * 0x1p-53 * colsum;
  const double f0 = colsum - f0e;  // a lower bound of f(0) (the kink bounds below)
  double lb, ub = fmin(fc + eps, colsum + f0e);
  const double eL = kL >= 0 ? edge(kL) : -INFINITY, eR = kR <= kNI ? edge(kR) : INFINITY;
  if (kL >= 0 && kR <= kNI && kL <= kR) {
    lb = f_lo(kL, SCL, CuL) - eps + fmin(0.0, gloL) * (eR - eL);
    ub = fmin(ub, fmin(f_hi(kL, SCL, CuL), f_hi(kR, SCR, CuR)) + eps);
  } else {
    lb = 0.0;  // the optimum lies beyond the bracket: only the trivial bound
    if (kL == kNI) ub = fmin(ub, f_hi(kNI, SC62, Cu62) + eps);
  }
  if (eL <= 0.0 && 0.0 <= eR) {
    // the penalty's kink: g(0-) <= 2 W(r < eR) - T - lam, g(0+) >= 2 W(r < eL) - T + lam;
    // f(v) >= f0 + g(0-) v on v <= 0 and f(v) >= f0 + g(0+) v on v >= 0
    const double g0m = 2.0 * (CR + dC) - T - lam, g0p = 2.0 * ((kL >= 0 ? CL : 0.0) - dC) - T + lam;
    const double left = isfinite(eL) ? f0 + fmax(0.0, g0m) * eL : (g0m <= 0.0 ? f0 : 0.0);
    const double right = isfinite(eR) ? f0 + fmin(0.0, g0p) * eR : (g0p >= 0.0 ? f0 : 0.0);
    lb = fmax(lb, fmin(left, right) - pert);
  }
  *lbo = fmax(0.0, lb);
  *ubo = ub;
  // where the optimum lies (seed for the exact solver), widened for the
  // rows' float ratios and edges
  if (kL >= 0 && kR <= kNI && kL <= kR) {
    const double d = 0x1p-19 * (fabs(eL) + fabs(eR) + fabs(lo) + fabs(hi)) + 0x1p-10 * w;
    *range = make_double2(eL - d, eR + d);
  } else {
    *range = make_double2(-INFINITY, INFINITY);
  }
  // the next pass's range: between the edges where the optimum provably lies
  // (a little wider), or, when a side is not in the bracket, extended there
  const float flo = (float)lo, fhi = (float)hi, span = fhi - flo;
  float a, b;
  if (kL >= 0 && kR <= kNI) {
    a = (float)edge(max(0, min(kL, kR - 1)));
    b = (float)edge(min(kNI, max(kR, kL + 1)));
  } else if (kR <= kNI) {  // optimum at or below lo
    a = fminf(smin, flo) - 2.f * span;
    b = (float)edge(kR);
  } else if (kL >= 0) {  // at or above the last edge
    a = (float)edge(kL);
    b = fmaxf(smax, fhi) + 2.f * span;
  } else {  // no edge is decisive (margins dominate): keep the range
    a = flo;
    b = fhi;
  }
  const float mg = 0.05f * (b - a);
  a -= mg;
  b += mg;
  if (!(b > a)) b = a + fmaxf(fabsf(a), 1e-30f) * 1e-6f;
  *next = make_float2(a, b);
}

// Sample bracket of one problem: float ratios of 32 strided rows, sorted in
// registers as packed 32-bit keys (order-preserving image of the ratio, low 8
// bits replaced by the row's weight quantised to 1/255 of the sample's
// largest), so every compare-exchange is a min and a max; returns the
// bracket +-delta ranks around the estimated crossing, that estimate (the
// residual's reference point) and the sample's extremes.  The bracket only
// steers the histogram: any bracket gives rigorous bounds.
__device__ __forceinline__ unsigned f2key(float f) {
  const unsigned b = __float_as_uint(f);
  return b ^ ((unsigned)((int)b >> 31) | 0x80000000u);
}
__device__ __forceinline__ float key2f(unsigned k) {
  return __uint_as_float(k ^ (((unsigned)((int)~k >> 31)) | 0x80000000u));
}

// lam_lo < lam_hi (one pass for several penalties): the bracket covers the
// estimated crossings of both, and 0 when lam_hi may kill the column.
// rep / nrep: the sample is rows (s * nrep + rep) of a stratified 32 * nrep
// row grid (nrep = 1: rows (2s + 1) n / 64).
__device__ __forceinline__ void sample_bracket1(const SelParams& P, int64_t p, int64_t tbase, int lane, double Tq,
                                                double unit, int delta, float* lo, float* hi, float* cen,
                                                float* smin, float* smax, double lam_lo, double lam_hi, int rep,
                                                int nrep) {
  const int64_t n = P.n;
  float sr[kSample], sw[kSample];
  float wmax = 0.f;
#pragma unroll
  for (int s = 0; s < kSample; ++s) {
    const int64_t r = ((2 * ((int64_t)s * nrep + rep) + 1) * n) / (2 * (int64_t)kSample * nrep);
    const float2 f = P.pf[p * P.np + r];
    sr[s] = P.Xft[tbase + r * 32 + lane] * f.x;
    sw[s] = fabsf(f.y);
    wmax = fmaxf(wmax, sw[s]);
  }
  const float wsc = wmax > 0.f ? 255.f / wmax : 0.f;
  unsigned key[kSample];
#pragma unroll
  for (int s = 0; s < kSample; ++s) key[s] = (f2key(sr[s]) & 0xffffff00u) | (unsigned)__float2uint_rn(sw[s] * wsc);
#pragma unroll
  for (int k = 2; k <= kSample; k <<= 1) {
#pragma unroll
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
#pragma unroll
      for (int i = 0; i < kSample; ++i) {
        const int l = i ^ jj;
        if (l > i) {
          const unsigned a = key[i], b = key[l];
          const bool up = (i & k) == 0;
          key[i] = up ? min(a, b) : max(a, b);
          key[l] = up ? max(a, b) : min(a, b);
        }
      }
    }
  }
  unsigned ws = 0, wn = 0;
#pragma unroll
  for (int s = 0; s < kSample; ++s) {
    const unsigned wq = key[s] & 0xffu;
    ws += wq;
    wn += key[s] < 0x80000000u ? wq : 0u;  // ratio < 0
  }
  const float d = ws > 0 ? 1.f - 2.f * (float)wn / (float)ws : 1.f;
  auto crossing = [&](double lam) {  // first s with prefix weight > the lam-shifted median
    const float rho = Tq > 0.0 ? (float)(lam / (Tq * unit)) : 0.f;
    const float f = d < -rho ? 0.5f * (1.f + rho) : (d >= rho ? 0.5f * (1.f - rho) : 0.5f);
    const float t = f * (float)ws;
    unsigned c = 0;
    int ss = kSample - 1;
    bool got = false;
#pragma unroll
    for (int s = 0; s < kSample; ++s) {
      c += key[s] & 0xffu;
      if (!got && (float)c > t) { ss = s; got = true; }
    }
    return ss;
  };
  const int sstar = crossing(lam_lo);
  const bool multi = lam_hi > lam_lo;
  const int s2 = multi ? crossing(lam_hi) : sstar;
  const int lo_i = max(min(sstar, s2) - delta, 0), hi_i = min(max(sstar, s2) + delta, kSample - 1);
  unsigned kl = 0, kh = 0, kce = 0;
#pragma unroll
  for (int s = 0; s < kSample; ++s) {
    if (s == lo_i) kl = key[s];
    if (s == hi_i) kh = key[s];
    if (s == sstar) kce = key[s];
  }
  float l = key2f(kl & 0xffffff00u), hh = key2f((kh & 0xffffff00u) | 0xffu), ce = key2f(kce & 0xffffff00u);
  if (!(hh > l)) {  // degenerate sample: a tiny bracket around it
    const float e = fmaxf(fabsf(l), 1e-30f) * 1e-3f;
    l -= e;
    hh += e;
  }
  if (multi && Tq > 0.0 && fabsf(d) <= (float)(lam_hi / (Tq * unit))) {  // may be dead at lam_hi
    l = fminf(l, 0.f);
    hh = fmaxf(hh, 0.f);
  }
  *lo = l;
  *hi = hh;
  *cen = fminf(fmaxf(ce, l), hh);
  *smin = key2f(key[0] & 0xffffff00u);
  *smax = key2f((key[kSample - 1] & 0xffffff00u) | 0xffu);
}

// Tall columns: nrep independent 32-row samples (interleaved strata); their
// crossing estimates are averaged and the bracket half-widths shrink by
// sqrt(nrep), the same coverage around an estimate sqrt(nrep) times tighter,
// so the histogram's bins (and the bounds' slack) narrow with it.  Short
// columns (the sample stage would cost a visible share of the pass) keep one.
#ifndef KB_SREP_ROWS
#define KB_SREP_ROWS 4096  // rows per extra sample
#endif
#ifndef KB_SREP_MAX
#define KB_SREP_MAX 12
#endif
__device__ __forceinline__ void sample_bracket_reps(const SelParams& P, int64_t p, int64_t tbase, int lane, double Tq,
                                                 double unit, int delta, float* lo, float* hi, float* cen,
                                                 float* smin, float* smax, double lam_lo, double lam_hi, int nrep) {
  float sc = 0.f, sl = 0.f, sh = 0.f, mn = INFINITY, mx = -INFINITY;
  bool zero = false;
#pragma unroll 1
  for (int rep = 0; rep < nrep; ++rep) {
    float l, h, c, a, b;
    sample_bracket1(P, p, tbase, lane, Tq, unit, delta, &l, &h, &c, &a, &b, lam_lo, lam_hi, rep, nrep);
    zero |= lam_hi > lam_lo && l <= 0.f && h >= 0.f;
    sc += c;
    sl += c - l;
    sh += h - c;
    mn = fminf(mn, a);
    mx = fmaxf(mx, b);
  }
  const float inv = 1.f / (float)nrep, shrink = rsqrtf((float)nrep);
  const float c = sc * inv;
  float l = c - sl * inv * shrink, h = c + sh * inv * shrink;
  if (!(h > l)) {
    const float e = fmaxf(fabsf(c), 1e-30f) * 1e-3f;
    l = c - e;
    h = c + e;
  }
  if (zero) {  // some sample saw the column possibly dead at lam_hi
    l = fminf(l, 0.f);
    h = fmaxf(h, 0.f);
  }
  *lo = l;
  *hi = h;
  *cen = fminf(fmaxf(c, l), h);
  *smin = mn;
  *smax = mx;
}
// TALL (a k_bound template flag, so short columns' kernels never carry the
// accumulators): nrep = n / KB_SREP_ROWS samples, at most KB_SREP_MAX.
__host__ __device__ __forceinline__ int sample_reps(int64_t n) {
  const int64_t q = n / KB_SREP_ROWS;
  return q < 1 ? 1 : (q > KB_SREP_MAX ? KB_SREP_MAX : (int)q);
}
template <bool TALL>
__device__ __forceinline__ void sample_bracket(const SelParams& P, int64_t p, int64_t tbase, int lane, double Tq,
                                               double unit, int delta, float* lo, float* hi, float* cen,
                                               float* smin, float* smax, double lam_lo, double lam_hi) {
  if (TALL)
    sample_bracket_reps(P, p, tbase, lane, Tq, unit, delta, lo, hi, cen, smin, smax, lam_lo, lam_hi,
                        sample_reps(P.n));
  else
    sample_bracket1(P, p, tbase, lane, Tq, unit, delta, lo, hi, cen, smin, smax, lam_lo, lam_hi, 0, 1);
}

// One bounding pass per (pivot, target) problem.  CONT = false: the range
// comes from a row sample (sample_bracket, half-width P.delta ranks).
// CONT = true (refinement for the pivots an earlier pass could not rule out):
// the range is the one the previous pass over the same problem left in
// P.NEXTr (row P.seeds[k] of that pass's pivot list, or k), i.e. where that
// pass proved the optimum lies, so the 62 bins shrink by ~60x per pass and
// the integration error with their square.  Every pass also writes the next
// range (P.NEXTw), the seed range for the exact solver (P.BRK) and the
// per-column bounds (P.LB / P.UB).
//
// Threads: a CTA is 4 pivots (2 pairs) x 64 targets (two 32-target tiles of
// Xft).  Each thread owns FOUR problems: the 2 pivots of its warp's pair x
// targets (lane, 32 + lane) of the tile pair, so one 16-byte broadcast load
// of a row pair's plane records serves 2 x 2 x 32 = 128 ratio elements and
// the shared-memory wavefronts per element drop to 30 / 512 (8 tile loads,
// 6 record loads, 16 atomics per 4-row group).  The 4 warps of a pair
// (quarters) split each chunk's rows (4-row groups q, q + 4) and add into the
// same histograms, so the CTA holds 8 warps for the histogram space of 2.
// SPLIT (few pivots, many rows: a grid too small to fill the GPU): the rows
// are also split over blockIdx.z; every CTA adds its histograms into P.GH
// (exact integer sums, any order), leaves its residual share in P.GE[z] and
// (z = 0) the ranges in P.GB, and k_bound_epi finishes each problem.
template <bool CONT, bool SPLIT, bool MULTI = false, bool TALL = false>
__global__ void __launch_bounds__(kBThreads, 2) k_bound(SelParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned* hist = (unsigned*)(smem + kBStages * kBStage);  // [2 pivots of a pair][kNB][kBSlots]
  __shared__ __align__(8) unsigned long long full[kBStages];
  __shared__ unsigned done[kBStages];   // warps finished with the stage's chunk
  __shared__ float sbr[2][5][kBSlots];  // brackets: problem (t, slot)'s (lo, hi, cen, smin, smax)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp / kBPairs, pair = warp % kBPairs;
  const int tq = quarter & 1, eq = quarter >> 1;  // the problem this thread prepares and finishes
  const int64_t n = P.n, m = P.m, np = P.np;
  const int64_t tile0 = (int64_t)blockIdx.x * 2;  // this CTA's two 32-target tiles of Xft
  const bool tile1 = (tile0 + 1) * 32 < m;         // the second one exists
  const int64_t gbase = (int64_t)blockIdx.y * np * kBPiv;  // this CTA's pivot group in the plane

  // this thread's own problem (tq, eq): bracketed before the main loop and
  // finished after it; its metadata is recomputed there instead of living
  // in registers through the loop
  const int64_t jq = (tile0 + eq) * 32 + lane;
  const int slq = pair * 64 + eq * 32 + lane;
  auto meta = [&](int64_t& k, int64_t& pv, bool& okk, bool& dg, double& T, double& u) {
    k = (int64_t)blockIdx.y * kBPiv + 2 * pair + tq;
    okk = k < P.npiv;
    pv = okk ? pivot_of(P, k) : 0;
    dg = okk && P.nnz[pv] == 0;
    T = okk && !dg ? P.tq[pv] : 0.0;
    u = ldexp(1.0, okk && !dg ? -P.spow[pv] : 0);
  };
  bool busy;  // the warp has a live problem
  {
    bool any = false;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int64_t k = (int64_t)blockIdx.y * kBPiv + 2 * pair + t;
      const bool okk = k < P.npiv;
      const int64_t pv = okk ? pivot_of(P, k) : 0;
      const bool dg = okk && P.nnz[pv] == 0;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t jj = (tile0 + e) * 32 + lane;
        any |= okk && !dg && jj < m && jj != pv;
      }
    }
    busy = __any_sync(0xffffffffu, any);
  }
  {  // each quarter prepares one of the four problems' brackets; all need all
    float b0 = -1.f, b1 = 1.f, b2 = 0.f, b3 = -1.f, b4 = 1.f;
    int64_t k, pv;
    bool okk, dg;
    double T, u;
    meta(k, pv, okk, dg, T, u);
    if (okk && !dg && jq < m && jq != pv) {
      if (CONT) {
        const float2 r = P.NEXTr[(P.seeds ? P.seeds[k] : k) * m + jq];
        b0 = b3 = r.x;
        b1 = b4 = r.y;
        b2 = 0.5f * (r.x + r.y);
      } else {
        sample_bracket<TALL>(P, pv, (tile0 + eq) * np * 32, lane, T, u, P.delta, &b0, &b1, &b2, &b3, &b4,
                       MULTI ? P.lams[0] : lam_of(P, k), MULTI ? P.lams[P.nlam - 1] : lam_of(P, k));
      }
    }
    float* d = &sbr[tq][0][slq];
    d[0] = b0;
    d[kBSlots] = b1;
    d[2 * kBSlots] = b2;
    d[3 * kBSlots] = b3;
    d[4 * kBSlots] = b4;
  }
  const int64_t nall = (n + kBRows - 1) / kBRows;
  const int64_t cb = SPLIT ? nall * blockIdx.z / gridDim.z : 0;  // this CTA's chunks [cb, cb + nch)
  const int64_t nch = SPLIT ? nall * (blockIdx.z + 1) / gridDim.z - cb : nall;
  // stage refill: local chunk c (global cb + c) goes to stage c % kBStages
  auto issue = [&](int64_t c) {
    const int st = (int)(c % kBStages);
    const int64_t i0 = (cb + c) * kBRows;
    unsigned char* base = smem + (size_t)st * kBStage;
    fence_proxy_async();
    mbar_expect_tx(&full[st], (unsigned)(tile1 ? kBStage : kBStage - kBTile));
    bulk_g2s(base, P.Xft + tile0 * np * 32 + i0 * 32, kBTile, &full[st]);
    if (tile1) bulk_g2s(base + kBTile, P.Xft + (tile0 + 1) * np * 32 + i0 * 32, kBTile, &full[st]);
    bulk_g2s(base + 2 * kBTile, P.gbp + (gbase + i0 * kBPiv) * 3 / 4, kBPlane, &full[st]);
  };
  if (tid == 0) {
    for (int s = 0; s < kBStages; ++s) {
      mbar_init(&full[s], 1);
      done[s] = 0u;
    }
    mbar_fence_init();
    for (int64_t c = 0; c < min((int64_t)kBStages, nch); ++c) issue(c);
  }
  for (int x = tid; x < 2 * kNB * kBSlots; x += kBThreads) hist[x] = 0u;
  __syncthreads();
  float cf[2][2], A[2][2], B[2][2];
  unsigned hb[2][2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int sl = pair * 64 + e * 32 + lane;
      const float l = sbr[t][0][sl], h = sbr[t][1][sl];
      cf[t][e] = sbr[t][2][sl];
      A[t][e] = (62.f / 63.f) / (h - l);
      B[t][e] = 0.5f / 63.f - l * A[t][e];
      hb[t][e] = smem_u32(hist + t * kNB * kBSlots + sl) - 0x4B000000u * (unsigned)(kBSlots * 4);
    }
  }

  unsigned fphase = 0;
  double ec[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // this quarter's share of e_j(c) of the four problems
  for (int64_t c = 0; c < nch; ++c) {
    const int st = (int)(c % kBStages);
    mbar_wait(&full[st], (fphase >> st) & 1u);
    fphase ^= 1u << st;
    if (busy) {
      const unsigned char* sb = smem + (size_t)st * kBStage;
      const float* ta = (const float*)sb;  // [2 tiles][kBRows][32]
      // records of this warp's pivot pair: 3 float4 per row pair and pivot pair
      const float4* rec = (const float4*)(sb + 2 * kBTile) + pair * 3;
      float racc[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll kBGUnroll
      for (int r0 = 4 * quarter; r0 < kBRows; r0 += 4 * kBQuarters) {
        float av[2][4];
        float4 yw[4];  // (y0, x0, y1, x1) of row r0 + u
        uint2 wu[4];
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int u = 0; u < 4; ++u) av[e][u] = ta[e * kBRows * 32 + (r0 + u) * 32 + lane];
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {  // row pairs (r0, r0+1), (r0+2, r0+3)
          const float4* rp = rec + ((r0 >> 1) + h2) * (kBPairs * 3);
          const float4 L0 = rp[0], L1 = rp[1], L2 = rp[2];
          yw[2 * h2] = make_float4(L0.x, L0.z, L0.y, L0.w);
          wu[2 * h2] = make_uint2(__float_as_uint(L1.x), __float_as_uint(L1.y));
          yw[2 * h2 + 1] = make_float4(L1.z, L2.x, L1.w, L2.y);
          wu[2 * h2 + 1] = make_uint2(__float_as_uint(L2.z), __float_as_uint(L2.w));
        }
        // both pivots of the pair at once (packed pairs; same bits as scalar)
        unsigned a0[2][4], a1[2][4];
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float2 q = fmul2(make_float2(av[e][u], av[e][u]), make_float2(yw[u].x, yw[u].z));
            const float2 b = ffma2(make_float2(__saturatef(fmaf(q.x, A[0][e], B[0][e])),
                                               __saturatef(fmaf(q.y, A[1][e], B[1][e]))),
                                   make_float2(63.f, 63.f), make_float2(8388608.f, 8388608.f));
            a0[e][u] = hb[0][e] + __float_as_uint(b.x) * (unsigned)(kBSlots * 4);
            a1[e][u] = hb[1][e] + __float_as_uint(b.y) * (unsigned)(kBSlots * 4);
          }
#pragma unroll
        for (int e = 0; e < 2; ++e) {  // |a - c b| (dropped rows: |a|), pairwise within the 4 rows
          float e0[4], e1[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float2 r = ffma2(make_float2(-cf[0][e], -cf[1][e]), make_float2(yw[u].y, yw[u].w),
                                   make_float2(av[e][u], av[e][u]));
            e0[u] = fabsf(r.x);
            e1[u] = fabsf(r.y);
          }
          racc[0][e] += (e0[0] + e0[1]) + (e0[2] + e0[3]);
          racc[1][e] += (e1[0] + e1[1]) + (e1[2] + e1[3]);
        }
        // fire-and-forget shared adds (the other quarters add into the same bins)
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0[e][u]), "r"(wu[u].x));
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a1[e][u]), "r"(wu[u].y));
          }
      }
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e) ec[t][e] += (double)racc[t][e];
    }
    __syncwarp();
    if (lane == 0) {
      // the last warp done with the stage refills it (no producer waits)
      unsigned old;
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                   : "=r"(old)
                   : "r"(smem_u32(&done[st]))
                   : "memory");
      if (old == kBWarps - 1) {
        done[st] = 0u;
        if (c + kBStages < nch) issue(c + kBStages);
      }
    }
  }
  // every chunk has been waited for, so no bulk copy is in flight: the stage
  // buffers carry the quarters' residual shares to the problem's finisher
  __syncthreads();  // also: every quarter's histogram adds are in
  double* ecx = (double*)smem;  // [quarter][t][e][pair][lane]
#pragma unroll
  for (int t = 0; t < 2; ++t)
#pragma unroll
    for (int e = 0; e < 2; ++e) ecx[((quarter * 2 + t) * 2 + e) * (kBPairs * 32) + pair * 32 + lane] = ec[t][e];
  __syncthreads();
  double ect = 0.0;
#pragma unroll
  for (int q = 0; q < kBQuarters; ++q) ect += ecx[((q * 2 + tq) * 2 + eq) * (kBPairs * 32) + pair * 32 + lane];
  const int64_t jj = jq;
  const int sl = slq;
  const float tlo = sbr[tq][0][sl], thi = sbr[tq][1][sl], tcf = sbr[tq][2][sl];
  int64_t kq, pq;
  bool okq, dgq;
  double Tqq, utq;
  meta(kq, pq, okq, dgq, Tqq, utq);
  if (MULTI) {
    // every penalty in P.lams (ascending): the column bounds summed over the
    // warp's 32 targets (one pivot), one atomic per warp and penalty
    const bool live = okq && jj < m && !dgq && jj != pq;
    Prefix H{hist + tq * kNB * kBSlots + sl, kBSlots};
    H.build();  // once for every penalty
    for (int l = 0; l < P.nlam; ++l) {
      double lb = 0.0, ub = 0.0;
      float2 nx = make_float2(tlo, thi);
      if (live) {
        double2 rg;
        column_bounds(H, ldexp(utq, 21), (double)tlo, (double)thi, (double)tcf, ect, Tqq * utq,
                      P.lams[l], P.colsum[jj], n, sbr[tq][3][sl], sbr[tq][4][sl], &lb, &ub, &rg, &nx);
      } else if (okq && jj < m && dgq) {
        lb = ub = P.colsum[jj];  // fit.py:66-72: v = 0, error = sum |x|
      }
      // each penalty's next range, for a continuing pass per (penalty, pivot) entry
      if (P.NEXTm && okq && jj < m) P.NEXTm[((int64_t)l * P.npiv + kq) * m + jj] = nx;
      lb = warp_sum(lb);
      ub = warp_sum(ub);
      if (lane == 0 && okq) {
        atomicAdd(&P.LBm[l * P.npiv + kq], lb);
        atomicAdd(&P.UBm[l * P.npiv + kq], ub);
      }
    }
    return;
  }
  if (jj >= m || !okq) return;
  const int64_t o = kq * m + jj;
  if (SPLIT) {
    const unsigned* hc = hist + tq * kNB * kBSlots + sl;
    for (int b = 0; b < kNB; ++b) {
      const unsigned x = hc[b * kBSlots];
      if (x) atomicAdd(&P.GH[o * kNB + b], x);
    }
    P.GE[(int64_t)blockIdx.z * P.npiv * m + o] = ect;
    if (blockIdx.z == 0) {
      float* g = P.GB + o * 5;
      g[0] = tlo;
      g[1] = thi;
      g[2] = tcf;
      g[3] = sbr[tq][3][sl];
      g[4] = sbr[tq][4][sl];
    }
    return;
  }
  if (dgq || jj == pq) {
    const double z = dgq ? P.colsum[jj] : 0.0;  // fit.py:66-72: v = 0, error = sum |x|
    P.LB[o] = z;
    P.UB[o] = z;
    P.BRK[o] = make_double2(-INFINITY, INFINITY);
    P.NEXTw[o] = make_float2(tlo, thi);
    return;
  }
  double lb, ub;
  Prefix H{hist + tq * kNB * kBSlots + sl, kBSlots};
  H.build();
  column_bounds(H, ldexp(utq, 21), (double)tlo, (double)thi, (double)tcf, ect, Tqq * utq,
                lam_of(P, kq), P.colsum[jj], n, sbr[tq][3][sl], sbr[tq][4][sl], &lb, &ub, &P.BRK[o], &P.NEXTw[o]);
  P.LB[o] = lb;
  P.UB[o] = ub;
}

// Epilogue of a SPLIT k_bound: thread per (pivot, target) problem, the
// merged histogram, the residual shares summed in z order, column_bounds.
__global__ void k_bound_epi(SelParams P, int nsplit) {
  const int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t m = P.m;
  if (o >= P.npiv * m) return;
  const int64_t kk = o / m, j = o - kk * m, p = pivot_of(P, kk);
  const float* g = P.GB + o * 5;
  if (P.nnz[p] == 0 || j == p) {
    const double z = P.nnz[p] == 0 ? P.colsum[j] : 0.0;
    P.LB[o] = z;
    P.UB[o] = z;
    P.BRK[o] = make_double2(-INFINITY, INFINITY);
    P.NEXTw[o] = make_float2(g[0], g[1]);
    return;
  }
  double ec = 0.0;
  for (int z = 0; z < nsplit; ++z) ec += P.GE[(int64_t)z * P.npiv * m + o];
  const double ut = ldexp(1.0, -P.spow[p]);
  double lb, ub;
  Prefix H{P.GH + o * kNB, 1};
  H.build();
  column_bounds(H, ldexp(ut, 21), (double)g[0], (double)g[1], (double)g[2], ec, P.tq[p] * ut,
                lam_of(P, kk), P.colsum[j], P.n, g[3], g[4], &lb, &ub, &P.BRK[o], &P.NEXTw[o]);
  P.LB[o] = lb;
  P.UB[o] = ub;
}

// Penalty of v_p = 1 for every pivot and penalty of a multi-penalty pass.
__global__ void k_bound_finish(SelParams P, double* __restrict__ lb, double* __restrict__ ub) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.npiv * P.nlam) return;
  const int64_t l = t / P.npiv, kk = t - l * P.npiv;
  const double pen = P.nnz[pivot_of(P, kk)] ? P.lams[l] : 0.0;
  lb[t] += pen;
  ub[t] += pen;
}
