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
// Layout: a CTA is 4 pivots x 64 targets (256 problems) in 8 warps, two CTAs
// per SM (KB_TGT = 128: 16 warps, one CTA per SM -- slower, kept as a build
// option).  A thread owns EIGHT problems, the four pivots x two targets
// (lane, lane + 32); the 8 warps split each 64-row chunk's rows.  Per row a
// thread loads its two x_ij (one 8-byte load) and the four pivots' (y | x | w)
// records (three broadcast 16-byte loads) and does 8 ratio elements, so the
// shared-memory pipe carries 8 atomics + 2 tile + 3 record wavefronts per 256
// elements (k_bound below).

#ifndef KB_TGT
#define KB_TGT 64   // targets per CTA: 64 (8 warps, 2 CTAs per SM) or 128 (16 warps, 1 CTA per SM)
#endif
constexpr int kBPiv = 4;                   // pivots per CTA (k_group_bound's plane groups)
constexpr int kBTgt = KB_TGT;              // targets per CTA
constexpr int kBE = kBTgt / 32;            // 32-target tiles per CTA
constexpr int kBTE = 2;                    // tiles (targets) per thread
constexpr int kBTH = kBE / kBTE;           // target halves
constexpr int kBProb = kBPiv * kBTgt;      // problems per CTA
constexpr int kBThreads = kBProb;          // one problem per thread in the prologue and epilogue
constexpr int kBWarps = kBThreads / 32;
constexpr int kBRG = kBWarps / kBTH;       // row groups (warps per target half)
constexpr int kBMinBlocks = kBTgt == 64 ? 2 : 1;
#ifndef KB_ROWS
#define KB_ROWS 64
#endif
#ifndef KB_STAGES
#define KB_STAGES 2
#endif
#ifndef KB_FLUSH
#define KB_FLUSH (256 / KB_ROWS)  // chunks between FP32 -> FP64 residual flushes (<= 16 row pairs, see below)
#endif
constexpr int kBRows = KB_ROWS;            // rows per staged chunk
constexpr int kBRowsW = kBRows / kBRG;     // rows per warp per chunk
constexpr int kBTile = kBRows * kBTgt * 4;  // the rows' x_ij of the CTA's targets (k_tile's xq order)
constexpr int kBPlane = kBRows * kBPiv * 12;  // k_group_bound records: 48 B per row
constexpr int kBStage = kBTile + kBPlane;
constexpr int kBStages = KB_STAGES;
constexpr int kBHist = kBPiv * kNB * kBTgt * 4;  // [pivot][bin][target slot], exact 32-bit sums
static_assert(kBPiv == kGroupBoundPiv, "k_bound reads k_group_bound's plane groups");
static_assert(kBTgt == 64 || kBTgt == 128, "k_tile lays out 64- or 128-target groups");
static_assert(kBRowsW % 2 == 0 && kBRows % kBRG == 0, "a warp takes whole row pairs of a chunk");
static_assert(KB_FLUSH * kBRowsW <= 32, "residual summation margin (column_bounds) covers 16 row pairs per flush");
static_assert(kBStages * kBStage >= kBRG * kBProb * 8, "stage buffers hold the warps' residual shares");
constexpr int kBLamGroup = 4;              // penalties per pivot-sum round of a multi-penalty epilogue
constexpr size_t kBoundSmem = (size_t)kBStages * kBStage + kBHist;
// bracket half-width in sample ranks: narrow for the one-pass bound (tight
// bins), wider when later passes refine it (fewer optima outside)
#ifndef KB_DELTA1
#define KB_DELTA1 8
#endif
#ifndef KB_DELTAN
#define KB_DELTAN 10
#endif
// the steering pass over a row sample (tall data): its histogram only has to
// locate the crossing, so a slightly narrower bracket pays (C4 40.4 -> 39.1 ms
// at 9 ranks; 6 ranks falls off a cliff: too many crossings outside)
#ifndef KB_DELTAS
#define KB_DELTAS 9
#endif
constexpr int kBDelta1 = KB_DELTA1, kBDeltaN = KB_DELTAN, kBDeltaS = KB_DELTAS;

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
  // static indices only (a select chain and predicated loads): the struct stays
  // in registers, so h keeps its address space (shared loads, no stack frame)
  __device__ __forceinline__ unsigned long long sc(int k) const {
    const int b = k >> 3, q0 = k & ~7;
    unsigned long long s = sc8[0];
#pragma unroll
    for (int i = 1; i < 8; ++i) s = b == i ? sc8[i] : s;
#pragma unroll
    for (int d = 0; d < 7; ++d)
      if (q0 + d < k) s += h[(q0 + d) * hs];
    return s;
  }
};

// Bounds of one column optimum, split into the penalty-free setup (margins,
// edge signs, the prefix sums around the sample centre) and the per-penalty
// part, so a multi-penalty pass sets a column up once (ColumnBounds::at).
struct ColumnBounds {
  const Prefix& H;
  double q, lo, hi, c, ec, T, colsum;
  double w, dC, pert, eps, iq2, q2, dc, f0e, f0;
  int z0, z1, kc;
  long long CuC, SCC, CuC1, Cu0, Cu62, SC62;

  __device__ __forceinline__ double edge(int k) const { return lo + (double)k * w; }

  __device__ __forceinline__ ColumnBounds(const Prefix& H_, double q_, double lo_, double hi_, double c_, double ec_,
                                          double T_, double colsum_, int64_t n)
      : H(H_), q(q_), lo(lo_), hi(hi_), c(c_), ec(ec_), T(T_), colsum(colsum_) {
    w = (hi - lo) / (double)kNI;
    // margins: the 32-bit weights are within q/2 of |x_ip| each (so any
    // cumulative weight within n q / 2), the residual terms within 2^-22 of
    // |a| + |c b|, and their per-chunk float sums
    dC = 0.5000001 * (double)n * q;
    // every row's float ratio (and the float bin edges) sit within pert / w_i
    // of its binned position, so f moves by at most pert when the rows are
    // moved into their bins; the bounds below hold for that moved problem
    pert = 0x1p-22 * colsum + T * (0x1p-21 * (fabs(lo) + fabs(hi)) + 0x1p-20 * w);
    // (k_bound: each thread's FP32 accumulator adds <= 16 two-row sums of
    // nonnegative terms between FP64 flushes, KB_FLUSH: relative error <= 17 u)
    eps = 0x1p-22 * (colsum + fabs(c) * T) + 20.0 * 0x1p-24 * ec + pert;
    // edges e_k = lo + k w (k = 0..62); C_k = q Cu_k = weight with r < e_k
    // (slots 0..k).  The subgradient bounds at edge k are
    //   glo(k) = 2 (C_k - dC) - T + lam sp(k) <= g(e_k+),  sp(k) = e_k >= 0 ? 1 : -1,
    //   ghi(k) = 2 (C_k + dC) - T + lam sm(k) >= g(e_k-),  sm(k) = e_k >  0 ? 1 : -1,
    // on bin [e_k, e_k+1] g lies in [glo(k), ghi(k+1)], and their integrals
    //   Ilo(k) = sum_{q<k} w glo(q),  Ihi(k) = sum_{q<k} w ghi(q+1)
    // need only the exact integer prefix sums Cu_k, SC_k = sum_{q<k} Cu_q and
    // the edge-sign counts, so the walk over the edges is integer-only.
    z0 = min(kNB - 1, max(0, (int)ceil(-lo / w)));  // edges e_0 .. e_z0-1 are < 0
    while (z0 > 0 && edge(z0 - 1) >= 0.0) --z0;
    while (z0 < kNB - 1 && edge(z0) < 0.0) ++z0;
    z1 = z0;  // edges e_0 .. e_z1-1 are <= 0
    while (z1 < kNB - 1 && edge(z1) <= 0.0) ++z1;
    kc = min(kNI - 1, max(0, (int)floor((c - lo) / w)));
    iq2 = 0.5 / q;
    q2 = 2.0 * q;
    CuC = H.cu(kc);
    SCC = (long long)H.sc(kc);
    CuC1 = H.cu(kc + 1);
    Cu0 = H.cu(0);
    Cu62 = H.cu(kNI);
    SC62 = (long long)H.sc(kNI);
    dc = c - edge(kc);
    // f(0) = sum_i |x_ij|: the dead value; colsum carries the rounding of an
    // n-term f64 sum (any order): within (n + 128) 2^-53 of it
    f0e = (double)(n + 128) * 0x1p-53 * colsum;
    f0 = colsum - f0e;  // a lower bound of f(0) (the kink bounds below)
  }

  __device__ __forceinline__ void at(double lam, float smin, float smax, double* lbo, double* ubo, double2* range,
                                     float2* next) const {
    const double fc = ec + lam * fabs(c);
    // integer thresholds, rounded so that passing them implies the double test:
    // ghi(k) <= 0 <=> Cu_k <= (T - 2 dC - lam sm) / 2q;  glo(k) >= 0 <=> Cu_k >= (T + 2 dC - lam sp) / 2q
    // (Cu_k < 2^32: a threshold is "none pass" / "all pass" outside [0, 2^32 - 1])
    auto xle = [&](double x) { return x * iq2 * (1.0 - 0x1p-44) - 0x1p-8; };
    auto xge = [&](double x) { return x * iq2 * (1.0 + 0x1p-44) + 0x1p-8; };
    const double xLm = xle(T - 2.0 * dC + lam), xLp = xle(T - 2.0 * dC - lam);  // sm = -1 / +1
    const double xRm = xge(T + 2.0 * dC + lam), xRp = xge(T + 2.0 * dC - lam);  // sp = -1 / +1
    // kL = last edge with ghi <= 0, kR = first with glo >= 0: Cu_k grows and
    // the thresholds only drop at the sign change, so both tests are monotone
    // in k and two bisections over the prefix sums find them
    const bool hasL_m = xLm >= 0.0, hasL_p = xLp >= 0.0;
    const unsigned uLm = __double2uint_rd(fmin(xLm, 4294967295.0)), uLp = __double2uint_rd(fmin(xLp, 4294967295.0));
    const bool hasR_m = xRm <= 4294967295.0, hasR_p = xRp <= 4294967295.0;
    const unsigned uRm = __double2uint_ru(fmax(xRm, 0.0)), uRp = __double2uint_ru(fmax(xRp, 0.0));
    auto pL = [&](int k) {
      const unsigned cu = H.cu(k);
      return k >= z1 ? (hasL_p & (cu <= uLp)) : (hasL_m & (cu <= uLm));
    };
    auto pR = [&](int k) {
      const unsigned cu = H.cu(k);
      return k >= z0 ? (hasR_p & (cu >= uRp)) : (hasR_m & (cu >= uRm));
    };
    // fixed six-step bisections over edges 0..62 (branch-free): kL in [-1, 62]
    // (pL holds up to it), kR in [0, 63] (pR holds from it; 63 = kNI + 1: not
    // in the bracket)
    static_assert(kNI + 1 == 63, "six steps cover edges -1..62");
    int kL = -1, kR = -1;
#pragma unroll
    for (int st = 32; st; st >>= 1) {
      kL = pL(kL + st) ? kL + st : kL;
      kR = pR(kR + st) ? kR : kR + st;
    }
    ++kR;
    const long long CuL = kL >= 0 ? (long long)H.cu(kL) : 0, SCL = kL >= 0 ? (long long)H.sc(kL) : 0;
    const long long CuR = kR <= kNI ? (long long)H.cu(kR) : 0, SCR = kR <= kNI ? (long long)H.sc(kR) : 0;
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
    const double fkc_lo = fc - dc * ghiC, fkc_hi = fc - dc * gloC;
    auto f_lo = [&](int k, long long SC, long long Cu) {
      return k >= kc ? fkc_lo + (Ilo(k, SC) - IloC) : fkc_lo - (IhiC - Ihi(k, SC, Cu));
    };
    auto f_hi = [&](int k, long long SC, long long Cu) {
      return k >= kc ? fkc_hi + (Ihi(k, SC, Cu) - IhiC) : fkc_hi - (IloC - Ilo(k, SC));
    };
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
    if (range) {
      if (kL >= 0 && kR <= kNI && kL <= kR) {
        const double d = 0x1p-19 * (fabs(eL) + fabs(eR) + fabs(lo) + fabs(hi)) + 0x1p-10 * w;
        *range = make_double2(eL - d, eR + d);
      } else {
        *range = make_double2(-INFINITY, INFINITY);
      }
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
};

__device__ __forceinline__ void column_bounds(const Prefix& H, double q, double lo, double hi, double c,
                                              double ec, double T, double lam, double colsum, int64_t n,
                                              float smin, float smax, double* lbo, double* ubo, double2* range,
                                              float2* next) {
  ColumnBounds(H, q, lo, hi, c, ec, T, colsum, n).at(lam, smin, smax, lbo, ubo, range, next);
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
  // weights quantised to a byte against 4x the pivot's mean weight (they only
  // steer the bracket), so each key is built as its row arrives
  const double tw = Tq * unit;
  const float wsc = tw > 0.0 ? (float)(255.0 * (double)P.nnz[p] / (4.0 * tw)) : 0.f;
  unsigned key[kSample];
  // rows (2 (s nrep + rep) + 1) n / (64 nrep), in float (any rows would do;
  // a 64-bit division by the runtime nrep would cost a register-hungry call)
  const float rstep = (float)n / (float)(2 * kSample * nrep);
#pragma unroll
  for (int s = 0; s < kSample; ++s) {
    const int64_t r = min(n - 1, (int64_t)((float)(2 * (s * nrep + rep) + 1) * rstep));
    const float2 f = P.pf[p * P.np + r];
    const float wq = fminf(255.f, fabsf(f.y) * wsc);
    key[s] = (f2key(P.Xft[tbase + r * 32 + lane] * f.x) & 0xffffff00u) | (unsigned)__float2uint_rn(wq);
  }
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

// Steering (P.steer = s): the histogram of a 1-in-s chunk sample of the rows
// locates where the column's lambda-shifted weighted median lies; the next
// pass brackets that location widened by the sample's error, so its 62 bins
// are several times narrower than a 32-row sample's bracket allows (tall
// data, where one pass cannot prune deflated components).  Only steers: any
// range gives rigorous bounds in the pass that uses it.
//   Sample weight T_s (exact sum of the sampled u32 weights), penalty scaled
//   to the sample, lam_s = lam T_s / T; the crossing's cumulative weight lies
//   in [(T_s - lam_s) / 2, (T_s + lam_s) / 2] (both signs of v, and the dead
//   zone between), widened by delta = 3 T_s / sqrt(n_s) for the sampling
//   error of a weighted quantile (n_s = nnz / s sampled rows).
__device__ __forceinline__ float2 steer_range(const Prefix& H, float lo, float hi, double lam, double T, long long nnz,
                                              int s, double q, float smin, float smax) {
  const unsigned tot = H.cu(kNB - 1);
  const float span = hi - lo;
  if (tot == 0u) return make_float2(lo, hi);
  const double Ts = q * (double)tot;
  const double ns = fmax(1.0, (double)nnz / (double)s);
  const double lam_s = T > 0.0 ? lam * Ts / T : 0.0;
  const double delta = 3.0 * Ts / sqrt(ns);
  const double glo = 0.5 * (Ts - lam_s) - delta, ghi = 0.5 * (Ts + lam_s) + delta;
  // smallest k with C_k >= g: the crossing lies below edge k (slot k)
  auto first_ge = [&](double g) {
    int a = -1, b = kNB - 1;  // C at slot kNB - 1 is the total
    while (b - a > 1) {
      const int mid = (a + b) >> 1;
      if (q * (double)H.cu(mid) >= g) b = mid;
      else a = mid;
    }
    return b;
  };
  const int ka = first_ge(glo), kb = first_ge(ghi);
  const double w = ((double)hi - (double)lo) / (double)kNI;
  float a = ka <= 0 ? fminf(smin, lo) - 2.f * span : (float)((double)lo + (double)(ka - 1) * w);
  float b = kb >= kNI + 1 ? fmaxf(smax, hi) + 2.f * span : (float)((double)lo + (double)kb * w);
  const float mg = 0.02f * (b - a);
  a -= mg;
  b += mg;
  if (!(b > a)) b = a + fmaxf(fabsf(a), 1e-30f) * 1e-6f;
  return make_float2(a, b);
}

// One bounding pass per (pivot, target) problem.  CONT = false: the range
// comes from a row sample (sample_bracket, half-width P.delta ranks).
// CONT = true (refinement for the pivots an earlier pass could not rule out):
// the range is the one the previous pass over the same problem left in
// P.NEXTr (row P.seeds[k] of that pass's pivot list, or k), i.e. where that
// pass proved the optimum lies, so the 62 bins shrink by ~60x per pass and
// the integration error with their square.
//
// Outputs: every pass adds its column bounds, rounded outward to the
// fixed-point grid 2^-fxk, into the per-pivot integer sums P.LBq / P.UBq
// (exact, so independent of the order CTAs finish in; k_bound_finish turns
// them into per-pivot bounds).  Every pass also writes per problem the next
// range (P.NEXTw, 8 bytes) and, unless P.lean, the seed range for the exact
// solver (P.BRK) and the column bounds (P.LB / P.UB): a lean first pass over
// every pivot skips those 32 bytes per problem (the continuing passes over
// the few survivors write them).  MULTI: every penalty of P.lams gets its own epilogue (the
// histogram is penalty-free), the sums go to row l of LBq / UBq and the next
// ranges (if P.NEXTm) to NEXTm[l].
//
// Threads: a CTA is 4 pivots x 128 targets (four 32-target tiles of Xft), 16
// warps.  Warp w works on target half th = w % 2 (tiles 2 th, 2 th + 1) and
// rows rg * 4 .. rg * 4 + 3 (rg = w / 2) of every 32-row chunk; a thread owns
// the eight problems (pivot t, tile e of its half) of its lane and adds into
// the CTA's histograms ([pivot][bin][e * 32 + lane]: every atomic instruction
// touches 32 consecutive words, one per bank).  Prologue and epilogue: thread
// tid prepares and finishes problem q = tid = t * 128 + e * 32 + lane.
// SPLIT (few pivots, many rows: a grid too small to fill the GPU): the rows
// are also split over blockIdx.z; every CTA adds its histograms into P.GH
// (exact integer sums, any order), leaves its residual share in P.GE[z] and
// (z = 0) the ranges in P.GB, and k_bound_epi finishes each problem.
template <bool CONT, bool SPLIT, bool MULTI = false, bool TALL = false>
__global__ void __launch_bounds__(kBThreads, kBMinBlocks) k_bound(SelParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned* hist = (unsigned*)(smem + kBStages * kBStage);  // [kBPiv][kNB][kBTgt]
  __shared__ __align__(8) unsigned long long full[kBStages];   // chunk landed (TMA transaction count)
  __shared__ unsigned done[kBStages];      // warps finished with the stage's chunk
  __shared__ float sbr[5][kBProb];         // problem q: (lo, hi, cen, smin, smax)
  __shared__ unsigned long long psum[kBWarps][2];  // per-warp pivot sums (lb, ub)
  __shared__ unsigned long long psumg[MULTI ? kBWarps : 1][kBLamGroup][2];  // the same per penalty group
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int th = warp % kBTH, rg = warp / kBTH;
  const int64_t n = P.n, m = P.m, np = P.np;
  // CTA -> (target group bx, pivot group by).  Plain order is target-group
  // fastest; when the target tiles outgrow L2 (tall and wide data) the groups
  // are cut into bands of P.band target groups, pivot-group-major inside a
  // band, so the CTAs resident together share one band's tiles in L2 instead
  // of each pulling a different tile from HBM
  int64_t bx, by;
  {
    const int64_t T = gridDim.x, G = gridDim.y, L = (int64_t)blockIdx.y * T + blockIdx.x;
    const int64_t B = min((int64_t)P.band, T), band = L / (B * G), rem = L - band * B * G;
    const int64_t bw = min(B, T - band * B);
    by = rem / bw;
    bx = band * B + rem % bw;
  }
  const int64_t tile0 = bx * kBE;    // this CTA's first 32-target tile of Xft
  const int64_t gbase = by * np;     // this CTA's pivot group in the plane (rows)

  // the metadata of this thread's epilogue problem q = tid
  const int qt = tid / kBTgt, qs = tid % kBTgt;  // pivot, target slot (e * 32 + lane)
  const int64_t qk = by * kBPiv + qt;
  const int64_t qj = tile0 * 32 + qs;
  auto meta = [&](int64_t& pv, bool& okk, bool& dg, double& T, double& u) {
    okk = qk < P.npiv;
    pv = okk ? pivot_of(P, qk) : 0;
    dg = okk && P.nnz[pv] == 0;
    T = okk && !dg ? P.tq[pv] : 0.0;
    u = ldexp(1.0, okk && !dg ? -P.spow[pv] : 0);
  };
  const int64_t nall = (n + kBRows - 1) / kBRows;
  const int64_t cb = SPLIT ? nall * blockIdx.z / gridDim.z : 0;  // this CTA's chunks [cb, cb + nch)
  // a steering pass (P.steer = s > 1, never SPLIT) takes every s-th chunk
  const int64_t cstep = !SPLIT && P.steer > 1 ? P.steer : 1;
  const int64_t nch = SPLIT ? nall * (blockIdx.z + 1) / gridDim.z - cb : (nall + cstep - 1) / cstep;
  // stage refill: local chunk c (global cb + c) goes to stage c % kBStages
  // (no proxy fence in the loop: the ring is only ever read by generic
  // loads there, and a fence would drain the issuing warp's histogram atomics)
  auto issue = [&](int64_t c) {
    const int st = (int)(c % kBStages);
    const int64_t i0 = (cb + c * cstep) * kBRows;
    unsigned char* base = smem + (size_t)st * kBStage;
    mbar_expect_tx(&full[st], (unsigned)(kBTile + kBPlane));
    bulk_g2s(base, P.Xq + (bx * np + i0) * kBTgt, kBTile, &full[st]);
    bulk_g2s(base + kBTile, P.gbp + (gbase + i0) * 3, kBPlane, &full[st]);
  };
  if (tid == 0) {
    for (int s = 0; s < kBStages; ++s) {
      mbar_init(&full[s], 1);
      done[s] = 0u;
    }
    mbar_fence_init();
    fence_proxy_async();
    for (int64_t c = 0; c < min((int64_t)kBStages, nch); ++c) issue(c);
  }
  {  // bracket of problem tid while the first chunks are in flight
    float b0 = -1.f, b1 = 1.f, b2 = 0.f, b3 = -1.f, b4 = 1.f;
    int64_t pv;
    bool okk, dg;
    double T, u;
    meta(pv, okk, dg, T, u);
    if (okk && !dg && qj < m && qj != pv) {
      if (CONT) {
        const float2 r = P.NEXTr[(P.seeds ? P.seeds[qk] : qk) * m + qj];
        b0 = b3 = r.x;
        b1 = b4 = r.y;
        b2 = 0.5f * (r.x + r.y);
      } else {
        sample_bracket<TALL>(P, pv, (qj >> 5) * np * 32, lane, T, u, P.delta, &b0, &b1, &b2, &b3, &b4,
                             MULTI ? P.lams[0] : lam_of(P, qk), MULTI ? P.lams[P.nlam - 1] : lam_of(P, qk));
      }
    }
    sbr[0][tid] = b0;
    sbr[1][tid] = b1;
    sbr[2][tid] = b2;
    sbr[3][tid] = b3;
    sbr[4][tid] = b4;
  }
  for (int x = tid; x < kBPiv * kNB * kBTgt; x += kBThreads) hist[x] = 0u;
  __syncthreads();
  // this thread's eight problems: bin map t = sat(r A + B) (63 t + 2^23 has
  // the bin in its low bits), residual reference point c
  float A[kBPiv][kBTE], B[kBPiv][kBTE];
  float2 nc[kBPiv / 2][kBTE];  // (-c_{2h}, -c_{2h+1}) as a register pair for FFMA2
#pragma unroll
  for (int t = 0; t < kBPiv; ++t)
#pragma unroll
    for (int ee = 0; ee < kBTE; ++ee) {
      const int q = t * kBTgt + (th * kBTE + ee) * 32 + lane;
      const float l = sbr[0][q], hh = sbr[1][q];
      A[t][ee] = (62.f / 63.f) / (hh - l);
      B[t][ee] = 0.5f / 63.f - l * A[t][ee];
      if (t & 1) nc[t >> 1][ee].y = -sbr[2][q];
      else nc[t >> 1][ee].x = -sbr[2][q];
    }
  // bin b of (t, e) -> hist + ((t * kNB + b) * kBTgt + e * 32 + lane) words;
  // 63 t + 2^23 has bits 0x4B000000 + b
  const unsigned hb = smem_u32(hist + th * kBTE * 32 + lane) - 0x4B000000u * (unsigned)(kBTgt * 4);

  unsigned fphase = 0;
  float2 racc[kBPiv / 2][kBTE];  // (pivot 2h, pivot 2h + 1) pairs: one FADD2 per row
  double ec[kBPiv][kBTE];  // this warp's share of e_j(c) of the eight problems
#pragma unroll
  for (int t = 0; t < kBPiv; ++t)
#pragma unroll
    for (int ee = 0; ee < kBTE; ++ee) {
      if (t % 2 == 0) racc[t / 2][ee] = make_float2(0.f, 0.f);
      ec[t][ee] = 0.0;
    }
  int nflush = 0;
  const bool e1_dead = (tile0 + th * kBTE + 1) * 32 >= m;  // targets of slot e = 1 all past column m - 1
  for (int64_t c = 0; c < nch; ++c) {
    const int st = (int)(c % kBStages);
    mbar_wait(&full[st], (fphase >> st) & 1u);
    fphase ^= 1u << st;
    const unsigned char* sb = smem + (size_t)st * kBStage;
    const float2* ta = (const float2*)sb + th * 32 + lane;  // [kBRows][half][lane]: this thread's two targets
    const float4* rec = (const float4*)(sb + kBTile);       // [kBRows][3]
    // the thread's second target slot past the last column (the ragged last
    // group): a warp-uniform half-width body
    auto rows = [&](auto ne) {
      constexpr int NE = decltype(ne)::value;
#pragma unroll
      for (int u2 = 0; u2 < kBRowsW; u2 += 2) {
        float2 rr[2][kBPiv / 2][kBTE];  // x_ij - c x_ip of the row pair, pivots (2h, 2h + 1)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int r = rg * kBRowsW + u2 + v;
          static_assert(kBTE == 2, "one 8-byte load per row");
          const float2 xv = ta[r * (kBTgt / 2)];
          const float x[kBTE] = {xv.x, xv.y};
          const float4 Y = rec[r * 3], X = rec[r * 3 + 1], W = rec[r * 3 + 2];
#pragma unroll
          for (int h = 0; h < kBPiv / 2; ++h) {
            const float2 yy = h ? make_float2(Y.z, Y.w) : make_float2(Y.x, Y.y);
            const float2 xx = h ? make_float2(X.z, X.w) : make_float2(X.x, X.y);
            const unsigned w0 = __float_as_uint(h ? W.z : W.x), w1 = __float_as_uint(h ? W.w : W.y);
#pragma unroll
            for (int ee = 0; ee < NE; ++ee) {
              const float2 q = fmul2(make_float2(x[ee], x[ee]), yy);
              const float2 bb = ffma2(make_float2(__saturatef(fmaf(q.x, A[2 * h][ee], B[2 * h][ee])),
                                                  __saturatef(fmaf(q.y, A[2 * h + 1][ee], B[2 * h + 1][ee]))),
                                      make_float2(63.f, 63.f), make_float2(8388608.f, 8388608.f));
              const unsigned a0 = hb + __float_as_uint(bb.x) * (unsigned)(kBTgt * 4) +
                                  (unsigned)(((2 * h) * kNB * kBTgt + ee * 32) * 4);
              const unsigned a1 = hb + __float_as_uint(bb.y) * (unsigned)(kBTgt * 4) +
                                  (unsigned)(((2 * h + 1) * kNB * kBTgt + ee * 32) * 4);
              // fire-and-forget shared adds (the other warps add into the same bins)
              asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a0), "r"(w0));
              asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a1), "r"(w1));
              // x_ij - c x_ip of both pivots (dropped rows: x_ij)
              rr[v][h][ee] = ffma2(nc[h][ee], xx, make_float2(x[ee], x[ee]));
            }
          }
        }
        // the row pair's |terms| summed first, then added (two FADD2 per four
        // elements; the pair sums keep the accumulation error at 16 u per flush)
#pragma unroll
        for (int h = 0; h < kBPiv / 2; ++h)
#pragma unroll
          for (int ee = 0; ee < NE; ++ee)
            racc[h][ee] = fadd2(racc[h][ee], fadd2(fabs2(rr[0][h][ee]), fabs2(rr[1][h][ee])));
      }
    };
    if (e1_dead) rows(std::integral_constant<int, 1>{});
    else rows(std::integral_constant<int, kBTE>{});
    if (++nflush == KB_FLUSH || c + 1 == nch) {
      nflush = 0;
#pragma unroll
      for (int t = 0; t < kBPiv; ++t)
#pragma unroll
        for (int ee = 0; ee < kBTE; ++ee) {
          ec[t][ee] += (double)(t % 2 ? racc[t / 2][ee].y : racc[t / 2][ee].x);
          if (t % 2) racc[t / 2][ee] = make_float2(0.f, 0.f);
        }
    }
    __syncwarp();
    if (lane == 0) {
      // the last warp done with the stage refills it (no producer waits).
      // Relaxed: this warp's loads of the stage have all returned (their
      // values fed the arithmetic above), and a release here would also
      // wait for the warp's in-flight histogram atomics every chunk.
      unsigned old;
      asm volatile("atom.relaxed.cta.shared::cta.add.u32 %0, [%1], 1;"
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
  // buffers carry the row groups' residual shares to the problems' finishers
  __syncthreads();  // also: every warp's histogram adds are in
  double* ecx = (double*)smem;  // [row group][q]
#pragma unroll
  for (int t = 0; t < kBPiv; ++t)
#pragma unroll
    for (int ee = 0; ee < kBTE; ++ee) ecx[rg * kBProb + t * kBTgt + (th * kBTE + ee) * 32 + lane] = ec[t][ee];
  __syncthreads();
  const int fx = P.fxk ? *P.fxk : 0;
  // x 2^fx as one multiply (exact for normal results, as ldexp; an upper
  // bound whose scaled value underflows still rounds up to 1)
  const double fxs = ldexp(1.0, fx);
  auto fx_down = [&](double x) { return (unsigned long long)__double2ull_rd(x * fxs); };
  auto fx_up = [&](double x) {
    const unsigned long long r = __double2ull_ru(x * fxs);
    return (unsigned long long)(r == 0ull && x > 0.0 ? 1ull : r);
  };
  double ect = 0.0;
#pragma unroll
  for (int g = 0; g < kBRG; ++g) ect += ecx[g * kBProb + tid];
  const float tlo = sbr[0][tid], thi = sbr[1][tid], tcf = sbr[2][tid];
  // per-pivot fixed-point sums of one penalty's column bounds (lb rounded
  // down, ub up; both clamped to the column's f(0) bound, which keeps lb a
  // lower bound and the sums below 2^61): warp sums, then the pivot's four
  // warps in a fixed order, one integer atomic per (pivot, CTA)
  auto pivot_sums = [&](double lb, double ub, int64_t row) {
    unsigned long long ql = 0, qu = 0;
    if (P.LBq) {
      ql = fx_down(lb);
      qu = fx_up(ub);
    }
    for (int o = 16; o; o >>= 1) {
      ql += __shfl_xor_sync(0xffffffffu, ql, o);
      qu += __shfl_xor_sync(0xffffffffu, qu, o);
    }
    if (lane == 0) {
      psum[warp][0] = ql;
      psum[warp][1] = qu;
    }
    __syncthreads();
    constexpr int WP = kBWarps / kBPiv;  // warps per pivot (q = tid: pivot t = warp / WP)
    if (P.LBq && tid < kBPiv) {
      const int64_t k = by * kBPiv + tid;
      if (k < P.npiv) {
        unsigned long long sl = 0, su = 0;
        for (int w = tid * WP; w < (tid + 1) * WP; ++w) {
          sl += psum[w][0];
          su += psum[w][1];
        }
        atomicAdd(&P.LBq[row * P.npiv + k], sl);
        atomicAdd(&P.UBq[row * P.npiv + k], su);
      }
    }
    __syncthreads();
  };
  // the same for kBLamGroup penalties at once (multi-penalty passes): one
  // pair of barriers per group instead of per penalty
  auto pivot_sums_group = [&](const double* lb, const double* ub, int l0) {
    static_assert(kBLamGroup == 4, "transposed reduction below");
    unsigned long long ql[kBLamGroup], qu[kBLamGroup];
#pragma unroll
    for (int g = 0; g < kBLamGroup; ++g) {
      ql[g] = fx_down(lb[g]);
      qu[g] = fx_up(ub[g]);
    }
    // transposed butterfly: each exchange halves the penalties a lane keeps,
    // so lane 8g + (any of 0..7) ends with penalty g's warp sum (6 exchanges
    // per quantity instead of 4 x 5; integer sums, order-free)
    const bool b4 = lane & 16, b3 = lane & 8;
    unsigned long long wl[2], wu[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      wl[j] = (b4 ? ql[2 + j] : ql[j]) + __shfl_xor_sync(0xffffffffu, b4 ? ql[j] : ql[2 + j], 16);
      wu[j] = (b4 ? qu[2 + j] : qu[j]) + __shfl_xor_sync(0xffffffffu, b4 ? qu[j] : qu[2 + j], 16);
    }
    unsigned long long sl = (b3 ? wl[1] : wl[0]) + __shfl_xor_sync(0xffffffffu, b3 ? wl[0] : wl[1], 8);
    unsigned long long su = (b3 ? wu[1] : wu[0]) + __shfl_xor_sync(0xffffffffu, b3 ? wu[0] : wu[1], 8);
#pragma unroll
    for (int o = 4; o; o >>= 1) {
      sl += __shfl_xor_sync(0xffffffffu, sl, o);
      su += __shfl_xor_sync(0xffffffffu, su, o);
    }
    if ((lane & 7) == 0) {
      psumg[warp][lane >> 3][0] = sl;
      psumg[warp][lane >> 3][1] = su;
    }
    __syncthreads();
    constexpr int WP = kBWarps / kBPiv;
    if (tid < kBPiv * kBLamGroup) {
      const int t = tid / kBLamGroup, g = tid % kBLamGroup;
      const int64_t k = by * kBPiv + t;
      if (k < P.npiv && l0 + g < P.nlam) {
        unsigned long long sl = 0, su = 0;
        for (int w = t * WP; w < (t + 1) * WP; ++w) {
          sl += psumg[w][g][0];
          su += psumg[w][g][1];
        }
        atomicAdd(&P.LBq[(int64_t)(l0 + g) * P.npiv + k], sl);
        atomicAdd(&P.UBq[(int64_t)(l0 + g) * P.npiv + k], su);
      }
    }
    __syncthreads();
  };
  int64_t pv;
  bool okk, dg;
  double T, u;
  meta(pv, okk, dg, T, u);
  const bool live = okk && qj < m && !dg && qj != pv;
  if (!SPLIT && !MULTI && P.steer > 1) {  // steering pass: the next range only
    if (okk && qj < m) {
      Prefix H{hist + qt * kNB * kBTgt + qs, kBTgt};
      H.build();
      P.NEXTw[qk * m + qj] = live ? steer_range(H, tlo, thi, lam_of(P, qk), T * u, P.nnz[pv], P.steer,
                                                ldexp(u, 21), sbr[3][tid], sbr[4][tid])
                                  : make_float2(tlo, thi);
    }
    return;
  }
  if (MULTI) {
    Prefix H{hist + qt * kNB * kBTgt + qs, kBTgt};
    H.build();  // once for every penalty
    // penalty-invariant per column: loaded once, not per penalty (the stores
    // below could alias them as far as the compiler knows)
    const double csj = okk && qj < m ? P.colsum[qj] : 0.0;
    const float smn = sbr[3][tid], smx = sbr[4][tid];
    float2* nxp = P.NEXTm && okk && qj < m ? P.NEXTm + qk * m + qj : nullptr;
    const int64_t nxs = P.npiv * m;
    const ColumnBounds CB(H, ldexp(u, 21), (double)tlo, (double)thi, (double)tcf, ect, T * u, live ? csj : 0.0, n);
    for (int l0 = 0; l0 < P.nlam; l0 += kBLamGroup) {
      double lbg[kBLamGroup], ubg[kBLamGroup];
#pragma unroll
      for (int g = 0; g < kBLamGroup; ++g) {
        const int l = l0 + g;
        double lb = 0.0, ub = 0.0;
        if (l < P.nlam) {
          float2 nx = make_float2(tlo, thi);
          if (live) {
            CB.at(P.lams[l], smn, smx, &lb, &ub, nullptr, &nx);
            ub = fmin(ub, csj * (1.0 + 0x1p-20));
            lb = fmin(lb, ub);
          } else if (dg) {
            lb = ub = csj;  // fit.py:66-72: v = 0, error = sum |x| (0 past the last target)
          }
          // each penalty's next range, for a continuing pass per (penalty, pivot) entry
          if (nxp) nxp[l * nxs] = nx;
        }
        lbg[g] = lb;
        ubg[g] = ub;
      }
      pivot_sums_group(lbg, ubg, l0);
    }
    return;
  }
  double lbv = 0.0, ubv = 0.0;
  if (okk && qj < m) {
    const int64_t o = qk * m + qj;
    if (SPLIT) {
      const unsigned* hc = hist + qt * kNB * kBTgt + qs;
      for (int b = 0; b < kNB; ++b) {
        const unsigned x = hc[b * kBTgt];
        if (x) atomicAdd(&P.GH[o * kNB + b], x);
      }
      P.GE[(int64_t)blockIdx.z * P.npiv * m + o] = ect;
      if (blockIdx.z == 0) {
        float* g = P.GB + o * 5;
        g[0] = tlo;
        g[1] = thi;
        g[2] = tcf;
        g[3] = sbr[3][tid];
        g[4] = sbr[4][tid];
      }
    } else if (!live) {
      const double z = dg ? P.colsum[qj] : 0.0;  // fit.py:66-72: v = 0, error = sum |x|
      lbv = ubv = z;
      P.NEXTw[o] = make_float2(tlo, thi);
      if (!P.lean) {
        P.LB[o] = z;
        P.UB[o] = z;
        P.BRK[o] = make_double2(-INFINITY, INFINITY);
      }
    } else {
      double2 rg2;
      float2 nx;
      Prefix H{hist + qt * kNB * kBTgt + qs, kBTgt};
      H.build();
      column_bounds(H, ldexp(u, 21), (double)tlo, (double)thi, (double)tcf, ect, T * u, lam_of(P, qk),
                    P.colsum[qj], n, sbr[3][tid], sbr[4][tid], &lbv, &ubv, &rg2, &nx);
      ubv = fmin(ubv, P.colsum[qj] * (1.0 + 0x1p-20));
      lbv = fmin(lbv, ubv);
      P.NEXTw[o] = nx;
      if (!P.lean) {
        P.LB[o] = lbv;
        P.UB[o] = ubv;
        P.BRK[o] = rg2;
      }
    }
  }
  if (!SPLIT) pivot_sums(lbv, ubv, 0);
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

// Per-pivot bounds from k_bound's fixed-point sums (rounded outward) plus
// the penalty of v_p = 1, for every pivot and penalty of the pass.
__global__ void k_bound_finish(SelParams P, double* __restrict__ lb, double* __restrict__ ub) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P.npiv * P.nlam) return;
  const int64_t l = t / P.npiv, kk = t - l * P.npiv;
  const int fx = *P.fxk;
  const double pen = P.nnz[pivot_of(P, kk)] ? (P.lams ? P.lams[l] : lam_of(P, kk)) : 0.0;
  lb[t] = __dadd_rd(ldexp(__ull2double_rd(P.LBq[t]), -fx), pen);
  ub[t] = __dadd_ru(ldexp(__ull2double_ru(P.UBq[t]), -fx), pen);
}
