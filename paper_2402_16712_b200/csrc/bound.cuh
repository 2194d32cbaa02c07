// bound.cuh -- pivot pruning for fit_line (included by l1b200.cu after
// select.cuh).
//
// fit_line (fit.py:88-102) needs only the winning pivot, and most pivots'
// objectives sit far above it.  k_bound runs ONE FP32 pass per (pivot p,
// target j) problem and bounds the column optimum
//     f_j* = min_v e_j(v) + lam |v|,   e_j(v) = sum_i |x_ij - v x_ip|
// from below and above:
//   * the pass histograms the ratios r_i = x_ij / x_ip over the sample bracket
//     (64 slots: below / 62 bins / above, as k_select's first pass) and sums
//     e_j at the sample centre c;
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
// Layout: a CTA is 8 pivots x 32 targets like k_select, but each thread owns
// TWO problems (pivots 2w, 2w+1 of its warp, same target): one load of the
// x_ij tile row and one 16-byte load of both pivots' (y, |x_ip|) serve both
// problems, halving the shared-memory loads per problem, and the two
// histogram read-modify-write chains interleave.

constexpr int kBWarps = 4;                 // warps per k_bound CTA (2 pivots each)
constexpr int kBThreads = kBWarps * 32;
constexpr int kBRows = 64;                 // rows per staged chunk
constexpr int kBTile = kBRows * 32 * 4;    // x_ij float tile [row][32 targets]
constexpr int kBPlane = kBRows * kWarps * 8;   // (y32, w32) [row][8 pivots]
constexpr int kBStage = kBTile + kBPlane;
constexpr int kBStages = 4;
constexpr int kBHist = 2 * kNB * kBThreads * 4;  // [problem][slot][thread]
constexpr size_t kBoundSmem = (size_t)kBStages * kBStage + kBHist;

// Bounds of one column optimum from its histogram h[slot * hs] over the
// bracket [lo, hi) (62 interior bins), e_j(c) = ec, the exact pivot weight T
// and the column's sum_i |x_ij| (f(0)).
__device__ __forceinline__ void column_bounds(const float* h, int hs, double lo, double hi, double c, double ec,
                                              double T, double lam, double colsum, int64_t n, double* lbo,
                                              double* ubo) {
  const double w = (hi - lo) / (double)kNI;
  // float margins: histogram sums (worst case n ulps of T), the residual
  // terms (2^-22 of |a| + |c b|) and their per-chunk float sums
  const double dC = (double)n * 0x1p-24 * T;
  const double eps = 0x1p-22 * (colsum + fabs(c) * T) + 64.0 * 0x1p-24 * ec;
  const double fc = ec + lam * fabs(c);
  // edges e_k = lo + k w (k = 0..62); C_k = weight with r < e_k = slots 0..k
  auto edge = [&](int k) { return lo + (double)k * w; };
  // one walk over the edges: C_k = weight with r < e_k (slots 0..k); the
  // subgradient bounds Glo(k) <= g(e_k+), Ghi(k) >= g(e_k-) are monotone in k,
  // so kL (last edge with Ghi <= 0) and kR (first with Glo >= 0) are seen in
  // order; I(k) = sum_{q<k} w g(q) integrates the per-bin bounds from e_0
  const int kc = min(kNI - 1, max(0, (int)floor((c - lo) / w)));
  int kL = -1, kR = kNB - 1;
  double CL = 0.0, CR = T;
  double Ilo = 0.0, Ihi = 0.0, IloC = 0.0, IhiC = 0.0, IloL = 0.0, IhiL = 0.0, IloR = 0.0, IhiR = 0.0;
  double gloC = 0.0, ghiC = 0.0, gloL = 0.0;
  {
    double C = (double)h[0];
    double ghiE = 2.0 * (C + dC) - T + (edge(0) > 0.0 ? lam : -lam);
    double gloE = 2.0 * (C - dC) - T + (edge(0) >= 0.0 ? lam : -lam);
    for (int k = 0; k <= kNI; ++k) {
      // at edge k: ghiE / gloE are its bounds, C its cumulative weight
      if (ghiE <= 0.0) { kL = k; CL = C; IloL = Ilo; IhiL = Ihi; gloL = gloE; }
      if (kR == kNB - 1 && gloE >= 0.0) { kR = k; CR = C; IloR = Ilo; IhiR = Ihi; }
      if (k == kc) { IloC = Ilo; IhiC = Ihi; }
      if (k == kNI || (kR < kNB - 1 && k > kc)) break;  // everything needed is captured
      const double Cn = C + (double)h[(k + 1) * hs];
      const double ghiN = 2.0 * (Cn + dC) - T + (edge(k + 1) > 0.0 ? lam : -lam);
      const double gloN = 2.0 * (Cn - dC) - T + (edge(k + 1) >= 0.0 ? lam : -lam);
      // g on [e_k, e_k+1] lies in [gloE, ghiN]
      if (k == kc) { gloC = gloE; ghiC = ghiN; }
      Ilo += w * gloE;
      Ihi += w * ghiN;
      C = Cn;
      ghiE = ghiN;
      gloE = gloN;
    }
  }
  // f at e_kc from f(c), then at any edge k from e_kc
  const double dc = c - edge(kc);
  const double fkc_lo = fc - dc * ghiC, fkc_hi = fc - dc * gloC;
  auto f_lo = [&](int k, double Ilk, double Ihk) { return k >= kc ? fkc_lo + (Ilk - IloC) : fkc_lo - (IhiC - Ihk); };
  auto f_hi = [&](int k, double Ilk, double Ihk) { return k >= kc ? fkc_hi + (Ihk - IhiC) : fkc_hi - (IloC - Ilk); };
  const double f0 = colsum;  // f(0): the dead value, exact
  double lb, ub = fmin(fc + eps, f0);
  const double eL = kL >= 0 ? edge(kL) : -INFINITY, eR = kR <= kNI ? edge(kR) : INFINITY;
  if (kL >= 0 && kR <= kNI && kL <= kR) {
    lb = f_lo(kL, IloL, IhiL) - eps + fmin(0.0, gloL) * (eR - eL);
    ub = fmin(ub, fmin(f_hi(kL, IloL, IhiL), f_hi(kR, IloR, IhiR)) + eps);
  } else {
    lb = 0.0;  // the optimum lies beyond the bracket: only the trivial bound
    if (kL == kNI) ub = fmin(ub, f_hi(kNI, Ilo, Ihi) + eps);
  }
  if (eL <= 0.0 && 0.0 <= eR) {
    // the penalty's kink: g(0-) <= 2 W(r < eR) - T - lam, g(0+) >= 2 W(r < eL) - T + lam;
    // f(v) >= f0 + g(0-) v on v <= 0 and f(v) >= f0 + g(0+) v on v >= 0
    const double g0m = 2.0 * (CR + dC) - T - lam, g0p = 2.0 * ((kL >= 0 ? CL : 0.0) - dC) - T + lam;
    const double left = isfinite(eL) ? f0 + fmax(0.0, g0m) * eL : (g0m <= 0.0 ? f0 : 0.0);
    const double right = isfinite(eR) ? f0 + fmin(0.0, g0p) * eR : (g0p >= 0.0 ? f0 : 0.0);
    lb = fmax(lb, fmin(left, right));
  }
  *lbo = fmax(0.0, lb);
  *ubo = ub;
}

// Sample bracket of one problem: float ratios of 32 strided rows, bitonic
// sorted in registers; returns the bracket +-kDelta ranks around the
// estimated crossing and that estimate (the residual's reference point).
__device__ __forceinline__ void sample_bracket(const SelParams& P, int64_t p, int64_t tbase, int lane, double Tq,
                                               double unit, float* lo, float* hi, float* cen) {
  const int64_t n = P.n;
  float sr[kSample], sw[kSample];
#pragma unroll
  for (int s = 0; s < kSample; ++s) {
    const int64_t r = ((2 * s + 1) * n) / (2 * kSample);
    const float2 f = P.pf[p * P.np + r];
    sr[s] = P.Xft[tbase + r * 32 + lane] * f.x;
    sw[s] = fabsf(f.y);
  }
#pragma unroll
  for (int k = 2; k <= kSample; k <<= 1) {
#pragma unroll
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
#pragma unroll
      for (int i = 0; i < kSample; ++i) {
        const int l = i ^ jj;
        if (l > i) {
          const bool up = (i & k) == 0;
          const bool x = up ? (sr[i] > sr[l]) : (sr[i] < sr[l]);
          const float ta = sr[i], tb = sr[l], wa = sw[i], wb = sw[l];
          sr[i] = x ? tb : ta;
          sr[l] = x ? ta : tb;
          sw[i] = x ? wb : wa;
          sw[l] = x ? wa : wb;
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
  const float rho = Tq > 0.0 ? (float)(P.lam / (Tq * unit)) : 0.f;
  const float d = ws > 0.f ? 1.f - 2.f * wn / ws : 1.f;
  const float f = d < -rho ? 0.5f * (1.f + rho) : (d >= rho ? 0.5f * (1.f - rho) : 0.5f);
  const float t = f * ws;
  float c = 0.f;
  int sstar = kSample - 1;
  bool got = false;
#pragma unroll
  for (int s = 0; s < kSample; ++s) {
    c += sw[s];
    if (!got && c > t) { sstar = s; got = true; }
  }
  const int lo_i = max(sstar - kDelta, 0), hi_i = min(sstar + kDelta, kSample - 1);
  float l = 0.f, hh = 0.f, ce = 0.f;
#pragma unroll
  for (int s = 0; s < kSample; ++s) {
    if (s == lo_i) l = sr[s];
    if (s == hi_i) hh = sr[s];
    if (s == sstar) ce = sr[s];
  }
  if (!(hh > l)) {  // degenerate sample: a tiny bracket around it
    const float e = fmaxf(fabsf(l), 1e-30f) * 1e-3f;
    l -= e;
    hh += e;
  }
  *lo = l;
  *hi = hh;
  *cen = fminf(fmaxf(ce, l), hh);
}

__global__ void __launch_bounds__(kBThreads, 2) k_bound(SelParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* hist = (float*)(smem + kBStages * kBStage);  // [2][kNB][kBThreads]
  __shared__ __align__(8) unsigned long long full[kBStages], empty[kBStages];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n = P.n, m = P.m, np = P.np;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const int64_t tbase = (int64_t)blockIdx.x * np * 32;  // this CTA's target tile
  const int64_t gbase = (int64_t)blockIdx.y * np * 8;   // this CTA's pivot group

  int64_t kk[2], p[2];
  bool ok[2], degen[2], act[2];
  double Tq[2], unit[2];
  float lo[2], hi[2], cen[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    kk[t] = (int64_t)blockIdx.y * kWarps + 2 * warp + t;
    ok[t] = kk[t] < P.npiv;
    p[t] = ok[t] ? pivot_of(P, kk[t]) : 0;
    degen[t] = ok[t] && P.nnz[p[t]] == 0;
    act[t] = ok[t] && !degen[t] && j < m && j != p[t];
    Tq[t] = ok[t] && !degen[t] ? P.tq[p[t]] : 0.0;
    unit[t] = ldexp(1.0, ok[t] && !degen[t] ? -P.spow[p[t]] : 0);
    lo[t] = hi[t] = cen[t] = 0.f;
    if (act[t]) sample_bracket(P, p[t], tbase, lane, Tq[t], unit[t], &lo[t], &hi[t], &cen[t]);
    else { lo[t] = -1.f; hi[t] = 1.f; }
  }

  if (tid == 0) {
    for (int s = 0; s < kBStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kBWarps);
    }
    mbar_fence_init();
  }
  float A[2], B[2], cf[2];
  unsigned hb[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    A[t] = (62.f / 63.f) / (hi[t] - lo[t]);
    B[t] = 0.5f / 63.f - lo[t] * A[t];
    cf[t] = cen[t];
#pragma unroll
    for (int b = 0; b < kNB; ++b) hist[(t * kNB + b) * kBThreads + tid] = 0.f;
    hb[t] = smem_u32(hist + t * kNB * kBThreads + tid) - 0x4B000000u * (unsigned)(kBThreads * 4);
  }
  fence_proxy_async();
  __syncthreads();

  const int64_t nch = (n + kBRows - 1) / kBRows;
  unsigned ephase = 0;
  auto issue = [&](int64_t c) {
    if (warp != 0) return;
    const int st = (int)(c % kBStages);
    if (c >= kBStages) {
      mbar_wait(&empty[st], (ephase >> st) & 1u);
      ephase ^= 1u << st;
    }
    if (lane == 0) {
      const int64_t i0 = c * kBRows;
      unsigned char* base = smem + (size_t)st * kBStage;
      fence_proxy_async();
      mbar_expect_tx(&full[st], (unsigned)kBStage);
      bulk_g2s(base, P.Xft + tbase + i0 * 32, kBTile, &full[st]);
      bulk_g2s(base + kBTile, P.gpf + gbase + i0 * 8, kBPlane, &full[st]);
    }
    __syncwarp();
  };
  const bool busy = __any_sync(0xffffffffu, act[0] || act[1]);
  double ec0 = 0.0, ec1 = 0.0;  // e_j(c) of both problems
  unsigned fphase = 0;
  for (int64_t c = 0; c < min((int64_t)(kBStages - 1), nch); ++c) issue(c);
  for (int64_t c = 0; c < nch; ++c) {
    if (c + kBStages - 1 < nch) issue(c + kBStages - 1);
    const int st = (int)(c % kBStages);
    mbar_wait(&full[st], (fphase >> st) & 1u);
    fphase ^= 1u << st;
    if (busy) {
      const unsigned char* sb = smem + (size_t)st * kBStage;
      const float* ta = (const float*)sb;
      const float4* pf4 = (const float4*)(sb + kBTile) + warp;  // (y, x_ip) of pivots 2w, 2w+1
      float r0acc = 0.f, r1acc = 0.f;
#pragma unroll 2
      for (int r0 = 0; r0 < kBRows; r0 += 4) {
        float av[4];
        float4 yw[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          av[u] = ta[(r0 + u) * 32 + lane];
          yw[u] = pf4[(r0 + u) * 4];
        }
        unsigned a0[4], a1[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const float q0 = av[u] * yw[u].x, q1 = av[u] * yw[u].z;
          a0[u] = hb[0] + __float_as_uint(fmaf(__saturatef(fmaf(q0, A[0], B[0])), 63.f, 8388608.f)) *
                              (unsigned)(kBThreads * 4);
          a1[u] = hb[1] + __float_as_uint(fmaf(__saturatef(fmaf(q1, A[1], B[1])), 63.f, 8388608.f)) *
                              (unsigned)(kBThreads * 4);
          r0acc += fabsf(fmaf(-cf[0], yw[u].y, av[u]));  // |a - c b| (dropped rows: |a|)
          r1acc += fabsf(fmaf(-cf[1], yw[u].w, av[u]));
        }
        // two independent read-modify-write chains, each in row order
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float h0, h1;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(h0) : "r"(a0[u]));
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(h1) : "r"(a1[u]));
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(a0[u]), "f"(h0 + fabsf(yw[u].y)));
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(a1[u]), "f"(h1 + fabsf(yw[u].w)));
        }
      }
      ec0 += (double)r0acc;
      ec1 += (double)r1acc;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  if (j >= m) return;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    if (!ok[t]) continue;
    const int64_t o = kk[t] * m + j;
    if (degen[t] || j == p[t]) {
      const double z = degen[t] ? P.colsum[j] : 0.0;  // fit.py:66-72: v = 0, error = sum |x|
      P.LB[o] = z;
      P.UB[o] = z;
      continue;
    }
    double lb, ub;
    column_bounds(hist + t * kNB * kBThreads + tid, kBThreads, (double)lo[t], (double)hi[t], (double)cf[t],
                  t == 0 ? ec0 : ec1, Tq[t] * unit[t], P.lam, P.colsum[j], n, &lb, &ub);
    P.LB[o] = lb;
    P.UB[o] = ub;
  }
}
