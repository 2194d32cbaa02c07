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
//   weight exceeds G (its exact bits; a zero takes the sign of its own row).
//
// k_select (one thread = one problem, warp = one pivot x 32 targets, CTA = 8
// pivots sharing every TMA-staged tile of X) runs a fixed pass schedule:
//   sample   32 strided rows, float ratios sorted in registers -> bracket
//   pass A   FP32: r ~ a32*y32, 32-bin value-space histogram over the bracket
//   pass A2  FP32: 32 sub-bins inside A's crossing bin -> window (~1 element)
//   pass B   exact weights: float classification with a guard band, exact
//            fl(a/b) only near the window; exact weight below the window,
//            exact Wneg (signs are exact) -> G; window rows collected and
//            resolved from exact keys
//   pass E   residual sum_i |x_ij - v_j x_ip| in row order
// A problem whose window misses the crossing or holds more than kCapB rows
// (heavy ties) is queued, with the exact key interval known to hold its
// crossing, for k_straggle (warp per problem, exact throughout).  The float
// passes only steer the search: every decision that reaches an output is
// made with exact integer weights (integer-valued doubles < 2^53, exact in
// any summation order) and exact f64 keys.

constexpr int kNBA = 32;           // pass-A / A2 bins
constexpr int kCapB = 8;           // rows collected per problem in pass B
constexpr int kDelta = 6;          // +- sample ranks around the estimated crossing
constexpr int kStages = 3;         // TMA pipeline depth
constexpr float kGuard = 0x1p-19f; // relative guard band of the float ratios

struct SelParams {
  const double* Xt;      // X in 32-column tiles: ((j/32)*np + i)*32 + j%32
  const float* Xft;      // float copy of Xt
  const double* gpb;     // shard pivot planes in 8-pivot groups: (g*np + i)*8 + w
  const double* gpy;
  const double* gpw;
  const float2* gpf;
  const double* Xc;      // column-major m x n
  const double* pb;      // [m][n] x_ip
  const double* py;      // [m][n] hoisted reciprocal (NaN: dropped row)
  const double* pw;      // [m][n] fixed-point weight (exact integer)
  const float2* pf;      // [m][n] (float y, float |x_ip|)
  const double* tq;
  const int* spow;
  const long long* nnz;
  const double* colsum;
  int64_t n, m, mp, np;   // np: plane row length (multiple of 32)
  int64_t p_begin, p_stride, npiv;
  double lam;
  double* V;             // [npiv][m]
  double* E;             // [npiv][m]
  Straggler* strag;
  unsigned long long* nstrag;
  int* status;
};

// Exact region test: returns false for a dead column, else sets G.  All
// operands are integers below 2^53 held in doubles, so every step is exact
// (thresholds are clamped to 2^54: beyond every reachable D).
__device__ __forceinline__ bool region_G(double Tq, double wneg, double Lsc, double* G) {
  const double cap = 0x1p54;
  const double Lf = fmin(floor(Lsc), cap), Lc = fmin(ceil(Lsc), cap);
  const double D = Tq - 2.0 * wneg;
  double thr;
  if (D < -Lf) thr = -Lf;
  else if (D >= Lc) thr = Lc;
  else return false;
  *G = floor(0.5 * (Tq - thr));  // Tq - thr >= 0
  return true;
}

// smem planes of one staged chunk (kRows rows); a pass stages only the
// planes it reads, so its stage is small and the 60 KB ring holds many.
constexpr int kTileF = kRows * 32 * 4;           // a32
constexpr int kTileA = kRows * 32 * 8;           // a (f64)
constexpr int kPlane8 = kWarps * kRows * 8;      // pf / pb / py / pw: [row][8 pivots]
constexpr int kRing = 60 * 1024;
constexpr int kMaxStages = 10;
constexpr int kHist = kNBA + 2;   // per-thread histogram slots (A2: below / 32 / above)

template <typename RowT>
constexpr size_t select_smem() {
  return (size_t)kRing + sizeof(float) * kHist * kBS + sizeof(RowT) * kCapB * kBS;
}

enum : unsigned { W_F = 1, W_A = 2, W_PF = 4, W_PB = 8, W_PY = 16, W_PW = 32 };

// Byte offsets of the planes inside one stage for a given plane set.
struct StageLayout {
  int f, a, pf, pb, py, pw, bytes, nst;
  __device__ explicit StageLayout(unsigned want) {
    int o = 0;
    f = o; o += (want & W_F) ? kTileF : 0;
    a = o; o += (want & W_A) ? kTileA : 0;
    pf = o; o += (want & W_PF) ? kPlane8 : 0;
    pb = o; o += (want & W_PB) ? kPlane8 : 0;
    py = o; o += (want & W_PY) ? kPlane8 : 0;
    pw = o; o += (want & W_PW) ? kPlane8 : 0;
    bytes = o;
    nst = min(kMaxStages, kRing / o);
  }
};

template <typename RowT>
__global__ void __launch_bounds__(kBS, 2) k_select(SelParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  float* hist = (float*)(smem + kRing);                                   // [kHist][kBS]
  RowT* cbuf = (RowT*)(hist + kHist * kBS);                              // [kCapB][kBS]
  __shared__ __align__(8) unsigned long long full[kMaxStages], empty[kMaxStages];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n = P.n, m = P.m, np = P.np;
  const int64_t kk = (int64_t)blockIdx.y * kWarps + warp;
  const bool piv_ok = kk < P.npiv;
  const int64_t p = piv_ok ? P.p_begin + kk * P.p_stride : 0;
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  const int64_t j = j0 + lane;
  const bool degenerate = piv_ok && P.nnz[p] == 0;
  const bool active = piv_ok && !degenerate && j < m && j != p;
  const int64_t jc = j < m ? j : m - 1;

  double Tq = 0.0;
  double Lsc = 0.0;
  if (piv_ok && !degenerate) {
    Tq = P.tq[p];
    Lsc = ldexp(P.lam, P.spow[p]);
  }
  const float lam32 = (float)P.lam;

  // ---- TMA pipeline ----------------------------------------------------------
  // Producer: the lanes of warp 0 issue the bulk copies of chunk c into stage
  // c % nst once every warp has released it (empty barrier); consumers wait
  // on that stage's full barrier only.  Parities are tracked per barrier, so
  // passes may use different stage layouts; a pass starts after a CTA
  // barrier, when every earlier stage has been released.
  if (tid == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  unsigned fphase = 0, ephase = 0, used = 0;  // per-barrier bits
  int nvalid = 0;
  for (int w = 0; w < kWarps; ++w) nvalid += ((int64_t)blockIdx.y * kWarps + w) < P.npiv;
  const int64_t nch = (n + kRows - 1) / kRows;
  const int64_t tbase = (int64_t)blockIdx.x * np * 32;  // this CTA's target tile
  const int64_t gbase = (int64_t)blockIdx.y * np * 8;   // this CTA's pivot group
  auto issue = [&](const StageLayout& L, int64_t c, unsigned want) {
    if (warp != 0) return;
    const int st = (int)(c % L.nst);
    if ((used >> st) & 1u) {
      mbar_wait(&empty[st], (ephase >> st) & 1u);
      ephase ^= 1u << st;
    }
    used |= 1u << st;
    if (lane == 0) {
      const int64_t i0 = c * kRows;
      unsigned char* base = smem + (size_t)st * L.bytes;
      fence_proxy_async();
      mbar_expect_tx(&full[st], (unsigned)L.bytes);
      if (want & W_F) bulk_g2s(base + L.f, P.Xft + tbase + i0 * 32, kTileF, &full[st]);
      if (want & W_A) bulk_g2s(base + L.a, P.Xt + tbase + i0 * 32, kTileA, &full[st]);
      if (want & W_PF) bulk_g2s(base + L.pf, P.gpf + gbase + i0 * 8, kPlane8, &full[st]);
      if (want & W_PB) bulk_g2s(base + L.pb, P.gpb + gbase + i0 * 8, kPlane8, &full[st]);
      if (want & W_PY) bulk_g2s(base + L.py, P.gpy + gbase + i0 * 8, kPlane8, &full[st]);
      if (want & W_PW) bulk_g2s(base + L.pw, P.gpw + gbase + i0 * 8, kPlane8, &full[st]);
    }
    __syncwarp();
  };
  // body(stage base, layout, rows, first_row) on every chunk
  auto sweep = [&](unsigned want, bool busy, auto&& body) {
    const StageLayout L(want);
    __syncthreads();  // every stage of the previous pass has been consumed
    for (int64_t c = 0; c < min((int64_t)(L.nst - 1), nch); ++c) issue(L, c, want);
    for (int64_t c = 0; c < nch; ++c) {
      if (c + L.nst - 1 < nch) issue(L, c + L.nst - 1, want);
      const int st = (int)(c % L.nst);
      mbar_wait(&full[st], (fphase >> st) & 1u);
      fphase ^= 1u << st;
      if (busy) body((const unsigned char*)smem + (size_t)st * L.bytes, L, (int)min((int64_t)kRows, n - c * kRows),
                     c * kRows);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  };
  auto tF = [&](const unsigned char* b, const StageLayout& L) { return (const float*)(b + L.f); };
  auto tA = [&](const unsigned char* b, const StageLayout& L) { return (const double*)(b + L.a); };
  // plane entries of row r for this warp's pivot: [r * 8 + warp]
  auto pF = [&](const unsigned char* b, const StageLayout& L) { return (const float2*)(b + L.pf) + warp; };
  auto pB = [&](const unsigned char* b, const StageLayout& L) { return (const double*)(b + L.pb) + warp; };
  auto pY = [&](const unsigned char* b, const StageLayout& L) { return (const double*)(b + L.py) + warp; };
  auto pW = [&](const unsigned char* b, const StageLayout& L) { return (const double*)(b + L.pw) + warp; };

  // ---- sample: float ratios of 32 strided rows, sorted -> value bracket ----
  float lo = 0.f, hi = 0.f;
  if (active) {
    float sr[kSample], sw[kSample];
#pragma unroll
    for (int s = 0; s < kSample; ++s) {
      int64_t r = ((2 * s + 1) * n) / (2 * kSample);
      float2 f = P.pf[p * P.np + r];
      sr[s] = P.Xft[tbase + r * 32 + lane] * f.x;
      sw[s] = f.y;
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
            bool x = up ? (sr[i] > sr[l]) : (sr[i] < sr[l]);
            float ta = sr[i], tb = sr[l], wa = sw[i], wb = sw[l];
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
    float rho = Tq > 0.0 ? (float)(Lsc / Tq) : 0.f;
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
  }
  if (!(hi > lo)) {  // degenerate sample (or idle lane): a tiny bracket around it
    float e = fmaxf(fabsf(lo), 1e-30f) * 1e-3f;
    lo -= e;
    hi += e;
  }
  const bool warp_active = __any_sync(0xffffffffu, active);

  // ---- pass A: 32-bin FP32 histogram over [lo, hi) (edge bins = tails) ------
  // bin(r) = RN(clamp(r * s + o)) is monotone in r: interior bin b <-> r in
  // [lo + (b-1) w, lo + b w), w = (hi - lo) / 30.
  const float sA = (float)(kNBA - 2) / (hi - lo);
  const float oA = 0.5f - lo * sA;
#pragma unroll
  for (int b = 0; b < kNBA; ++b) hist[b * kBS + tid] = 0.f;
  float wn32 = 0.f;
  sweep(W_F | W_PF, warp_active, [&](const unsigned char* sb, const StageLayout& L, int rmax, int64_t) {
    const float* ta = tF(sb, L);
    const float2* pf = pF(sb, L);
#pragma unroll 4
    for (int r = 0; r < rmax; ++r) {
      const float2 yw = pf[r * 8];
      const float q = ta[r * 32 + lane] * yw.x;
      const float t = fminf(fmaxf(fmaf(q, sA, oA), 0.f), (float)(kNBA - 1));
      const int b = __float_as_int(t + 8388608.f) - 0x4B000000;
      hist[b * kBS + tid] += yw.y;
      if (q < 0.f) wn32 += yw.y;
    }
  });
  float T32 = 0.f;
#pragma unroll
  for (int b = 0; b < kNBA; ++b) T32 += hist[b * kBS + tid];
  const float D32 = T32 - 2.f * wn32;
  const float G32 = 0.5f * (T32 - (D32 < -lam32 ? -lam32 : (D32 >= lam32 ? lam32 : 0.f)));
  // A2 range: the crossing bin of A (edge bins: a widened band beyond the bracket)
  float lo2, hi2;
  {
    float cum = 0.f;
    int bw = kNBA - 1;
    bool got = false;
#pragma unroll
    for (int b = 0; b < kNBA; ++b) {
      float h = hist[b * kBS + tid];
      if (!got && cum + h > G32) { bw = b; got = true; }
      if (!got) cum += h;
    }
    const float w = (hi - lo) / (float)(kNBA - 2);
    if (bw == 0) { lo2 = lo - 8.f * (hi - lo); hi2 = lo + 0.5f * w; }
    else if (bw == kNBA - 1) { lo2 = hi - 0.5f * w; hi2 = hi + 8.f * (hi - lo); }
    else { lo2 = lo + ((float)bw - 1.5f) * w; hi2 = lo + ((float)bw + 0.5f) * w; }
  }

  // ---- pass A2: 32 sub-bins over [lo2, hi2); slot 0 = below, 33 = above ----
  const float sA2 = (float)kNBA / (hi2 - lo2);
  const float oA2 = 0.5f - lo2 * sA2;
#pragma unroll
  for (int b = 0; b < kHist; ++b) hist[b * kBS + tid] = 0.f;
  sweep(W_F | W_PF, warp_active, [&](const unsigned char* sb, const StageLayout& L, int rmax, int64_t) {
    const float* ta = tF(sb, L);
    const float2* pf = pF(sb, L);
#pragma unroll 4
    for (int r = 0; r < rmax; ++r) {
      const float2 yw = pf[r * 8];
      const float q = ta[r * 32 + lane] * yw.x;
      const float t = fminf(fmaxf(fmaf(q, sA2, oA2), 0.f), (float)(kHist - 1));
      hist[(__float_as_int(t + 8388608.f) - 0x4B000000) * kBS + tid] += yw.y;
    }
  });
  // window = the crossing sub-bin, widened by the float error band
  double Lw = -INFINITY, Hw = INFINITY;
  {
    float cum = hist[tid];  // slot 0: below lo2
    int bw = -1;
#pragma unroll
    for (int b = 0; b < kNBA; ++b) {
      float h = hist[(b + 1) * kBS + tid];
      if (bw < 0 && cum + h > G32) bw = b;
      if (bw < 0) cum += h;
    }
    const double w2 = ((double)hi2 - (double)lo2) / (double)kNBA;
    if (bw >= 0) {
      double a = (double)lo2 + (double)bw * w2, b = a + w2;
      Lw = a - (fabs(a) * 0x1p-18 + w2 * 0.02);
      Hw = b + (fabs(b) * 0x1p-18 + w2 * 0.02);
    } else if (cum <= G32) {  // beyond hi2: leave the window open upward
      Lw = (double)hi2 - fabs((double)hi2) * 0x1p-18;
    } else {                  // below lo2
      Hw = (double)lo2 + fabs((double)lo2) * 0x1p-18;
    }
  }

  // ---- pass B: exact weights; exact ratios only near the window ------------
  // Float ratios carry < 2^-21 relative error, so any element whose float
  // ratio is outside [Lw, Hw) by more than the guard band is classified
  // exactly without dividing.  Signs are exact (FLOATSAFE inputs).
  const float Lg = (float)(Lw - fabs(Lw) * (double)kGuard);
  const float Hg = (float)(Hw + fabs(Hw) * (double)kGuard);
  double wb = 0.0, win = 0.0, wneg = 0.0;
  int cnt = 0;
  sweep(W_F | W_PF | W_PW | W_A | W_PB | W_PY, warp_active,
        [&](const unsigned char* sb, const StageLayout& L, int rmax, int64_t i0) {
    const float* ta = tF(sb, L);
    const float2* pf = pF(sb, L);
    const double* pw = pW(sb, L);
#pragma unroll 4
    for (int r = 0; r < rmax; ++r) {
      const float q32 = ta[r * 32 + lane] * pf[r * 8].x;
      const double wq = pw[r * 8];
      if (q32 < 0.f) wneg += wq;
      if (q32 < Lg) wb += wq;
      if (q32 >= Lg && q32 < Hg) {  // near or inside: decide exactly
        const double q = ratio_fast(tA(sb, L)[r * 32 + lane], pB(sb, L)[r * 8], pY(sb, L)[r * 8]);
        if (q < Lw) {
          wb += wq;
        } else if (q < Hw) {
          win += wq;
          if (cnt < kCapB) cbuf[cnt * kBS + tid] = (RowT)(i0 + r);
          ++cnt;
        }
      }
    }
  });

  double v = 0.0;
  bool done = !active;
  if (active) {
    double G = 0.0;
    if (!region_G(Tq, wneg, Lsc, &G)) {
      done = true;  // dead column (fit.py:60-63 returns +0.0)
    } else if (wb <= G && G < wb + win && cnt <= kCapB) {
      // resolve: exact keys of the window rows into this thread's (now free)
      // histogram slots, stable insertion by key, then the prefix walk
      unsigned long long* key = (unsigned long long*)hist;       // [kCapB][kBS]
      double* wgt = (double*)hist + kCapB * kBS;                 // [kCapB][kBS]
      const double* xcol = P.Xc + jc * n;
      for (int c = 0; c < cnt; ++c) {
        const int row = (int)cbuf[c * kBS + tid];
        const unsigned long long k = key64(ratio_fast(xcol[row], P.pb[p * P.np + row], P.py[p * P.np + row]));
        const double w = P.pw[p * P.np + row];
        int d = c;
        while (d > 0 && key[(d - 1) * kBS + tid] > k) {
          key[d * kBS + tid] = key[(d - 1) * kBS + tid];
          wgt[d * kBS + tid] = wgt[(d - 1) * kBS + tid];
          cbuf[d * kBS + tid] = cbuf[(d - 1) * kBS + tid];
          --d;
        }
        key[d * kBS + tid] = k;
        wgt[d * kBS + tid] = w;
        cbuf[d * kBS + tid] = (RowT)row;
      }
      double cum = wb;
      for (int c = 0; c < cnt && !done; ++c) {
        cum += wgt[c * kBS + tid];
        if (cum > G) {
          const unsigned long long k = key[c * kBS + tid];
          const int row = (int)cbuf[c * kBS + tid];
          v = k == kZeroKey ? __ddiv_rn(xcol[row], P.pb[p * P.np + row]) : key64_inv(k);
          done = true;
        }
      }
    }
    if (!done) {
      Straggler s;
      s.kk = (int)kk;
      s.j = (int)j;
      s.G = G;
      const unsigned long long KL = Lw == -INFINITY ? 0ULL : key64(Lw);
      const unsigned long long KH = Hw == INFINITY ? ~0ULL : key64(Hw);
      if (G < wb) { s.lo = 0; s.hi = KL - 1; s.wb = 0; }
      else if (G >= wb + win) { s.lo = KH; s.hi = ~0ULL; s.wb = wb + win; }
      else { s.lo = KL; s.hi = KH - 1; s.wb = wb; }
      unsigned long long slot = atomicAdd(P.nstrag, 1ULL);
      P.strag[slot] = s;
    }
  }

  // ---- pass E: residual in row order ---------------------------------------
  double e = 0.0;
  const bool warp_err = __any_sync(0xffffffffu, active && done);
  sweep(W_A | W_PB, warp_err, [&](const unsigned char* sb, const StageLayout& L, int rmax, int64_t) {
    const double* ta = tA(sb, L);
    const double* pb = pB(sb, L);
#pragma unroll 4
    for (int r = 0; r < rmax; ++r) e += fabs(__dsub_rn(ta[r * 32 + lane], __dmul_rn(pb[r * 8], v)));
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
  s.G = -1.0;  // unknown: k_straggle computes Wneg and G first
  s.lo = 0;
  s.hi = ~0ULL;
  s.wb = 0.0;
  unsigned long long slot = atomicAdd(P.nstrag, 1ULL);
  P.strag[slot] = s;
}

// ----------------------------------------------------------- stragglers --
//
// One warp per queued problem, exact throughout, reading X column-major so
// the 32 lanes load 32 consecutive rows.  The record carries a key interval
// [lo, hi] known to contain the crossing and the exact weight below it.
// Each round either collects every element of the interval (<= kSCap) into
// shared memory, bitonic-sorts them by (key, row) and scans the prefix, or
// histograms the interval into 256 key buckets (shared int64 atomics) and
// narrows to the crossing bucket.  Ratios use the hoisted division when
// SAFE, IEEE __ddiv_rn otherwise.

constexpr int kSWarps = 4;
constexpr int kSCap = 1024;
constexpr int kSBins = 256;

struct SEnt {
  unsigned long long k;
  double w;
  int row;
  int pad;
};

constexpr size_t kStraggleSmem = (size_t)kSWarps * (kSCap * sizeof(SEnt) + kSBins * sizeof(double));

template <bool SAFE>
__device__ __forceinline__ double sratio(const SelParams& P, int64_t p, int64_t i, int64_t j) {
  const double a = P.Xc[j * P.n + i], b = P.pb[p * P.np + i];
  if (SAFE) return ratio_fast(a, b, P.py[p * P.np + i]);
  return b != 0.0 ? __ddiv_rn(a, b) : __longlong_as_double(0x7ff8000000000000LL);
}

__device__ __forceinline__ double warp_sum(double x) {
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <bool SAFE>
__global__ void __launch_bounds__(kSWarps * 32) k_straggle(SelParams P) {
  extern __shared__ __align__(16) unsigned char ssm[];
  SEnt(*ent)[kSCap] = reinterpret_cast<SEnt(*)[kSCap]>(ssm);
  double(*bins)[kSBins] = reinterpret_cast<double(*)[kSBins]>(ssm + (size_t)kSWarps * kSCap * sizeof(SEnt));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned long long total = *P.nstrag;
  const int64_t n = P.n, m = P.m;
  for (unsigned long long t = (unsigned long long)blockIdx.x * kSWarps + warp; t < total;
       t += (unsigned long long)gridDim.x * kSWarps) {
    Straggler s = P.strag[t];
    const int64_t kk = s.kk, j = s.j, p = P.p_begin + kk * P.p_stride;
    const double* pwp = P.pw + p * P.np;
    const double Tq = P.tq[p];
    const double Lsc = ldexp(P.lam, P.spow[p]);
    double G = s.G, wb = s.wb;
    unsigned long long lo = s.lo, hi = s.hi;
    bool dead = false;
    if (G < 0.0) {  // exact Wneg and key range first
      double wneg = 0.0;
      unsigned long long kmin = ~0ULL, kmax = 0;
      for (int64_t i = lane; i < n; i += 32) {
        const double w = pwp[i];
        if (w == 0.0) continue;
        const double q = sratio<SAFE>(P, p, i, j);
        const unsigned long long k = key64(q);
        if (q < 0.0) wneg += w;
        kmin = min(kmin, k);
        kmax = max(kmax, k);
      }
      wneg = warp_sum(wneg);
      for (int o = 16; o; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
      }
      dead = !region_G(Tq, wneg, Lsc, &G);
      lo = kmin;
      hi = kmax;
      wb = 0.0;
    }
    double v = 0.0;
    bool ok = dead;
    for (int round = 0; round < 40 && !ok; ++round) {
      int base = 0;
      for (int64_t i0 = 0; i0 < n; i0 += 32) {
        const int64_t i = i0 + lane;
        bool in = false;
        unsigned long long k = 0;
        double w = 0.0;
        if (i < n) {
          w = pwp[i];
          if (w != 0.0) {
            k = key64(sratio<SAFE>(P, p, i, j));
            in = k >= lo && k <= hi;
          }
        }
        const unsigned mask = __ballot_sync(0xffffffffu, in);
        const int pos = base + __popc(mask & ((1u << lane) - 1));
        if (in && pos < kSCap) ent[warp][pos] = SEnt{k, w, (int)i, 0};
        base += __popc(mask);
      }
      __syncwarp();
      if (base <= kSCap) {
        int np2 = 1;
        while (np2 < base) np2 <<= 1;
        for (int e = base + lane; e < np2; e += 32) ent[warp][e] = SEnt{~0ULL, 0.0, 0x7fffffff, 0};
        __syncwarp();
        for (int kq = 2; kq <= np2; kq <<= 1) {
          for (int jq = kq >> 1; jq > 0; jq >>= 1) {
            for (int e = lane; e < np2; e += 32) {
              const int l = e ^ jq;
              if (l > e) {
                const SEnt a = ent[warp][e], b = ent[warp][l];
                const bool gt = a.k > b.k || (a.k == b.k && a.row > b.row);
                if (gt == ((e & kq) == 0)) {
                  ent[warp][e] = b;
                  ent[warp][l] = a;
                }
              }
            }
            __syncwarp();
          }
        }
        double cum = wb;
        int hit = -1;
        for (int e0 = 0; e0 < base && hit < 0; e0 += 32) {
          const int e = e0 + lane;
          double x = e < base ? ent[warp][e].w : 0.0;
          for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          const unsigned cm = __ballot_sync(0xffffffffu, e < base && cum + x > G);
          if (cm) hit = e0 + __ffs(cm) - 1;
          cum += __shfl_sync(0xffffffffu, x, 31);
        }
        if (hit >= 0) {
          const SEnt h = ent[warp][hit];
          v = h.k == kZeroKey ? __ddiv_rn(P.Xc[j * n + h.row], P.pb[p * P.np + h.row]) : key64_inv(h.k);
          ok = true;
        }
        __syncwarp();
        if (!ok) break;  // cannot happen: the interval holds the crossing
      } else {
        int sh = (hi - lo == ~0ULL) ? 56 : ceil_log2_u64(hi - lo + 1) - 8;
        sh = sh > 0 ? sh : 0;
        for (int b = lane; b < kSBins; b += 32) bins[warp][b] = 0.0;
        __syncwarp();
        for (int64_t i = lane; i < n; i += 32) {
          const double w = pwp[i];
          if (w == 0.0) continue;
          const unsigned long long k = key64(sratio<SAFE>(P, p, i, j));
          // integer-valued doubles: exact, order-independent atomic sums
          if (k >= lo && k <= hi) atomicAdd(&bins[warp][(k - lo) >> sh], w);
        }
        __syncwarp();
        double cum = wb;
        int bsel = kSBins - 1;
        for (int b = 0; b < kSBins; ++b) {
          const double hb = bins[warp][b];
          if (cum + hb > G) { bsel = b; break; }
          cum += hb;
        }
        const unsigned long long nlo = lo + ((unsigned long long)bsel << sh);
        unsigned long long nhi = nlo + ((1ULL << sh) - 1);
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
    double e = 0.0;
    const double* pbp = P.pb + p * P.np;
    for (int64_t i = lane; i < n; i += 32) e += fabs(__dsub_rn(P.Xc[j * n + i], __dmul_rn(pbp[i], v)));
    for (int o = 16; o; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    if (lane == 0) {
      P.V[kk * m + j] = v;
      P.E[kk * m + j] = e;
    }
    __syncwarp();
  }
}
