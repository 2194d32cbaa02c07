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
//   F passes (P.nfloat of them: 1 for n <= 4096, 2 or 3 beyond): FP32 ratio
//            r ~ a32*y32 into a 64-slot per-thread histogram (below / 62 bins
//            / above) of the current range; the crossing bin becomes the
//            next range, and after the last pass the window [Lw, Hw)
//   pass B   exact: float classification with a guard band, exact fl(a/b)
//            only near the window; exact weight below the window, exact
//            Wneg (signs are exact) -> G; window rows collected (<= CAP).
//            The column residual is fused in (see the pass for the identity)
//   resolve  exact keys of the window rows, stable insertion by key, prefix
//            walk to the crossing, residual of the window rows.
// A problem whose window misses the crossing or holds more than CAP rows
// (heavy ties) is queued, with the exact key interval known to hold its
// crossing, for k_straggle (warp per problem, exact throughout).  The float
// passes only steer the search: every decision that reaches an output is
// made with exact integer weights (integer-valued doubles < 2^53, exact in
// any summation order) and exact f64 keys.

constexpr int kNB = 64;            // F-pass histogram slots: 0 below, 1..62, 63 above
constexpr int kNI = kNB - 2;       // interior bins
constexpr int kDelta = 7;          // +- sample ranks around the estimated crossing
constexpr float kGuard = 0x1p-19f; // relative guard band of the float ratios
constexpr double kBig = 1.7976931348623157e308;  // DBL_MAX: open window side

struct SelParams {
  const double* Xt;      // X in 32-column tiles: ((j/32)*np + i)*32 + j%32
  const float* Xft;      // float copy of Xt
  const float* Xq;       // k_bound's target-group tiles (k_tile's xq)
  const double2* gbw;    // shard (x_ip, wq_ip) records in 8-pivot groups: (g*np + i)*8 + w
  const float2* gpf;     // shard (float y_ip, float x_ip) in 8-pivot groups
  const unsigned* gwu;   // shard wq_ip / 2^21 (rounded) in 8-pivot groups
  const float4* gbp;     // k_bound plane (see k_group_bound)
  const double* Xc;      // column-major m x n
  const double* pb;      // [m][n] x_ip
  const double* py;      // [m][n] hoisted reciprocal (NaN: dropped row)
  const double* pw;      // [m][n] fixed-point weight (exact integer)
  const float2* pf;      // [m][n] (float y, float x_ip)
  const double* tq;
  const int* spow;
  const long long* nnz;
  const double* colsum;
  int64_t n, m, mp, np;   // np: plane row length (multiple of 32)
  int64_t p_begin, p_stride, npiv;
  const int64_t* pivots; // device pivot list (null: p_begin + k * p_stride)
  double lam;
  int nfloat;            // number of F passes (1..3)
  double* V;             // [npiv][m]
  double* E;             // [npiv][m]
  Straggler* strag;
  unsigned long long* nstrag;
  int* status;
  unsigned long long* tprobe;  // optional [grid][8] phase timestamps (profiling builds; null = off)
  // window records, k_select -> k_resolve (problem index kk * m + j)
  double* rG;
  double* rwb;
  double* res;
  double* rLw;
  double* rHw;
  int* rcnt;
  unsigned char* rrows;  // RowT [CAP][npiv*m]
  double* LB;            // bound mode: [npiv][m] lower / upper bound of each column's optimum
  double* UB;
  double2* BRK;          // bound mode: [npiv][m] range holding each column's optimum v
  const int64_t* seeds;  // seeded fit / continued bound: position in the previous bound call's list
  const float2* NEXTr;   // bound mode: ranges the previous pass left ([npiv][m])
  const float2* win;     // k_select: per-problem windows from k_bound passes (no sample / F passes)
  float2* NEXTw;         // bound mode: ranges this pass leaves
  int delta;             // bound mode: sample bracket half-width (ranks)
  unsigned* GH;          // split bound: merged histograms [npiv*m][64]
  double* GE;            // split bound: residual shares [z][npiv*m]
  float* GB;             // split bound: ranges [npiv*m][5]
  const double* lamk;    // per pivot-list entry penalty (entry lists), or null: lam for all
  const double* lams;    // multi-penalty bound: ascending penalties (device)
  int nlam;
  float2* NEXTm;         // multi-penalty bound: next ranges [nlam][npiv][m] (optional)
  double* LBm;           // multi-penalty bound: per (penalty, pivot) sums [nlam][npiv]
  double* UBm;
  unsigned long long* LBq;  // k_bound: per (penalty, pivot) column-bound sums, fixed point 2^-fxk ([nlam][npiv])
  unsigned long long* UBq;
  const int* fxk;        // fixed-point exponent (k_fxscale)
  int lean;              // k_bound: per-pivot sums and next ranges only (no LB / UB / BRK records)
  int steer;             // k_bound: a steering pass over every steer-th row chunk (next ranges only)
  int band;              // k_bound: target groups per raster band (>= gridDim.x: plain order)
};

__device__ __forceinline__ int64_t pivot_of(const SelParams& P, int64_t kk) {
  return P.pivots ? P.pivots[kk] : P.p_begin + kk * P.p_stride;
}

// Penalty of pivot-list entry kk (entry lists carry one per entry).
__device__ __forceinline__ double lam_of(const SelParams& P, int64_t kk) { return P.lamk ? P.lamk[kk] : P.lam; }

// acc += x if p, exactly (x, acc integer-valued): one select of the high
// word of 1.0 and one DFMA, instead of the add-and-select-both-halves the
// compiler's if-conversion emits.
__device__ __forceinline__ void padd(double& acc, double x, bool p) {
  acc = __fma_rn(x, __hiloint2double(p ? 0x3ff00000 : 0, 0), acc);
}

__device__ __forceinline__ double warp_sum(double x) {
  for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

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

// Shared memory: [cbuf | ring | histograms].  The F passes stream through
// cbuf + ring (cbuf is only filled by pass B), pass B through ring +
// histograms (those are dead by then), so each pass gets the deepest ring
// the 2-CTA/SM budget allows.  A pass stages only the planes it reads, in
// chunks of R rows (64 for the plain F pass, 32 otherwise).
constexpr int kRingMid = 16 * 1024;              // the ring both halves share
constexpr int kHistBytes = kNB * kBS * 4;        // per-thread histograms [slot][thread]
constexpr int kMaxStages = 8;

template <typename RowT, int CAP>
__host__ __device__ constexpr int cbuf_bytes() { return (int)(sizeof(RowT) * CAP * kBS); }
template <typename RowT, int CAP>
constexpr size_t select_smem() {
  return (size_t)cbuf_bytes<RowT, CAP>() + kRingMid + kHistBytes;
}

enum : unsigned { W_F = 1, W_A = 2, W_PF = 4, W_BW = 8 };

// Byte offsets of the planes inside one stage for a given plane set and
// chunk height R; the ring is [base, base + ring).
struct StageLayout {
  int f, a, pf, bw, bytes, nst, R, base;
  __device__ StageLayout(unsigned want, int rows, int ring_base, int ring) {
    R = rows;
    base = ring_base;
    int o = 0;
    f = o; o += (want & W_F) ? R * 32 * 4 : 0;        // a32 tile [row][32 targets]
    a = o; o += (want & W_A) ? R * 32 * 8 : 0;        // a (f64) tile
    pf = o; o += (want & W_PF) ? R * kWarps * 8 : 0;  // (y32, w32) [row][8 pivots]
    bw = o; o += (want & W_BW) ? R * kWarps * 16 : 0; // (x_ip, wq) [row][8 pivots]
    bytes = o;
    nst = min(kMaxStages, ring / o);
  }
};

template <typename RowT, int CAP>
__global__ void __launch_bounds__(kBS, 2) k_select(SelParams P) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int kCb = cbuf_bytes<RowT, CAP>();
  RowT* cbuf = (RowT*)smem;                                               // [CAP][kBS]
  float* hist = (float*)(smem + kCb + kRingMid);                          // [kNB][kBS]
  __shared__ __align__(8) unsigned long long full[kMaxStages], empty[kMaxStages];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t n = P.n, m = P.m, np = P.np;
  const int64_t kk = (int64_t)blockIdx.y * kWarps + warp;
  const bool piv_ok = kk < P.npiv;
  const int64_t p = piv_ok ? pivot_of(P, kk) : 0;
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  const int64_t j = j0 + lane;
  const bool degenerate = piv_ok && P.nnz[p] == 0;
  const bool active = piv_ok && !degenerate && j < m && j != p;

  double Tq = 0.0;
  double Lsc = 0.0;
  int sp = 0;
  if (piv_ok && !degenerate) {
    Tq = P.tq[p];
    sp = P.spow[p];
    Lsc = ldexp(P.lam, sp);
  }
  const double unit = ldexp(1.0, -sp);
  // windows handed in by k_bound passes (fit_impl's seeded windows): no sample
  // bracket and no F passes, pass B starts on them (a missed crossing or an
  // overflowing window goes to the straggler solver, as always)
  const bool winm = P.win != nullptr;
  const bool exact_f = !winm && P.nfloat >= 2;  // multi-pass: exact bases and exact Wneg in the F passes

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
      const int64_t i0 = c * L.R;
      unsigned char* base = smem + L.base + (size_t)st * L.bytes;
      fence_proxy_async();
      mbar_expect_tx(&full[st], (unsigned)L.bytes);
      if (want & W_F) bulk_g2s(base + L.f, P.Xft + tbase + i0 * 32, L.R * 32 * 4, &full[st]);
      if (want & W_A) bulk_g2s(base + L.a, P.Xt + tbase + i0 * 32, L.R * 32 * 8, &full[st]);
      if (want & W_PF) bulk_g2s(base + L.pf, P.gpf + gbase + i0 * 8, L.R * kWarps * 8, &full[st]);
      if (want & W_BW) bulk_g2s(base + L.bw, P.gbw + gbase + i0 * 8, L.R * kWarps * 16, &full[st]);
    }
    __syncwarp();
  };
  // body(stage base, layout, rows, first_row) on every chunk of R rows
  auto sweep = [&](unsigned want, int rows, int ring_base, int ring, bool busy, auto&& body) {
    const StageLayout L(want, rows, ring_base, ring);
    const int64_t nch = (n + rows - 1) / rows;
    fence_proxy_async();  // generic writes to the ring space (histograms) before async copies
    __syncthreads();      // every stage of the previous pass has been consumed
    for (int64_t c = 0; c < min((int64_t)(L.nst - 1), nch); ++c) issue(L, c, want);
    for (int64_t c = 0; c < nch; ++c) {
      if (c + L.nst - 1 < nch) issue(L, c + L.nst - 1, want);
      const int st = (int)(c % L.nst);
      mbar_wait(&full[st], (fphase >> st) & 1u);
      fphase ^= 1u << st;
      if (busy) body((const unsigned char*)smem + L.base + (size_t)st * L.bytes, L,
                     (int)min((int64_t)rows, n - c * rows), c * rows);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  };
  constexpr int kRingFB = 0, kRingFS = kCb + kRingMid;              // F passes: cbuf + ring
  constexpr int kRingBB = kCb, kRingBS = kRingMid + kHistBytes;     // pass B: ring + histograms
  auto tF = [&](const unsigned char* b, const StageLayout& L) { return (const float*)(b + L.f); };
  auto tA = [&](const unsigned char* b, const StageLayout& L) { return (const double*)(b + L.a); };
  // plane entries of row r for this warp's pivot: [r * 8 + warp]
  auto pF = [&](const unsigned char* b, const StageLayout& L) { return (const float2*)(b + L.pf) + warp; };
  auto pBW = [&](const unsigned char* b, const StageLayout& L) { return (const double2*)(b + L.bw) + warp; };

  unsigned long long* tp = P.tprobe ? P.tprobe + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * 8 : nullptr;
  auto stamp = [&](int k) {
    if (tp && tid == 0) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); tp[k] = t; }
  };
  stamp(0);
  // ---- sample: float ratios of 32 strided rows, sorted -> value bracket ----
  float lo = 0.f, hi = 0.f;
  if (active && !winm) {
    float sr[kSample], sw[kSample];
#pragma unroll
    for (int s = 0; s < kSample; ++s) {
      int64_t r = ((2 * s + 1) * n) / (2 * kSample);
      float2 f = P.pf[p * P.np + r];
      sr[s] = P.Xft[tbase + r * 32 + lane] * f.x;
      sw[s] = fabsf(f.y);
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

  __syncthreads();
  stamp(1);
  // ---- F passes: 64-slot FP32 histograms, each narrowing the range ---------
  // slot(r) = RN(63 * sat(r * A + B)): slot 0 <-> r < lo, slot b in 1..62 <->
  // r in [lo + (b-1) w, lo + b w) with w = (hi - lo) / 62, slot 63 <-> r >= hi
  // (up to float rounding at the edges, which the margins absorb).  The
  // slot address is one integer multiply-add of the magic-rounded bits.
  // Single pass (n <= 4096): float sums throughout -- a bin holds ~1/100 of
  // the weight, far above float rounding.  Several passes (large n): the bins
  // of later passes are tiny, so every pass also sums the exact weight of its
  // slot 0 (where the walk to the crossing starts) and pass 1 the exact Wneg
  // (exact G, and dead columns drop out of the later passes).
  double wneg = 0.0, G = 0.0;
  bool live = active;
  double Lw = -kBig, Hw = kBig;   // final window [Lw, Hw)
  float G32 = 0.f;
  if (winm && active) {
    const float2 r = P.win[kk * m + j];
    Lw = (double)r.x;
    Hw = (double)r.y;
  }
  for (int pass = 0; pass < (winm ? 0 : P.nfloat); ++pass) {
    const float A = (62.f / 63.f) / (hi - lo);
    const float B = 0.5f / 63.f - lo * A;
#pragma unroll
    for (int b = 0; b < kNB; ++b) hist[b * kBS + tid] = 0.f;
    const unsigned hbase = smem_u32(hist + tid) - 0x4B000000u * (unsigned)(kBS * 4);
    const bool busy = __any_sync(0xffffffffu, live);
    // One F pass over a staged chunk, all R rows (pad rows past n have
    // y = w = wq = 0 and add nothing).  Rows go in batches of 4: the tile and
    // plane loads and slot arithmetic of a batch are issued first, then the
    // four histogram read-modify-writes, whose program order (volatile asm)
    // keeps same-slot updates correct -- so only the RMWs, not the loads,
    // form the serial chain.  KIND 0: float single pass (+ float Wneg);
    // 1: exact first pass (+ exact Wneg and slot-0 weight); 2: exact later
    // pass (+ slot-0 weight); 3: float single pass for a lambda far below one
    // bin's weight, where G = T/2 up to << a bin and no Wneg is needed.
    float wn32 = 0.f;
    double wlow = 0.0;
    auto fbody = [&](const unsigned char* sb, const StageLayout& L, auto kind) {
      constexpr int K = decltype(kind)::value;
      const float* ta = tF(sb, L);
      const float2* pf = pF(sb, L);
      const double2* bw = pBW(sb, L);
#pragma unroll 2
      for (int r0 = 0; r0 < L.R; r0 += 4) {
        float2 yw[4];
        float av[4];
        double wq[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          yw[u] = pf[(r0 + u) * 8];
          av[u] = ta[(r0 + u) * 32 + lane];
          if (K == 1 || K == 2) wq[u] = bw[(r0 + u) * 8].y;
        }
        unsigned addr[4];
        float q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          q[u] = av[u] * yw[u].x;
          const float uu = __saturatef(fmaf(q[u], A, B));
          addr[u] = hbase + __float_as_uint(fmaf(uu, 63.f, 8388608.f)) * (unsigned)(kBS * 4);
        }
        // read-modify-writes in row order (volatile asm keeps same-slot
        // updates ordered); the loads and slot arithmetic above are not
        // part of the serial chain
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float h;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(h) : "r"(addr[u]));
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr[u]), "f"(h + fabsf(yw[u].y)));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (K == 0 && q[u] < 0.f) wn32 += fabsf(yw[u].y);  // K 3: lambda too small to move G (no Wneg needed)
          if (K == 1) padd(wneg, wq[u], q[u] < 0.f);                     // exact: signs of q32 are exact
          if (K == 1 || K == 2) padd(wlow, wq[u], addr[u] == hbase + 0x4B000000u * (unsigned)(kBS * 4));  // slot 0
        }
      }
    };
    double base;
    if (!exact_f) {  // single float pass (pass == 0)
      // warp-uniform (one pivot per warp): lambda below 1e-4 of the pivot's
      // total weight shifts G by far less than a bin holds
      const bool tiny_lam = P.lam <= 1e-4 * Tq * unit;
      sweep(W_F | W_PF, 64, kRingFB, kRingFS, busy, [&](const unsigned char* sb, const StageLayout& L, int, int64_t) {
        if (tiny_lam) fbody(sb, L, std::integral_constant<int, 3>{});
        else fbody(sb, L, std::integral_constant<int, 0>{});
      });
      float T32 = 0.f;
#pragma unroll
      for (int b = 0; b < kNB; ++b) T32 += hist[b * kBS + tid];
      const float lam32 = (float)P.lam;
      if (tiny_lam) {
        G32 = 0.5f * T32;  // pass B decides the region (and deadness) exactly
      } else {
        const float D32 = T32 - 2.f * wn32;
        G32 = 0.5f * (T32 - (D32 < -lam32 ? -lam32 : (D32 >= lam32 ? lam32 : 0.f)));
        // certainly dead (float error of D32 is far below the slack): skip pass B
        if (fabsf(D32) + 1e-7f * (float)n * T32 < lam32 * (1.f - 1e-6f)) live = false;
      }
      base = (double)hist[tid];
    } else if (pass == 0) {
      sweep(W_F | W_PF | W_BW, 32, kRingFB, kRingFS, busy, [&](const unsigned char* sb, const StageLayout& L, int, int64_t) {
        fbody(sb, L, std::integral_constant<int, 1>{});
      });
      if (live && !region_G(Tq, wneg, Lsc, &G)) live = false;  // dead column
      base = wlow * unit;
    } else {
      sweep(W_F | W_PF | W_BW, 32, kRingFB, kRingFS, busy, [&](const unsigned char* sb, const StageLayout& L, int, int64_t) {
        fbody(sb, L, std::integral_constant<int, 2>{});
      });
      base = wlow * unit;
    }
    // crossing slot: walk the interior bins from the weight below the range
    const double Gd = exact_f ? G * unit : (double)G32;
    double cum = base;
    int bw = 0;
    if (!(cum > Gd)) {
      bw = kNB - 1;
#pragma unroll 8
      for (int b = 1; b < kNB - 1; ++b) {
        const double h = (double)hist[b * kBS + tid];
        if (cum + h > Gd) { bw = b; break; }
        cum += h;
      }
    }
    const float w = (hi - lo) / (float)kNI;
    if (pass + 1 < P.nfloat) {
      float nlo, nhi;
      if (bw == 0) { nlo = lo - 8.f * (hi - lo); nhi = lo + 0.05f * w; }
      else if (bw == kNB - 1) { nlo = hi - 0.05f * w; nhi = hi + 8.f * (hi - lo); }
      else { nlo = lo + ((float)bw - 1.05f) * w; nhi = lo + ((float)bw + 0.05f) * w; }
      lo = nlo;
      hi = nhi;
      if (!(hi > lo)) {
        float e = fmaxf(fabsf(lo), 1e-30f) * 1e-3f;
        lo -= e;
        hi += e;
      }
    } else {
      const double wd = ((double)hi - (double)lo) / (double)kNI;
      if (bw == 0) {
        Hw = (double)lo + (fabs((double)lo) * 0x1p-18 + wd * 0.02);
      } else if (bw == kNB - 1) {
        Lw = (double)hi - (fabs((double)hi) * 0x1p-18 + wd * 0.02);
      } else {
        const double a = (double)lo + (double)(bw - 1) * wd, b = a + wd;
        Lw = a - (fabs(a) * 0x1p-18 + wd * 0.02);
        Hw = b + (fabs(b) * 0x1p-18 + wd * 0.02);
      }
    }
  }

  stamp(2);
  // ---- pass B: exact weights + fused residual; the window is collected -----
  // Float ratios carry < 2^-21 relative error, so an element whose float
  // ratio is below Lg (Lw less a guard band) is certainly below the window
  // and one at or above Hg certainly above it (signs are exact: FLOATSAFE
  // inputs).  Everything in [Lg, Hg) -- the window and its guard bands -- is
  // only collected (row index) and classified exactly in the resolve, so the
  // pass is branch-free.
  // Residual: with one finite reference point c0 in {Lw, Hw} and v in
  // [Lw, Hw), every element outside the window satisfies
  //   |x_ij - v x_ip| = |x_ij - c0 x_ip| +- (v - c0) |x_ip|   (+ below, - above)
  // exactly in real arithmetic, so the pass sums |x_ij - c0 x_ip| now and the
  // resolve adds (v - c0)(W_below - W_above); (v - c0) is window-sized, so
  // nothing cancels.  Dropped rows (x_ip = 0: y32 = 0, wq = 0, exact ratio
  // NaN) carry no weight and add |x_ij|.
  const float Lg = (float)(Lw - fabs(Lw) * (double)kGuard);
  const float Hg = (float)(Hw + fabs(Hw) * (double)kGuard);
  const double c0 = Lw > -kBig ? Lw : Hw;
  double wb = 0.0, es = 0.0;
  int cnt = 0;
  const unsigned cb0 = smem_u32(cbuf + tid);
  auto bbody = [&](const unsigned char* sb, const StageLayout& L, int rmax, int64_t i0, auto want_wneg) {
    const float* ta = tF(sb, L);
    const float2* pf = pF(sb, L);
    const double2* bwp = pBW(sb, L);
    const double* xa = tA(sb, L);
    // batches of 4 rows: loads first, then the (branch-free) bookkeeping;
    // pad rows past n (all zeros) add nothing and are never collected
#pragma unroll 2
    for (int r0 = 0; r0 < L.R; r0 += 4) {
      float q32[4];
      double2 bw[4];
      double a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        q32[u] = ta[(r0 + u) * 32 + lane] * pf[(r0 + u) * 8].x;
        bw[u] = bwp[(r0 + u) * 8];  // (x_ip, wq)
        a[u] = xa[(r0 + u) * 32 + lane];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (decltype(want_wneg)::value) padd(wneg, bw[u].y, q32[u] < 0.f);
        const bool below = q32[u] < Lg;
        const bool inw = (!below) & (q32[u] < Hg) & (r0 + u < rmax);  // bitwise: no branches
        padd(wb, bw[u].y, below);
        if (inw & (cnt < CAP)) {
          const unsigned addr = cb0 + (unsigned)(cnt * kBS * sizeof(RowT));
          const RowT row = (RowT)(i0 + r0 + u);
          if (sizeof(RowT) == 2) asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)row));
          else asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"((unsigned)row));
        }
        cnt += inw;
        es += fabs(__fma_rn(-bw[u].x, c0, a[u]));  // the resolve takes the window rows back out
      }
    }
  };
  const bool busyB = __any_sync(0xffffffffu, live);
  if (exact_f)
    sweep(W_F | W_A | W_PF | W_BW, 32, kRingBB, kRingBS, busyB,
          [&](const unsigned char* sb, const StageLayout& L, int rmax, int64_t i0) {
      bbody(sb, L, rmax, i0, std::false_type{});
    });
  else
    sweep(W_F | W_A | W_PF | W_BW, 32, kRingBB, kRingBS, busyB,
          [&](const unsigned char* sb, const StageLayout& L, int rmax, int64_t i0) {
      bbody(sb, L, rmax, i0, std::true_type{});
    });
  __syncthreads();  // the ring (incl. the histogram space) is free for the resolve keys
  stamp(3);

  if (live && !exact_f && !region_G(Tq, wneg, Lsc, &G)) live = false;  // exact dead test
  double v = 0.0, e = 0.0;
  bool done = !active;
  if (active && !live) {
    done = true;  // dead column (fit.py:60-63 returns +0.0): residual = sum_i |x_ij|
    e = P.colsum[j];
  }
  // hand the window to k_resolve (its exact keys need scattered L2 loads, so
  // it runs as its own high-occupancy kernel instead of holding this CTA's
  // shared memory), or an overflowing window to the straggler solver
  if (piv_ok && j < m) {
    const int64_t prob = kk * m + j;
    const int64_t NP = P.npiv * m;
    const bool rec = active && live && cnt <= CAP;
    P.rcnt[prob] = rec ? cnt : -1;
    if (rec) {
      P.rG[prob] = G;
      P.rwb[prob] = wb;
      P.res[prob] = es;
      P.rLw[prob] = Lw;
      P.rHw[prob] = Hw;
      RowT* rows = (RowT*)P.rrows;
      for (int c = 0; c < cnt; ++c) rows[c * NP + prob] = cbuf[c * kBS + tid];
      done = true;  // k_resolve writes V / E (or queues a straggler)
    }
  }
  if (active && live && cnt > CAP) {
    // window overflow (heavy ties / wide window): the crossing is most likely
    // in [Lg, Hg); the straggler solver widens the interval itself if not
    Straggler s;
    s.kk = (int)kk;
    s.j = (int)j;
    s.G = G;
    s.lo = key64((double)Lg - fabs((double)Lg) * 0x1p-20);
    s.hi = key64((double)Hg + fabs((double)Hg) * 0x1p-20);
    s.wb = 0.0;
    unsigned long long slot = atomicAdd(P.nstrag, 1ULL);
    P.strag[slot] = s;
  }

  __syncthreads();
  stamp(4);
  if (piv_ok && j < m) {
    if (degenerate) {
      P.V[kk * m + j] = 0.0;
      P.E[kk * m + j] = P.colsum[j];
    } else if (j == p) {
      P.V[kk * m + j] = 1.0;
      P.E[kk * m + j] = 0.0;
    } else if (active && !live) {
      P.V[kk * m + j] = v;
      P.E[kk * m + j] = e;
    }
  }
}

// ---------------------------------------------------------------- resolve --
//
// One thread per (pivot, target) problem with a window record from
// k_select: exact keys of the collected rows (loads batched for ILP, the
// kernel runs at high occupancy to hide the L2 latency), guard-band rows
// below Lw / at or above Hw join the sides, the window rows are sorted by
// (key, row) -- stable insertion; rows were collected in ascending order --
// and walked to the crossing.  Residual: pass B summed |x_ij - c0 x_ip| over
// every row; the window rows are taken back out and re-added as
// |x_ij - fl(v x_ip)| (core.py:93 rounding), and the sides move from c0 to v
// by (v - c0)(W_below - W_above) exactly as in the pass-B identity.

constexpr int kRBS = 128;  // threads per k_resolve block

constexpr int kNSB = 16;  // exact-weight sub-bins of the window in k_resolve
constexpr int kList = 8;  // rows of the crossing sub-bin ordered exactly

template <typename RowT, int CAP>
constexpr size_t resolve_smem() {
  return (size_t)kRBS * (kNSB * 2 * sizeof(double) + kList * (2 * sizeof(double) + 1));
}

// Thread per problem; work linear in the window size (no sort of the whole
// window): (1a) exact keys of the collected rows, guard-band rows settled,
// the window rows' exact weights (and weighted offsets, for the residual)
// summed into 16 sub-bins that split [Lw, Hw) monotonically in the exact
// ratio; the walk finds the crossing sub-bin; (1b) the rows of that sub-bin
// (usually one or two) are re-gathered and ordered exactly by (key, row).
template <typename RowT, int CAP>
__global__ void __launch_bounds__(kRBS) k_resolve(SelParams P) {
  extern __shared__ __align__(16) unsigned char rsm[];
  double* sbW = (double*)rsm;                                         // [kNSB][kRBS]
  double* sbR = sbW + kNSB * kRBS;                                    // [kNSB][kRBS]
  unsigned long long* lk = (unsigned long long*)(sbR + kNSB * kRBS);  // [kList][kRBS]
  double* lw = (double*)(lk + kList * kRBS);                          // [kList][kRBS]
  unsigned char* lc = (unsigned char*)(lw + kList * kRBS);            // [kList][kRBS]
  const int tid = threadIdx.x;
  const int64_t NP = P.npiv * P.m;
  const int64_t prob = (int64_t)blockIdx.x * kRBS + tid;
  if (prob >= NP) return;
  const int cnt = P.rcnt[prob];
  if (cnt < 0) return;
  const int64_t m = P.m, n = P.n;
  const int64_t kk = prob / m, j = prob - kk * m;
  const int64_t p = pivot_of(P, kk);
  const double G = P.rG[prob], Lw = P.rLw[prob], Hw = P.rHw[prob];
  double wb = P.rwb[prob], es = P.res[prob];
  const double c0 = Lw > -kBig ? Lw : Hw;
  const double Tq = P.tq[p];
  const int sp = P.spow[p];
  const double unit = ldexp(1.0, -sp);
  const double scale2 = ldexp(1.0, sp);  // |x_ip| * 2^s is exact: a power-of-two product
  const double* xcol = P.Xc + j * n;
  const double* pbp = P.pb + p * P.np;
  const RowT* rows = (const RowT*)P.rrows;
  const unsigned long long KL = key64(Lw), KH = key64(Hw);
  // sub-bin s <-> exact ratio r in [Lw + s/scale, Lw + (s+1)/scale); an open
  // window (an infinite edge) puts every row in sub-bin 0
  const double span = Hw - Lw;
  const bool finite = span > 0.0 && span < 1e300;
  const double scale = finite ? (double)kNSB / span : 0.0;
  const double width = finite ? span * (1.0 / kNSB) : 0.0;
  auto subbin = [&](double r) { return min(kNSB - 1, max(0, (int)((r - Lw) * scale))); };
  // reference point of a sub-bin for the weighted offsets (any fixed value
  // near the sub-bin works; it only keeps the sums small)
  auto edge = [&](int sb) { return finite ? __fma_rn((double)sb, width, Lw) : 0.0; };
  for (int sb = 0; sb < kNSB; ++sb) {
    sbW[sb * kRBS + tid] = 0.0;
    sbR[sb * kRBS + tid] = 0.0;
  }
  // exact key and weight of collected row c (x_ij, x_ip gathered -- L2
  // resident; the pivot's reciprocal and weight recomputed as K0 did)
  auto gather4 = [&](int c0i, double* a, double* bb) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool ok = c0i + u < cnt;
      const int row = ok ? (int)rows[(c0i + u) * NP + prob] : 0;
      a[u] = ok ? xcol[row] : 0.0;
      bb[u] = ok ? pbp[row] : 0.0;
    }
  };
  double win = 0.0;
  for (int c0i = 0; c0i < cnt; c0i += 4) {  // phase 1a
    double a[4], bb[4];
    gather4(c0i, a, bb);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (c0i + u >= cnt) break;
      if (bb[u] == 0.0) continue;  // dropped row: no weight, |x_ij| already in es
      const double w = rint(fabs(bb[u]) * scale2);
      const double q = ratio_fast(a[u], bb[u], recip_refined(bb[u]));
      const unsigned long long k = key64(q);
      if (k < KL) { wb += w; continue; }
      if (k >= KH) continue;
      es -= fabs(__fma_rn(-bb[u], c0, a[u]));  // pass B added every row
      win += w;
      const int sb = subbin(q);
      sbW[sb * kRBS + tid] += w;
      sbR[sb * kRBS + tid] += w * (q - edge(sb));
    }
  }
  bool ok = wb <= G && G < wb + win;
  int sstar = 0;
  double cum = wb;
  if (ok) {
    for (sstar = 0; sstar < kNSB - 1; ++sstar) {
      const double h = sbW[sstar * kRBS + tid];
      if (cum + h > G) break;
      cum += h;
    }
  }
  // phase 1b: the crossing sub-bin's rows, ordered exactly (stable insertion;
  // collection order is row order)
  int nl = 0;
  if (ok) {
    for (int c0i = 0; c0i < cnt && nl <= kList; c0i += 4) {
      double a[4], bb[4];
      gather4(c0i, a, bb);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (c0i + u >= cnt || bb[u] == 0.0) continue;
        const double q = ratio_fast(a[u], bb[u], recip_refined(bb[u]));
        const unsigned long long k = key64(q);
        if (k < KL || k >= KH || subbin(q) != sstar) continue;
        if (nl == kList) { nl = kList + 1; break; }
        int d = nl++;
        while (d > 0 && lk[(d - 1) * kRBS + tid] > k) {
          lk[d * kRBS + tid] = lk[(d - 1) * kRBS + tid];
          lw[d * kRBS + tid] = lw[(d - 1) * kRBS + tid];
          lc[d * kRBS + tid] = lc[(d - 1) * kRBS + tid];
          --d;
        }
        lk[d * kRBS + tid] = k;
        lw[d * kRBS + tid] = rint(fabs(bb[u]) * scale2);
        lc[d * kRBS + tid] = (unsigned char)(c0i + u);
      }
    }
    ok = nl <= kList;  // heavy ties inside one sub-bin: the straggler solver takes it
  }
  double v = 0.0;
  if (ok) {
    ok = false;
    for (int c = 0; c < nl; ++c) {
      cum += lw[c * kRBS + tid];
      if (cum > G) {
        const unsigned long long k = lk[c * kRBS + tid];
        if (k == kZeroKey) {  // a zero takes the sign of its own row
          const int row = (int)rows[(int)lc[c * kRBS + tid] * NP + prob];
          v = __ddiv_rn(xcol[row], pbp[row]);
        } else {
          v = key64_inv(k);
        }
        ok = true;
        break;
      }
    }
  }
  if (!ok) {
    Straggler s;
    s.kk = (int)kk;
    s.j = (int)j;
    s.G = G;
    if (G < wb) { s.lo = 0; s.hi = KL - 1; }               // crossing below the window
    else if (G >= wb + win) { s.lo = KH; s.hi = ~0ULL; }   // above it
    else { s.lo = KL; s.hi = KH - 1; }                     // inside, heavy ties
    s.wb = 0.0;
    unsigned long long slot = atomicAdd(P.nstrag, 1ULL);
    P.strag[slot] = s;
    return;
  }
  // window residual at v: whole sub-bins below / above v from their sums
  // (sum w (v - r) = W (v - edge) - R, sum w (r - v) = R + W (edge - v)),
  // the crossing sub-bin's rows one by one (|x_ij - v x_ip| = |x_ip||r - v|)
  double ew = 0.0;
  for (int sb = 0; sb < kNSB; ++sb) {
    const double W = sbW[sb * kRBS + tid], R = sbR[sb * kRBS + tid];
    if (sb < sstar) ew += W * (v - edge(sb)) - R;
    else if (sb > sstar) ew += R + W * (edge(sb) - v);
  }
  for (int c = 0; c < nl; ++c) ew += lw[c * kRBS + tid] * fabs(key64_inv(lk[c * kRBS + tid]) - v);
  const double wa = Tq - wb - win;  // exact
  P.V[prob] = v;
  P.E[prob] = es + ew * unit + (v - c0) * ((wb - wa) * unit);
}

// Route every problem of a shard to the straggler queue (inputs outside the
// fast path's exponent window use k_straggle for everything).
__global__ void k_queue_all(SelParams P) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= P.npiv * P.m) return;
  int64_t kk = idx / P.m, j = idx - kk * P.m;
  int64_t p = pivot_of(P, kk);
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
  const int64_t sr = P.seeds ? P.seeds[kk] : -1;
  if (sr >= 0) {
    // seeded: the bound passes' range for v, widened by a few float ulps;
    // a range that misses is widened by k_straggle itself
    const double2 r = P.BRK[sr * P.m + j];
    if (r.x > -INFINITY && r.y < INFINITY && r.x <= r.y) {
      s.lo = key64(r.x - fabs(r.x) * 0x1p-18 - 0x1p-1000);
      s.hi = key64(r.y + fabs(r.y) * 0x1p-18 + 0x1p-1000);
    }
  }
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

constexpr int kSWarps = 8;
constexpr int kSCap = 128;   // interval elements collected and sorted per round
constexpr int kSBins = 256;  // radix bins when the interval holds more
constexpr int kSUnroll = 4;  // rows per lane in flight (loads hoisted for ILP)

struct SEnt {
  unsigned long long k;
  double w;
  int row;
  int pad;
};

constexpr size_t kStraggleSmem =
    (size_t)kSWarps * (kSCap * sizeof(SEnt) + kSBins * sizeof(unsigned long long));

template <bool SAFE>
__device__ __forceinline__ double sratio(const SelParams& P, double a, double b, double y) {
  if (SAFE) return ratio_fast(a, b, y);
  return b != 0.0 ? __ddiv_rn(a, b) : __longlong_as_double(0x7ff8000000000000LL);
}


// Visit every row with nonzero weight of problem (p, j): f(row, key, weight).
// kSUnroll rows per lane are loaded before any is used, so a warp keeps
// 4 x 4 independent loads in flight per lane (the loop is latency-bound).
template <bool SAFE, typename F>
__device__ __forceinline__ void for_rows(const SelParams& P, int64_t p, int64_t j, int lane, F&& f) {
  const int64_t n = P.n;
  const double* xc = P.Xc + j * n;
  const double* pb = P.pb + p * P.np;
  const double* py = P.py + p * P.np;
  const double* pw = P.pw + p * P.np;
  for (int64_t i0 = 0; i0 < n; i0 += 32 * kSUnroll) {
    double a[kSUnroll], b[kSUnroll], y[kSUnroll], w[kSUnroll];
#pragma unroll
    for (int u = 0; u < kSUnroll; ++u) {
      const int64_t i = i0 + u * 32 + lane;
      const bool ok = i < n;
      a[u] = ok ? xc[i] : 0.0;
      b[u] = ok ? pb[i] : 0.0;
      y[u] = ok ? py[i] : 0.0;
      w[u] = ok ? pw[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kSUnroll; ++u) {
      const int64_t i = i0 + u * 32 + lane;
      const bool ok = i < n && w[u] != 0.0;
      const unsigned long long k = ok ? key64(sratio<SAFE>(P, a[u], b[u], y[u])) : 0ULL;
      f(ok, (int)i, k, w[u]);
    }
  }
}

template <bool SAFE>
__global__ void __launch_bounds__(kSWarps * 32, 3) k_straggle(SelParams P) {
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
    const int64_t kk = s.kk, j = s.j, p = pivot_of(P, kk);
    const double Tq = P.tq[p];
    const double Lsc = ldexp(lam_of(P, kk), P.spow[p]);
    double G = s.G;
    unsigned long long lo = s.lo, hi = s.hi;
    bool dead = false;
    // G unknown with a seeded range: the first collecting pass sums Wneg too
    bool needG = G < 0.0 && !(lo == 0 && hi == ~0ULL);
    if (G < 0.0 && !needG) {  // exact Wneg and key range first
      double wneg = 0.0;
      unsigned long long kmin = ~0ULL, kmax = 0;
      for_rows<SAFE>(P, p, j, lane, [&](bool ok, int, unsigned long long k, double w) {
        if (!ok) return;
        if (k < kZeroKey) wneg += w;  // key below +-0 <=> ratio < 0
        kmin = min(kmin, k);
        kmax = max(kmax, k);
      });
      wneg = warp_sum(wneg);
      for (int o = 16; o; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
      }
      dead = !region_G(Tq, wneg, Lsc, &G);
      lo = kmin;
      hi = kmax;
    }
    double v = 0.0;
    bool ok = dead;
    // Each round visits every row once, recomputing the exact weight below
    // the interval (so an interval from k_select need not come with one),
    // and either collects the interval (<= kSCap elements: sort + walk) or
    // narrows it by a 256-bin exact radix histogram.  A walk that misses
    // moves the interval to the side holding the crossing.
    for (int round = 0; round < 64 && !ok; ++round) {
      double wbl = 0.0;  // exact weight with key < lo
      if (lo == hi) {
        // one key left (heavy exact ties): the value is that key; only a
        // zero needs the crossing row itself (its sign), found by an
        // in-order prefix walk over the tied rows
        if (lo != kZeroKey) {
          v = key64_inv(lo);
          ok = true;
          break;
        }
        for_rows<SAFE>(P, p, j, lane, [&](bool okr, int, unsigned long long k, double w) {
          if (okr && k < lo) wbl += w;
        });
        double cum = warp_sum(wbl);
        int hit_row = -1;
        for_rows<SAFE>(P, p, j, lane, [&](bool okr, int row, unsigned long long k, double w) {
          double x = (okr && k == lo) ? w : 0.0;
          for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          const unsigned cm = __ballot_sync(0xffffffffu, x > 0.0 && cum + x > G);
          if (hit_row < 0 && cm) hit_row = __shfl_sync(0xffffffffu, row, __ffs(cm) - 1);
          cum += __shfl_sync(0xffffffffu, x, 31);
        });
        if (hit_row < 0) break;
        v = __ddiv_rn(P.Xc[j * n + hit_row], P.pb[p * P.np + hit_row]);
        ok = true;
        break;
      }
      // collect the interval's elements (in row order) if they fit
      int base = 0;
      double wneg = 0.0;
      for_rows<SAFE>(P, p, j, lane, [&](bool okr, int row, unsigned long long k, double w) {
        const bool in = okr && k >= lo && k <= hi;
        if (okr && k < lo) wbl += w;
        if (needG && okr && k < kZeroKey) wneg += w;
        const unsigned mask = __ballot_sync(0xffffffffu, in);
        const int pos = base + __popc(mask & ((1u << lane) - 1));
        if (in && pos < kSCap) ent[warp][pos] = SEnt{k, w, row, 0};
        base += __popc(mask);
      });
      wbl = warp_sum(wbl);
      __syncwarp();
      if (needG) {
        needG = false;
        if (!region_G(Tq, warp_sum(wneg), Lsc, &G)) {  // dead: v = 0
          v = 0.0;
          ok = true;
          break;
        }
      }
      if (G < wbl) {  // the crossing lies below the interval
        hi = lo - 1;
        lo = 0;
        continue;
      }
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
        double cum = wbl;
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
        } else {  // the crossing lies above the interval
          if (hi == ~0ULL) break;  // cannot happen: weights above sum to Tq
          lo = hi + 1;
          hi = ~0ULL;
        }
        __syncwarp();
      } else {
        // narrow: exact weight per key bucket (integer-valued weights, so
        // 64-bit integer shared atomics are exact and order-independent)
        int sh = (hi - lo == ~0ULL) ? 56 : ceil_log2_u64(hi - lo + 1) - 8;
        sh = sh > 0 ? sh : 0;
        for (int b = lane; b < kSBins; b += 32) bins[warp][b] = 0ULL;
        __syncwarp();
        for_rows<SAFE>(P, p, j, lane, [&](bool okr, int, unsigned long long k, double w) {
          if (okr && k >= lo && k <= hi) atomicAdd(&bins[warp][(k - lo) >> sh], (unsigned long long)w);
        });
        __syncwarp();
        double cum = wbl;
        int bsel = kSBins - 1;
        for (int b = 0; b < kSBins; ++b) {
          const double hb = (double)bins[warp][b];
          if (cum + hb > G) { bsel = b; break; }
          cum += hb;
        }
        const unsigned long long nlo = lo + ((unsigned long long)bsel << sh);
        unsigned long long nhi = nlo + ((1ULL << sh) - 1);
        if (nhi > hi || nhi < nlo) nhi = hi;
        lo = nlo;
        hi = nhi;
        __syncwarp();
      }
    }
    if (!ok) {
      if (lane == 0) atomicExch(P.status, L1B_EINTERNAL);
      v = 0.0;
    }
    double e = 0.0;
    const double* pbp = P.pb + p * P.np;
    const double* xc = P.Xc + j * n;
#pragma unroll 4
    for (int64_t i = lane; i < n; i += 32) e += fabs(__dsub_rn(xc[i], __dmul_rn(pbp[i], v)));
    e = warp_sum(e);
    if (lane == 0) {
      P.V[kk * m + j] = v;
      P.E[kk * m + j] = e;
    }
    __syncwarp();
  }
}

// ------------------------------------------------ block-per-problem solver --
//
// The seeded exact fit of a few candidate pivots over tall data (n large):
// k_straggle's rounds with a whole CTA per problem, rows strided over its
// 256 threads, so few problems still fill the GPU.  Each round visits every
// row once: exact weight below the key interval, Wneg on the first round
// (for G), and the interval's elements collected into shared memory; if they
// fit (<= kBlkCap) they are bitonic-sorted by (key, row) and walked in order,
// else a second visit narrows the interval by a 256-bucket exact histogram.
// Starts on the range the bound cascade left (P.BRK row P.seeds[k]).

constexpr int kBlkThreads = 256;
constexpr int kBlkCap = 2048;
constexpr size_t kBlkSmem = (size_t)kBlkCap * sizeof(SEnt) + kSBins * sizeof(unsigned long long);

__device__ __forceinline__ double block_sum(double x, double* red) {
  x = warp_sum(x);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();  // red is reused
  if (l == 0) red[w] = x;
  __syncthreads();
  double t = 0.0;
  for (int k = 0; k < kBlkThreads / 32; ++k) t += red[k];  // fixed order, every thread
  return t;
}

template <bool SAFE>
__global__ void __launch_bounds__(kBlkThreads) k_block_solve(SelParams P) {
  extern __shared__ __align__(16) unsigned char bsm[];
  SEnt* ent = reinterpret_cast<SEnt*>(bsm);
  unsigned long long* bins = reinterpret_cast<unsigned long long*>(bsm + (size_t)kBlkCap * sizeof(SEnt));
  __shared__ double red[kBlkThreads / 32];
  __shared__ int cnt_s;
  const int tid = threadIdx.x;
  const int64_t n = P.n, m = P.m;
  for (int64_t prob = blockIdx.x; prob < P.npiv * m; prob += gridDim.x) {
    const int64_t kk = prob / m, j = prob - kk * m, p = pivot_of(P, kk);
    if (P.nnz[p] == 0 || j == p) {  // degenerate pivot / the pivot's own column
      if (tid == 0) {
        P.V[prob] = P.nnz[p] == 0 ? 0.0 : 1.0;
        P.E[prob] = P.nnz[p] == 0 ? P.colsum[j] : 0.0;
      }
      continue;
    }
    const double Tq = P.tq[p], Lsc = ldexp(lam_of(P, kk), P.spow[p]);
    unsigned long long lo = 0, hi = ~0ULL;
    const int64_t sr = P.seeds ? P.seeds[kk] : -1;
    if (sr >= 0) {
      const double2 r = P.BRK[sr * m + j];
      if (r.x > -INFINITY && r.y < INFINITY && r.x <= r.y) {
        lo = key64(r.x - fabs(r.x) * 0x1p-18 - 0x1p-1000);
        hi = key64(r.y + fabs(r.y) * 0x1p-18 + 0x1p-1000);
      }
    }
    const double* xc = P.Xc + j * n;
    const double* pb = P.pb + p * P.np;
    const double* py = P.py + p * P.np;
    const double* pw = P.pw + p * P.np;
    auto row_key = [&](int64_t i, double* w) -> unsigned long long {
      *w = pw[i];
      return key64(sratio<SAFE>(P, xc[i], pb[i], py[i]));
    };
    double G = -1.0, v = 0.0;
    bool ok = false;
    for (int round = 0; round < 64 && !ok; ++round) {
      const bool needG = G < 0.0;
      if (lo == hi && !needG) {
        // one key left (heavy exact ties): the value is that key; only a zero
        // needs the crossing row itself (its sign), found by an in-order
        // prefix walk over the tied rows, 256 rows at a time
        if (lo != kZeroKey) {
          v = key64_inv(lo);
          ok = true;
          break;
        }
        double wb = 0.0;
        for (int64_t i = tid; i < n; i += kBlkThreads) {
          double w;
          const unsigned long long k = row_key(i, &w);
          if (w != 0.0 && k < lo) wb += w;
        }
        double cum = block_sum(wb, red);
        int hit_row = -1;
        for (int64_t i0 = 0; i0 < n && hit_row < 0; i0 += kBlkThreads) {
          const int64_t i = i0 + tid;
          double x = 0.0;
          if (i < n) {
            double w;
            const unsigned long long k = row_key(i, &w);
            x = (w != 0.0 && k == lo) ? w : 0.0;
          }
          // inclusive block scan of x in row order
          double y = x;
          for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, y, o);
            if ((tid & 31) >= o) y += t;
          }
          __syncthreads();
          if ((tid & 31) == 31) red[tid >> 5] = y;
          __syncthreads();
          double off = 0.0, tot = 0.0;
          for (int k = 0; k < kBlkThreads / 32; ++k) {
            off += k < (tid >> 5) ? red[k] : 0.0;
            tot += red[k];
          }
          const bool hit = x > 0.0 && cum + off + y > G;
          if (tid == 0) cnt_s = 0x7fffffff;
          __syncthreads();
          if (hit) atomicMin(&cnt_s, tid);
          __syncthreads();
          if (cnt_s != 0x7fffffff) hit_row = (int)(i0 + cnt_s);
          cum += tot;
          __syncthreads();
        }
        if (hit_row >= 0) {
          v = __ddiv_rn(xc[hit_row], pb[hit_row]);
          ok = true;
        }
        break;
      }
      if (tid == 0) cnt_s = 0;
      __syncthreads();
      double wbl = 0.0, wneg = 0.0;
      for (int64_t i = tid; i < n; i += kBlkThreads) {
        double w;
        const unsigned long long k = row_key(i, &w);
        if (w == 0.0) continue;  // x_ip = 0: not in the tableau (ratios.py:115)
        if (k < lo) wbl += w;
        if (needG && k < kZeroKey) wneg += w;
        if (k >= lo && k <= hi) {
          const int pos = atomicAdd(&cnt_s, 1);
          if (pos < kBlkCap) ent[pos] = SEnt{k, w, (int)i, 0};
        }
      }
      wbl = block_sum(wbl, red);
      if (needG) {
        wneg = block_sum(wneg, red);
        if (!region_G(Tq, wneg, Lsc, &G)) {  // dead: v = +0.0
          v = 0.0;
          ok = true;
          break;
        }
      }
      const int cnt = cnt_s;
      if (G < wbl) {  // the crossing lies below the interval
        hi = lo - 1;
        lo = 0;
        continue;
      }
      if (cnt <= kBlkCap) {
        int np2 = 1;
        while (np2 < cnt) np2 <<= 1;
        for (int e = cnt + tid; e < np2; e += kBlkThreads) ent[e] = SEnt{~0ULL, 0.0, 0x7fffffff, 0};
        __syncthreads();
        for (int kq = 2; kq <= np2; kq <<= 1) {
          for (int jq = kq >> 1; jq > 0; jq >>= 1) {
            for (int e = tid; e < np2; e += kBlkThreads) {
              const int l = e ^ jq;
              if (l > e) {
                const SEnt a = ent[e], b = ent[l];
                const bool gt = a.k > b.k || (a.k == b.k && a.row > b.row);
                if (gt == ((e & kq) == 0)) {
                  ent[e] = b;
                  ent[l] = a;
                }
              }
            }
            __syncthreads();
          }
        }
        // in-order walk (warp 0): the first element whose prefix exceeds G
        int hit = -1;
        if (tid < 32) {
          double cum = wbl;
          for (int e0 = 0; e0 < cnt && hit < 0; e0 += 32) {
            const int e = e0 + tid;
            double x = e < cnt ? ent[e].w : 0.0;
            for (int o = 1; o < 32; o <<= 1) {
              const double y = __shfl_up_sync(0xffffffffu, x, o);
              if (tid >= o) x += y;
            }
            const unsigned cm = __ballot_sync(0xffffffffu, e < cnt && cum + x > G);
            if (cm) hit = e0 + __ffs(cm) - 1;
            cum += __shfl_sync(0xffffffffu, x, 31);
          }
          if (tid == 0) cnt_s = hit;
        }
        __syncthreads();
        hit = cnt_s;
        if (hit >= 0) {
          const SEnt h = ent[hit];
          v = h.k == kZeroKey ? __ddiv_rn(xc[h.row], pb[h.row]) : key64_inv(h.k);
          ok = true;
        } else {  // the crossing lies above the interval
          if (hi == ~0ULL) break;
          lo = hi + 1;
          hi = ~0ULL;
        }
        __syncthreads();
      } else {
        // narrow: exact weight per key bucket, then the crossing bucket
        int sh = (hi - lo == ~0ULL) ? 56 : ceil_log2_u64(hi - lo + 1) - 8;
        sh = sh > 0 ? sh : 0;
        for (int b = tid; b < kSBins; b += kBlkThreads) bins[b] = 0ULL;
        __syncthreads();
        for (int64_t i = tid; i < n; i += kBlkThreads) {
          double w;
          const unsigned long long k = row_key(i, &w);
          if (w != 0.0 && k >= lo && k <= hi) atomicAdd(&bins[(k - lo) >> sh], (unsigned long long)w);
        }
        __syncthreads();
        if (tid == 0) {
          double cum = wbl;
          int bsel = kSBins - 1;
          for (int b = 0; b < kSBins; ++b) {
            const double hb = (double)bins[b];
            if (cum + hb > G) { bsel = b; break; }
            cum += hb;
          }
          red[0] = __longlong_as_double((long long)bsel);
        }
        __syncthreads();
        const int bsel = (int)__double_as_longlong(red[0]);
        const unsigned long long nlo = lo + ((unsigned long long)bsel << sh);
        unsigned long long nhi = nlo + ((1ULL << sh) - 1);
        if (nhi > hi || nhi < nlo) nhi = hi;
        lo = nlo;
        hi = nhi;
        __syncthreads();
      }
    }
    if (!ok) {
      if (tid == 0) atomicExch(P.status, L1B_EINTERNAL);
      v = 0.0;
    }
    double e = 0.0;
    for (int64_t i = tid; i < n; i += kBlkThreads) e += fabs(__dsub_rn(xc[i], __dmul_rn(pb[i], v)));
    e = block_sum(e, red);
    if (tid == 0) {
      P.V[prob] = v;
      P.E[prob] = e;
    }
    __syncthreads();
  }
}
