// Post-map, rounding and recombination by runs: the carry kernel of the large
// products (with k_carry_patch for the block carry-ins).
//
// A run is 64 consecutive coefficients: their bit offsets k b span exactly b
// limbs, so every run starts on a limb boundary whatever b is.  One thread
// owns one run.  It walks its coefficients in order: the post-map output
// from a sliding window of convolution values (beta* low, delta+ high; the
// same fused multiply-adds in the same order as the gather form of
// k_carry_lanes, so the values are bit-identical), the checked rounding
// (products_f64.cpp:16-27), and acc += e << sh on one signed 128-bit
// accumulator, emitting a finished limb whenever sh passes 64.  All threads
// of a warp emit at the same steps (every run starts at sh = 0), so the
// walk has no divergence, and a coefficient costs about 30 integer
// instructions plus its post-map, against more than a hundred for the
// per-limb lanes of k_carry_lanes.
//
// A run's convolution values arrive by one bulk copy per thread
// (cp.async.bulk on the warp's mbarrier) into a slot of the thread's own,
// whose stride is an odd multiple of 16 bytes: the threads' 128-bit reads
// at equal offsets fall in distinct banks.  The run's b limbs overwrite the
// slot's head in place.
//
// What leaves a run upward is split like the lanes of SignedAccumulator
// (products_f64.cpp:36-66): hi(lane) of the run's last limb, a value the
// next run adds to its first limb, and a carry d in {-1, 0, 1}.  With that
// split a block needs only the few coefficients of the limb below it (not
// the resolved carry of the whole block before it).  Each run then has a
// carry transfer function (first limb: limb_tf; the others pass +1 through
// all-ones and -1 through all-zero limbs; plus d), the block scans them,
// the limbs are fixed up for a zero carry into the block and stored, and
// the block's composed function goes to aggs[blk] for k_carry_patch.
//
// Runs that touch the wrap outputs of the cyclic maps, the fold region of
// the high product or the end of the coefficients are evaluated one
// coefficient per thread with the generic helpers first (from global
// memory), and their owners read the rounded values from the slot.
//
// Reference: products_f64.cpp:29-102 (SignedAccumulator, round_accumulate),
// maps_f64.cpp:140-188, 269-281, 350-384 (beta*, delta+).
#include "kernels.cuh"

namespace tmg {

namespace {

constexpr int kRT = kRunThreads;  // threads (runs) per block
constexpr int kRun = 64;          // coefficients per run
constexpr int kHaloBelow = 16;    // window of the limb below the block: 8 coefficients, their post-map inputs
constexpr int kHaloWin = kHaloBelow + 2;

// Slot geometry (doubles): [k0 - hlo, k0 + 64 + hhi) plus padding so that
// slot / 2 is odd.
template <int MODE, int LAM, int RUN = 64>
struct RunGeom {
  static constexpr int need_lo = MODE == kModeFull ? 0 : MODE == kModeLow ? (LAM > 2 ? LAM - 2 : 0) : LAM;
  static constexpr int hhi = MODE == kModeLow ? 2 : 0;
  static constexpr int hlo0 = (need_lo + 1) & ~1;
  static constexpr int pad0 = MODE == kModeFull ? 2 : 0;
  // slot / 2 odd: grow the lower halo by 2 when needed
  static constexpr int hlo = (((RUN + hlo0 + hhi + pad0) / 2) & 1) ? hlo0 : hlo0 + 2;
  static constexpr int slot = RUN + hlo + hhi + pad0;
  static_assert((slot / 2) % 2 == 1 && slot % 2 == 0, "slot stride must be an odd multiple of 16 bytes");
};

__device__ __forceinline__ void add_shifted(unsigned long long& lo, long long& hi, long long e, uint32_t sh) {
  const unsigned long long l = (unsigned long long)e << sh;
  const long long h = (e >> 1) >> (63 - sh);  // arithmetic; sh = 0 gives the sign word
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(l), "l"(h));
}

// The rare path of round8 (a magnitude of 2^51 or more, or a NaN), out of line.
__device__ __noinline__ void round8_wide(double& max_err, double& max_abs, uint32_t& flags, const double (&x)[8],
                                         long long (&e)[8]) {
  RoundAcc r;
  r.max_err = max_err;
  r.max_abs = max_abs;
  r.flags = flags;
  for (int q = 0; q < 8; ++q) e[q] = r.round(x[q]);
  max_err = r.max_err;
  max_abs = r.max_abs;
  flags = r.flags;
}

// Checked rounding of eight values at once (RoundAcc::round on each, same
// results): the magnitude maximum first, then the magic-number rounding of
// all eight when it stays below 2^51 (a NaN makes the maximum a NaN and
// takes the checked path).
__device__ __forceinline__ void round8(RoundAcc& ra, const double (&x)[8], long long (&e)[8]) {
  double am = ra.max_abs;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const double ax = fabs(x[q]);
    am = !(ax <= am) ? ax : am;
  }
  if (am < 2251799813685248.0) {
    ra.max_abs = am;
    double me = ra.max_err;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const double t = x[q] + 6755399441055744.0;
      const double r = t - 6755399441055744.0;
      const double d = fabs(x[q] - r);
      me = d > me ? d : me;
      e[q] = __double_as_longlong(t) - 0x4338000000000000ll;
    }
    ra.max_err = me;
  } else {
    // (copies: only these escape to the out-of-line call)
    double me = ra.max_err, ma = ra.max_abs, xl[8];
    uint32_t fl = ra.flags;
    long long el[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) xl[q] = x[q];
    round8_wide(me, ma, fl, xl, el);
#pragma unroll
    for (int q = 0; q < 8; ++q) e[q] = el[q];
    ra.max_err = me;
    ra.max_abs = ma;
    ra.flags = fl;
  }
}

// Coefficient k by the generic helpers (any k in [0, K)): the wrap outputs,
// the fold region, x_N.  The flat post-map term has the gather form's
// operation order, so interior values equal the walk's.
template <int MODE, int LAM>
__device__ __noinline__ long long coef_generic(const CarryArgs& a, int64_t k, double psi, RoundAcc& ra,
                                               uint32_t& flags) {
  const MapConsts& mc = a.mc;
  auto WS = [&](int64_t j) -> double { return __ldg(a.w + j); };
  if constexpr (MODE == kModeFull) {
    return ra.round(WS(k));
  } else {
    const int64_t N = mc.N;
    const double st = MODE == kModeLow ? double(N) : -double(N);
    const double step = mc.step, sc = mc.scale_out;
    auto pf = [&](int64_t j) -> double {
      double acc = 0.0;
#pragma unroll
      for (int r = LAM - 1; r >= 1; --r) {
        const int64_t i = j - r;
        if (i >= 0 && i < N) {
          const double id = double(i);
          double p = id, f = id + st;
#pragma unroll
          for (int t = 1; t < r; ++t) {
            p *= f;
            f += st;
          }
          acc = fma(WS(i), p * mc.cpost[r], acc);
        }
      }
      if (j >= 0 && j < N) acc = acc + WS(j);
      return acc;
    };
    if constexpr (MODE == kModeLow) {
      const int64_t i = k + 1;
      const double x = (i <= LAM - 1) ? postmap_low(mc, WS, i) : pf(i) * sc;
      long long e = ra.round(x);
      if (k == 0) {
        const long long c0v = ra.round(postmap_low(mc, WS, 0));
        if (c0v & ((1ll << mc.b) - 1)) flags |= kFlagLowNotDivisible;
        e += (c0v >> mc.b);
      }
      return e;
    } else {
      const int64_t hslow = int64_t(mc.nfold) + LAM - 2;  // hbuf(i) = post_flat(i) from here on
      auto hb = [&](int64_t i) -> double {
        if (i < 0 || i >= N) return 0.0;
        return (i < hslow) ? high_buf(mc, WS, i) : pf(i);
      };
      const double hp = hb(k - 1);
      double v = (k == N) ? psi - hp * step : hb(k) - hp * step;
      if (k < mc.nfold) v -= psi * mc.fold[k];
      return ra.round(v * sc);
    }
  }
}

// High product: limb m of t feeds w0_{m-q} (bits r..63) and w0_{m-q-1}
// (bits 0..r-1) of w0 = t >> s (see k_carry2.cu).
struct HighLimbs3 {
  int64_t hq, WL, sb;
  int hr;
  __device__ explicit HighLimbs3(const CarryArgs& a)
      : hq(int64_t(a.shift_s) >> 6), WL(a.ML - (int64_t(a.shift_s) >> 6)), sb(a.shift_s - 1),
        hr(int(a.shift_s & 63)) {}
  __device__ __forceinline__ void see(int64_t m, uint64_t x, uint32_t& hmin, uint32_t& sticky) const {
    if (hr == 0) {
      if (x != ~0ull && m - hq >= 0) hmin = min(hmin, uint32_t(m - hq));
    } else {
      const uint64_t lowm = (1ull << hr) - 1;
      if ((x >> hr) != (~0ull >> hr) && m - hq >= 0) hmin = min(hmin, uint32_t(m - hq));
      if ((x & lowm) != lowm && m - hq - 1 >= 0 && m - hq - 1 < WL) hmin = min(hmin, uint32_t(m - hq - 1));
    }
    const int64_t bit0 = 64 * m;
    if (bit0 + 64 <= sb) {
      if (x) sticky = 1;
    } else if (bit0 < sb) {
      if (x & ((1ull << (sb - bit0)) - 1)) sticky = 1;
    }
  }
};

// Flat post-map output j from a window: W[c - r] = w_{j - r}, jd = j as an
// exact double (the gather form of k_carry_lanes: same operations, same order).
template <int LAM>
__device__ __forceinline__ double pfd_w(double jd, const double* W, int c, double st, const double* cr) {
  double acc = 0.0;
#pragma unroll
  for (int r = LAM - 1; r >= 1; --r) {
    const double id = jd - double(r);
    double p = id, f = id + st;
#pragma unroll
    for (int t = 1; t < r; ++t) {
      p *= f;
      f += st;
    }
    acc = fma(W[c - r], p * cr[r], acc);
  }
  return acc + W[c];
}

// The walk's accumulator state of one run.
struct RunAcc {
  unsigned long long lo = 0;
  long long hi = 0;
  uint32_t sh = 0;
  uint32_t li = 0;              // limbs emitted
  unsigned long long rlo = 0;   // accumulator when the last limb's lane starts
  long long rhi = 0;
};

template <bool LAST>
__device__ __forceinline__ void run_step(RunAcc& s, long long e, uint32_t b, double* limbs,
                                         uint32_t i, uint32_t ilast) {
  if constexpr (LAST) {
    // coefficient ilast is the first of the run's last limb
    if (i == ilast) {
      s.rlo = s.lo;
      s.rhi = s.hi;
    }
  }
  add_shifted(s.lo, s.hi, e, s.sh);
  s.sh += b;
  if (s.sh >= 64u) {
    limbs[s.li] = __longlong_as_double((long long)s.lo);
    s.lo = (unsigned long long)s.hi;
    s.hi >>= 63;
    s.sh -= 64u;
    ++s.li;
  }
}


__host__ __device__ constexpr int gcd64(int b) { return b % 64 == 0 ? 64 : b % 32 == 0 ? 32 : b % 16 == 0 ? 16 : b % 8 == 0 ? 8 : b % 4 == 0 ? 4 : b % 2 == 0 ? 2 : 1; }

// Drives a run's eight-coefficient bodies.  With a compiled chunk width the
// shift pattern repeats every 64 / gcd(B, 64) coefficients (a whole number
// of limbs): one period is unrolled (static shifts, emission steps and limb
// offsets) and looped over, the last period apart (it holds the snapshot
// of the last limb's lane).  With a run-time width: a loop over the bodies.
template <int B, int RUN, class Body>
__device__ __forceinline__ void walk_periods(RunAcc& s, double* slot, Body& body) {
  if constexpr (B == 0) {
#pragma unroll 1
    for (uint32_t i0 = 0; i0 < RUN - 8; i0 += 8) body(i0, slot, std::false_type{});
    body(RUN - 8, slot, std::true_type{});
  } else {
    constexpr uint32_t g = uint32_t(gcd64(B)), PER = 64u / g, LPP = uint32_t(B) / g, NP = uint32_t(RUN) / PER;
    static_assert(PER >= 8 && PER % 8 == 0 && RUN % PER == 0, "period of whole bodies");
#pragma unroll 1
    for (uint32_t it = 0; it + 1 < NP; ++it) {
      s.sh = 0;
      s.li = 0;
#pragma unroll
      for (uint32_t j = 0; j < PER; j += 8) body(it * PER + j, slot + it * LPP, std::false_type{});
    }
    s.sh = 0;
    s.li = 0;
#pragma unroll
    for (uint32_t j = 0; j + 8 < PER; j += 8) body((NP - 1) * PER + j, slot + (NP - 1) * LPP, std::false_type{});
    body(RUN - 8, slot + (NP - 1) * LPP, std::true_type{});
  }
}

// B: the chunk width as a compile-time constant (the walk unrolls fully and
// every shift, emission step and slot offset is static), or 0 for any b.
// RUN: coefficients per run, 64, or 32 for an even compiled width (b / 2
// limbs per run, smaller slots, more resident warps).
template <int MODE, int LAM, int B, int RUN = 64>
__global__ void __launch_bounds__(kRT, (RUN == 32 ? 5 : 3)) k_carry_runs(const __grid_constant__ CarryArgs a) {
  using G = RunGeom<MODE, LAM, RUN>;
  static_assert(RUN == 64 || (RUN == 32 && B != 0 && B % 2 == 0), "runs are whole limbs");
  constexpr int kRun = RUN;  // (shadows the 64-coefficient default)
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t s_mbar[kRT / 32];
  __shared__ uint32_t sw[32];
  __shared__ long long s_lanehi[kRT / 32];
  __shared__ long long s_halo[8];
  __shared__ double s_terms[kMaxRootTerms + 1];
  __shared__ __align__(16) double s_hw[kHaloWin];  // w_{kblk - 16} .. w_{kblk + 1} (interior blocks)
  __shared__ double s_psi;
  __shared__ uint32_t s_flags, s_first, s_hmin, s_sticky, s_last;
  __shared__ int s_cin;
  __shared__ double2 s_red[kRT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const MapConsts& mc = a.mc;
  const uint32_t b = B ? uint32_t(B) : uint32_t(mc.b);
  const uint32_t rl = b * uint32_t(RUN) / 64u;  // limbs per run
  const int64_t K = a.K, N = mc.N;
  const int64_t blk = blockIdx.x;
  const int64_t bl = int64_t(kRT) * rl;  // limbs per block
  const int64_t ms = blk * bl;
  const int64_t me = min(a.ML, ms + bl);
  const int64_t kblk = blk * int64_t(kRT) * kRun;  // first coefficient of the block
  const int64_t k0 = kblk + int64_t(tid) * kRun;
  const int64_t m0 = ms + int64_t(tid) * rl;
  double* slots = reinterpret_cast<double*>(smem_raw);
  double* slot = slots + size_t(tid) * G::slot;
  constexpr bool hmode = MODE == kModeHigh, lowm = MODE == kModeLow, fullm = MODE == kModeFull;
  // single pass (a.runs_lb): the block's carry-in by a decoupled look-back;
  // the look-back words carry the product's generation (advanced by the row pass)
  const bool lb = a.runs_lb != 0;
  uint32_t gen = 0;
  if (lb && warp == 0) gen = *a.gen;

  // interior runs: every post-map input inside [0, N) away from the wrap
  // outputs and the fold region, all 64 coefficients below K
  bool interior;
  if constexpr (fullm) {
    interior = k0 + kRun <= K;
  } else {
    const int64_t hs0 = int64_t(mc.nfold) + LAM - 2;
    interior = k0 >= kRun && k0 + kRun + 1 <= N && k0 + kRun <= K && (lowm || k0 - 1 >= hs0);
  }
  const bool live = m0 < a.ML && k0 < K;  // the run has limbs to write and coefficients
  // Blocks whose runs are all interior (block-uniform, from the block's
  // range alone) go straight to the walk: nothing to evaluate generically,
  // no psi, no barrier before the walk.
  const int64_t kblk_end = kblk + int64_t(kRT) * kRun;
  bool blk_interior;
  if constexpr (fullm) {
    blk_interior = kblk_end <= K && ms + bl <= a.ML;
  } else {
    const int64_t hs0 = int64_t(mc.nfold) + LAM - 2;
    blk_interior = kblk >= kRun && kblk_end + 1 <= N && kblk_end <= K && ms + bl <= a.ML &&
                   (lowm || kblk - 1 >= hs0) && kblk - 8 >= mc.nfold;
  }
  // the run's window by one bulk copy per thread on the warp's mbarrier
  {
    uint32_t bytes = 0;
    if (interior && live) {
      int64_t hi_idx = k0 + kRun + G::hhi;
      if (hi_idx > a.wlen) hi_idx = a.wlen;
      bytes = uint32_t(hi_idx - (k0 - G::hlo)) * 8u;
    }
    // (interior blocks: the first warp also takes the window of the limb below the block)
    const bool halo_win = blk_interior && ms > 0 && warp == 0;
    const uint32_t total = __reduce_add_sync(0xffffffffu, bytes) + (halo_win ? uint32_t(kHaloWin) * 8u : 0u);
    if (lane == 0) {
      mbar_init(&s_mbar[warp], 1);
      mbar_expect_tx(&s_mbar[warp], total);
    }
    __syncwarp();
    if (bytes) bulk_g2s(slot, a.w + (k0 - G::hlo), bytes, &s_mbar[warp]);
    if (halo_win && lane == 0) bulk_g2s(s_hw, a.w + (kblk - kHaloBelow), uint32_t(kHaloWin) * 8u, &s_mbar[0]);
  }
  if (tid == 0) {
    s_flags = 0;
    s_first = 0xffffffffu;
    s_hmin = 0xffffffffu;
    s_sticky = 0;
    s_psi = 0.0;
  }
  RoundAcc ra;
  uint32_t flags = 0;
  if (!blk_interior) {
    // psi enters only x_N and the fold region k < nfold (delta+,
    // maps_f64.cpp:363-383): the first and the last block (the halo lane of
    // the block's first limb included).  Its hrho terms (high_psi,
    // pipeline.cuh) are chains of dependent loads: one term per thread, then
    // summed in high_psi's order.
    if (hmode && (kblk - 8 < mc.nfold || kblk_end > N)) {
      auto WS = [&](int64_t j) { return __ldg(a.w + j); };
      for (int d = 1 + tid; d <= mc.nhrho && d <= N; d += kRT) s_terms[d] = high_buf(mc, WS, N - d);
      __syncthreads();
      if (tid == 0) {
        double hrho = 0.0;
        for (int d = 1; d <= mc.nhrho && d <= N; ++d) hrho += s_terms[d] * mc.ipow[d];
        s_psi = (a.aux[0] - hrho * mc.root_neg_n) / mc.cofactor_scaled;
      }
    }
    // (the generic evaluator is out of line: it gets its own accumulator, so
    // that the walk's stays in registers)
    RoundAcc rg;
    uint32_t fg = 0;
    // runs outside the interior: one coefficient per thread into the run's slot
    const unsigned need = __ballot_sync(0xffffffffu, live && !interior);
    if (lane == 0) sw[warp] = need;
    __syncthreads();
    for (int wq = 0; wq < kRT / 32; ++wq) {
      unsigned mask = sw[wq];
      while (mask) {
        const int r = 32 * wq + __ffs(mask) - 1;
        mask &= mask - 1;
        const int64_t kr = kblk + int64_t(r) * kRun;
        for (int i = tid; i < kRun; i += kRT) {
          const int64_t k = kr + i;
          const long long e = k < K ? coef_generic<MODE, LAM>(a, k, s_psi, rg, fg) : 0;
          slots[size_t(r) * G::slot + i] = __longlong_as_double(e);
        }
      }
    }
    __syncthreads();
    ra.max_err = rg.max_err;
    ra.max_abs = rg.max_abs;
    ra.flags = rg.flags;
    flags = fg;
  }
  // first coefficient of the limb below the block: ceil(64 (ms - 1) / b), and 64 ms = b kblk
  const int64_t khalo = ms > 0 ? kblk - int64_t(64u / b) : kblk;
  // ---- the walk ----
  RunAcc s;
  // first coefficient of the run's last limb: ceil(64 (b - 1) / b)
  const uint32_t ilast = (64u * (rl - 1u) + b - 1u) / b;
  if (live) {
    if (interior) {
      mbar_wait(&s_mbar[warp], 0);
      const double2* s2 = reinterpret_cast<const double2*>(slot);
      if constexpr (fullm) {
        auto body = [&](uint32_t i0, double* limbs, auto lastc) {
          constexpr bool LASTB = decltype(lastc)::value;
          double x[8];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const double2 t = s2[i0 / 2 + q];
            x[2 * q] = t.x;
            x[2 * q + 1] = t.y;
          }
          long long ev[8];
          round8(ra, x, ev);
#pragma unroll
          for (int q = 0; q < 8; ++q) run_step<LASTB>(s, ev[q], b, limbs, i0 + q, ilast);
        };
        walk_periods<B, RUN>(s, slot, body);
      } else {
        // The flat post-map in scatter form: input w_i adds its row-r term
        // w_i (P_r(i) c_r), P_r(i) = i (i + st) ... (i + (r - 1) st), to the
        // pending sum of output i + r for r = lambda-1 .. 1 and closes output
        // i with + w_i.  Each output receives its rows in the gather form's
        // order (r = lambda-1 first, row 0 last) and the prefix products
        // P_1 .. P_{lambda-1} of one input are the gather form's own
        // products, so the values are bit-identical -- with one chain of
        // products per input instead of one per output and row (about 16
        // FP64 instructions per coefficient against 26 at lambda 5).
        // First input: lambda - 1 below the run's first output (low: j = k0 + 1;
        // high: k0 - 1, for the first difference).
        constexpr int off = G::hlo + (lowm ? 1 : 0) - (LAM - 1) - (hmode ? 1 : 0);  // its slot position
        static_assert(off >= 0, "window below the slot");
        constexpr int P0 = off + (LAM - 1) + (hmode ? 1 : 0);  // slot position of the run's first own input
        constexpr int pe = P0 & 1;                             // start one lower when odd
        constexpr int nv2 = (8 + pe + 1) / 2;                  // 16-byte loads per body
        static_assert((P0 - pe) + (kRun - 8) + 2 * nv2 <= G::slot, "window beyond the slot");
        const double st = lowm ? double(N) : -double(N);
        const double step = mc.step, sc = mc.scale_out;
        double cr[LAM];
#pragma unroll
        for (int r = 0; r < LAM; ++r) cr[r] = mc.cpost[r];
        double pend[LAM > 1 ? LAM - 1 : 1];  // pend[r - 1]: sum of output (next input + r - 1), rows >= r
#pragma unroll
        for (int r = 0; r < LAM - 1; ++r) pend[r] = 0.0;
        double idd = double(k0 + (lowm ? 1 : 0) - (LAM - 1) - (hmode ? 1 : 0));  // next input's index, exact
        auto step_in = [&](double w) -> double {
          const double out = pend[0] + w;
          double p = idd, f = idd + st;
          double np[LAM > 1 ? LAM - 1 : 1];
#pragma unroll
          for (int r = 1; r < LAM; ++r) {
            if (r > 1) {
              p *= f;
              f += st;
            }
            np[r - 1] = fma(w, p * cr[r], r < LAM - 1 ? pend[r] : 0.0);
          }
#pragma unroll
          for (int r = 0; r < LAM - 1; ++r) pend[r] = np[r];
          idd += 1.0;
          return out;
        };
        // the inputs below the run's own: their outputs are the run below's
#pragma unroll
        for (int q = 0; q < LAM - 1; ++q) (void)step_in(slot[off + q]);
        double hprev = 0.0;  // high: the previous flat output
        if constexpr (hmode) hprev = step_in(slot[off + LAM - 1]);
        auto body = [&](uint32_t i0, double* limbs, auto lastc) {
          constexpr bool LASTB = decltype(lastc)::value;
          double W[2 * nv2];
#pragma unroll
          for (int q = 0; q < nv2; ++q) {
            const double2 t = s2[(P0 - pe) / 2 + i0 / 2 + q];
            W[2 * q] = t.x;
            W[2 * q + 1] = t.y;
          }
          double x[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const double h = step_in(W[pe + q]);
            if constexpr (lowm) {
              x[q] = h * sc;
            } else {
              x[q] = (h - hprev * step) * sc;
              hprev = h;
            }
          }
          long long ev[8];
          round8(ra, x, ev);
#pragma unroll
          for (int q = 0; q < 8; ++q) run_step<LASTB>(s, ev[q], b, limbs, i0 + q, ilast);
        };
        walk_periods<B, RUN>(s, slot, body);
      }
    } else {
      // rounded coefficients from the slot (written above)
#pragma unroll 1
      for (uint32_t i = 0; i < kRun; ++i) {
        const long long e = __double_as_longlong(slot[i]);
        run_step<true>(s, e, b, slot, i, ilast);
      }
    }
  }
  // hi(lane) of the limb below the block: its coefficients, one per thread
  // (after the walk: only the block's first thread waits for them)
  if (ms > 0 && tid < 8) {
    const int64_t k = khalo + tid;
    long long e = 0;
    if (k < kblk && k < K) {
      RoundAcc rh;  // counted by the run that owns k
      if (blk_interior) {
        // from the staged window: s_hw[x] = w_{kblk - 16 + x}
        const int c = int(k - (kblk - kHaloBelow));
        if constexpr (fullm) {
          e = rh.round(s_hw[c]);
        } else {
          const double st = lowm ? double(N) : -double(N);
          double cr[LAM];
#pragma unroll
          for (int r = 0; r < LAM; ++r) cr[r] = mc.cpost[r];
          if constexpr (lowm) {
            e = rh.round(pfd_w<LAM>(double(k + 1), s_hw, c + 1, st, cr) * mc.scale_out);
          } else {
            const double h1 = pfd_w<LAM>(double(k), s_hw, c, st, cr);
            const double h0 = pfd_w<LAM>(double(k - 1), s_hw, c - 1, st, cr);
            e = rh.round((h1 - h0 * mc.step) * mc.scale_out);
          }
        }
      } else {
        uint32_t fh = 0;
        e = coef_generic<MODE, LAM>(a, k, s_psi, rh, fh);
      }
    }
    s_halo[tid] = e;
  }
  // hi(lane of the last limb) and the carry d the resolved walk adds to it
  long long lane_hi, cout = (long long)s.lo;  // after b emissions the accumulator is the carry out
  {
    // lane = acc_final - rho, acc_final = (last limb, cout)
    const unsigned long long last = live ? (unsigned long long)__double_as_longlong(slot[rl - 1]) : 0ull;
    lane_hi = cout - s.rhi - (last < s.rlo ? 1 : 0);
  }
  const int d = int(cout - lane_hi);
  // value added to the run's first limb: hi(lane) of the run below
  long long hin = __shfl_up_sync(0xffffffffu, lane_hi, 1);
  if (lane == 31) s_lanehi[warp] = lane_hi;
  __syncthreads();
  if (lane == 0) {
    if (warp > 0) {
      hin = s_lanehi[warp - 1];
    } else {
      hin = 0;
      if (ms > 0) {
        unsigned long long l0 = 0;
        long long h0 = 0;
        uint32_t sh = uint32_t(khalo * int64_t(b) - 64 * (ms - 1));
        for (int i = 0; i < 8; ++i) {
          if (khalo + i < kblk) {
            add_shifted(l0, h0, s_halo[i], sh);
            sh += b;
          }
        }
        hin = h0;
      }
    }
  }
  // the run's transfer function: first limb, the wrapping limbs above, d
  uint32_t tf0 = kTfIdentity, f = kTfIdentity;
  unsigned long long x0 = 0;
  bool allones = true, allzero = true;
  const uint32_t nl = live ? uint32_t(min(int64_t(rl), a.ML - m0)) : 0u;  // limbs of the run below ML
  if (live) {
    const unsigned long long l0 = (unsigned long long)__double_as_longlong(slot[0]);
    const __int128 s0 = (__int128)l0 + (__int128)hin;
    tf0 = limb_tf(s0, flags);
    x0 = (unsigned long long)s0;
    unsigned long long ov = 0, av = ~0ull;
    for (uint32_t i = 1; i < rl; ++i) {
      const unsigned long long l = (unsigned long long)__double_as_longlong(slot[i]);
      ov |= l;
      av &= l;
    }
    allones = av == ~0ull;
    allzero = ov == 0;
    // F(c) = d + wrap(tf0(c))
    uint32_t enc = 0;
#pragma unroll
    for (int c = -1; c <= 1; ++c) {
      const int c1 = tf_apply(tf0, c);
      const int c2 = (c1 == 1 && allones) ? 1 : (c1 == -1 && allzero) ? -1 : 0;
      int o = d + c2;
      if (o < -1 || o > 1) {
        flags |= kFlagCarryRange;
        o = 0;
      }
      enc |= uint32_t(o + 1) << (8 * (c + 1));
    }
    f = enc;
  } else if (m0 < a.ML) {
    // a run above the coefficients: zero limbs (they pass the carries of the sign)
    for (uint32_t i = 0; i < rl; ++i) slot[i] = 0.0;
    const __int128 s0 = (__int128)hin;
    tf0 = limb_tf(s0, flags);
    x0 = (unsigned long long)s0;
    allones = false;
    allzero = true;
    uint32_t enc = 0;
#pragma unroll
    for (int c = -1; c <= 1; ++c) {
      const int c1 = tf_apply(tf0, c);
      const int c2 = (c1 == -1) ? -1 : 0;
      enc |= uint32_t(c2 + 1) << (8 * (c + 1));
    }
    f = enc;
  }
  uint32_t agg;
  const uint32_t ex = block_scan_tf(f, sw, &agg);
  // publish the aggregate (single pass) or leave it to k_carry_patch
  if (tid == 0) {
    if (!lb) {
      a.aggs[blk] = agg;
    } else if (blk != 0) {
      *(volatile unsigned long long*)(a.scan.state + blk) =
          (static_cast<unsigned long long>(gen) << 32) | (1ull << 30) | agg;
    }
  }
  // fix the run's limbs for a zero carry into the block; the carry-in is
  // added afterwards (single pass: below, once the look-back has it; two
  // kernels: by k_carry_patch)
  const bool haslimbs = m0 < a.ML;
  const uint32_t nlw = haslimbs ? uint32_t(min(int64_t(rl), a.ML - m0)) : 0u;  // limbs below ML
  (void)nl;
  const int cin0 = tf_apply(ex, 0);
  const bool top = haslimbs && a.ML - 1 < m0 + int64_t(rl);  // owns the top limb
  // what flows above the top limb for the carry cin into the run (the sign
  // of the recombined value)
  auto top_carry = [&](int cin) -> long long {
    const uint32_t lt = uint32_t(a.ML - 1 - m0);
    long long ct = (lt == rl - 1u) ? lane_hi + tf_apply(f, cin) : __double_as_longlong(slot[lt + 1]);
    if (ct < -1 || ct > 1) {
      flags |= kFlagCarryRange;
      ct = 0;
    }
    return ct;
  };
  if (haslimbs) {
    slot[0] = __longlong_as_double((long long)(x0 + (unsigned long long)(long long)cin0));
    int c = tf_apply(tf0, cin0);
    if (c != 0) {
      for (uint32_t i = 1; i < rl; ++i) {
        const unsigned long long l = (unsigned long long)__double_as_longlong(slot[i]);
        slot[i] = __longlong_as_double((long long)(l + (unsigned long long)(long long)c));
        if (c > 0 ? l != ~0ull : l != 0ull) {
          c = 0;
          break;
        }
      }
    }
    if (top && !lowm && !lb) {
      uint64_t* tail = hmode ? a.tbuf : reinterpret_cast<uint64_t*>(a.sbuf);
      tail[a.ML] = uint64_t(top_carry(cin0));
    }
  }
  flags |= ra.all_flags();
  {
    const double e = warp_max_nonneg(ra.max_err), m = warp_max_nonneg(ra.max_abs);
    if (lane == 0) s_red[warp] = make_double2(e, m);
  }
  if (tid == 0) {
    s_last = 0;
    if (a.lanes_cins && !lb) {
      __threadfence();
      s_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
    }
  }
  __syncthreads();
  // ---- coalesced stores of the block's limbs ----
  const int64_t OL = a.out_limbs;
  uint64_t* tail = hmode ? a.tbuf : reinterpret_cast<uint64_t*>(a.sbuf);
  const uint32_t nlb = uint32_t(me - ms);
  auto limb_at = [&](uint32_t ml) -> uint64_t {
    const uint32_t g = B ? ml / uint32_t(B ? B * RUN / 64 : 1) : fdiv(ml, a.fb);
    return uint64_t(__double_as_longlong(slots[size_t(g) * G::slot + (ml - g * rl)]));
  };
  auto store_limb = [&](int64_t m, uint64_t x) {
    if constexpr (hmode) {
      tail[m] = x;
    } else if (m < OL) {
      a.out[m] = (lowm && m == OL - 1 && (a.n & 63)) ? (x & ((1ull << (a.n & 63)) - 1)) : x;
    } else if (!lb) {
      tail[m] = x;
    }
  };
  uint32_t first = 0xffffffffu;
  for (uint32_t ml = tid; ml < nlb; ml += kRT) {
    const uint64_t x = limb_at(ml);
    store_limb(ms + ml, x);
    // two kernels, high: a carry-in changes no limb above the first one that
    // is neither 0 nor all ones
    if (hmode && x + 1 > 1 && first == 0xffffffffu) first = ml;
  }
  if (lb) {
    // ---- single pass: the block's carry-in, taken after the stores (the
    // blocks before have had that time to publish) ----
    if (warp == 0) {
      const int c = lookback_warp(a.scan.state, uint32_t(blk), agg, gen, 0, true);
      if (lane == 0) s_cin = c;
    }
    __syncthreads();
    const int cin_blk = s_cin;
    const int cin = tf_apply(ex, cin_blk);
    if (haslimbs && cin != cin0) {
      // add the difference to the run's limbs up to the first that does not
      // wrap, and store those again (the next run's carry-in already counts
      // a carry through this one)
      int dl = cin - cin0;
      for (uint32_t i = 0; i < nlw && dl != 0; ++i) {
        const unsigned long long l = (unsigned long long)__double_as_longlong(slot[i]);
        const unsigned long long x = l + (unsigned long long)(long long)dl;
        slot[i] = __longlong_as_double((long long)x);
        store_limb(m0 + i, x);
        dl = dl > 0 ? (x < l ? 1 : 0) : (x > l ? -1 : 0);
      }
    }
    if (top && !lowm) {
      // (reads the limb above the top one: after this thread's own patch)
      if (top_carry(cin) < 0) flags |= fullm ? uint32_t(kFlagNegative) : uint32_t(kFlagHighRange);
    }
    // the checks on final limbs: the full product's range, the high
    // product's nominations and sticky bits (below)
    if (fullm && me > OL - 1) {
      __syncthreads();
      const int hb = int((2 * a.n) & 63);
      for (uint32_t ml = tid; ml < nlb; ml += kRT) {
        const int64_t m = ms + ml;
        if (m >= OL - 1) {
          const uint64_t x = limb_at(ml);
          if (m == OL - 1 ? (hb && (x >> hb)) : x != 0) flags |= kFlagFullOverflow;
        }
      }
    }
  }
  if (flags) atomicOr(&s_flags, flags);
  if constexpr (hmode) {
    if (!lb) {
      first = __reduce_min_sync(0xffffffffu, first);
      if (lane == 0 && first != 0xffffffffu) atomicMin(&s_first, first);
    }
    __syncthreads();
    // nominations and sticky bits: single pass, of every limb; two kernels,
    // of the limbs no carry-in can change (all of block 0's, which has
    // none), k_carry_patch sees the others
    const HighLimbs3 hl(a);
    const uint32_t lfix = (blk == 0 || lb) ? 0u : (s_first == 0xffffffffu ? 0xffffffffu : s_first + 1u);
    uint32_t hmin = 0xffffffffu, sticky = 0;
    // single pass: a block above the sticky bits whose lowest possible
    // nomination (limb ms - hq - 1 of t >> s) cannot lower the one already
    // made by a block below it has nothing to add
    bool skip = false;
    if (lb && ms - hl.hq - 1 > 0 && 64 * ms >= hl.sb)
      skip = __ldcg(a.hstop) <= uint32_t(ms - hl.hq - 1);
    if (!skip) {
      for (uint32_t ml = tid; ml < nlb; ml += kRT) {
        if (ml >= lfix) hl.see(ms + ml, limb_at(ml), hmin, sticky);
      }
    }
    // w0's top limb has zero fill above bit 64 - r: never all ones
    if (hl.hr != 0 && blk == 0 && tid == 0 && hl.WL > 0) hmin = min(hmin, uint32_t(hl.WL - 1));
    hmin = __reduce_min_sync(0xffffffffu, hmin);
    sticky = __reduce_or_sync(0xffffffffu, sticky);
    if (lane == 0) {
      if (hmin != 0xffffffffu) atomicMin(&s_hmin, hmin);
      if (sticky) s_sticky = 1;
    }
  }
  __syncthreads();
  if (hmode && tid == 0) {
    if (s_hmin != 0xffffffffu) atomicMin(a.hstop, s_hmin);
    if (s_sticky) atomicOr(&a.status->high_sticky, 1u);
  }
  if (tid == 0) {
    double e = 0.0, m = 0.0;
#pragma unroll
    for (int w = 0; w < kRT / 32; ++w) {
      e = fmax(e, s_red[w].x);
      m = fmax(m, s_red[w].y);
    }
    status_merge(a.status, e, m, s_flags);
  }
  if (s_last) {
    // the last block to finish turns the per-block functions into each
    // block's carry-in (as k_carry_lanes)
    __threadfence();
    const uint32_t B = gridDim.x;
    const uint32_t Q = (B + kRT - 1) / kRT;
    const uint32_t i0 = uint32_t(tid) * Q, i1 = min(B, i0 + Q);
    uint32_t g = kTfIdentity;
    for (uint32_t i = i0; i < i1; ++i) g = tf_compose(g, __ldcg(a.aggs + i));
    uint32_t tot;
    uint32_t exb = block_scan_tf(g, sw, &tot);
    for (uint32_t i = i0; i < i1; ++i) {
      a.cins[i] = tf_apply(exb, 0);
      exb = tf_compose(exb, __ldcg(a.aggs + i));
    }
    if (tid == 0) *a.ticket = 0;
  }
}

template <int MODE>
CarryLanesFn runs_mode(int lam, int b) {
  // compiled chunk widths: what select_params picks from 2^22 to 2^30 bits
  if (lam == 4 && b == 13) return k_carry_runs<MODE, 4, 13>;
  if (lam == 5 && b == 12) return k_carry_runs<MODE, 5, 12, 32>;
  if (lam == 5 && b == 11) return k_carry_runs<MODE, 5, 11>;
  switch (lam) {
    case 3: return k_carry_runs<MODE, 3, 0>;
    case 4: return k_carry_runs<MODE, 4, 0>;
    case 5: return k_carry_runs<MODE, 5, 0>;
    case 6: return k_carry_runs<MODE, 6, 0>;
    default: return nullptr;
  }
}

template <int MODE>
size_t runs_smem_mode(int lam) {
  switch (lam) {
    case 3: return size_t(kRT) * RunGeom<MODE, 3>::slot * 8;
    case 4: return size_t(kRT) * RunGeom<MODE, 4>::slot * 8;
    case 5: return size_t(kRT) * RunGeom<MODE, 5>::slot * 8;
    case 6: return size_t(kRT) * RunGeom<MODE, 6>::slot * 8;
    default: return 0;
  }
}

}  // namespace

CarryLanesFn carry_runs_kernel(int mode, int lam, int b, bool compiled_b) {
  if (!compiled_b) b = 0;
  if (mode == kModeFull) {
    switch (b) {
      case 18: return k_carry_runs<kModeFull, 0, 18>;
      case 19: return k_carry_runs<kModeFull, 0, 19>;
      case 20: return k_carry_runs<kModeFull, 0, 20>;
      default: return k_carry_runs<kModeFull, 0, 0>;
    }
  }
  return mode == kModeLow ? runs_mode<kModeLow>(lam, b) : runs_mode<kModeHigh>(lam, b);
}

// coefficients per run of the kernel carry_runs_kernel returns
int carry_runs_len(int mode, int lam, int b, bool compiled_b) {
  return (compiled_b && mode != kModeFull && lam == 5 && b == 12) ? 32 : 64;
}

size_t carry_runs_smem(int mode, int lam, int run) {
  if (run == 32) {
    return size_t(kRT) * (mode == kModeLow ? RunGeom<kModeLow, 5, 32>::slot : RunGeom<kModeHigh, 5, 32>::slot) * 8;
  }
  if (mode == kModeFull) return size_t(kRT) * RunGeom<kModeFull, 0>::slot * 8;
  return mode == kModeLow ? runs_smem_mode<kModeLow>(lam) : runs_smem_mode<kModeHigh>(lam);
}

}  // namespace tmg
