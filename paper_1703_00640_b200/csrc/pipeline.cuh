// Pieces of the product pipeline shared by the fused single-CTA kernel and
// the multi-pass kernels: pre-map, post-map, rounding with the reference's
// tripwire, recombination lanes and carry transfer functions.
#pragma once

#include "common.cuh"
#include "digits.cuh"

namespace tmg {

enum Mode : int32_t { kModeFull = 0, kModeLow = 1, kModeHigh = 2 };

// ----------------------------------------------------------------------------
// Pre-map (alpha* for low, gamma+ for high) at transform index j < N.
// D(i) returns the balanced digit of chunk i (0 <= i < N); top is chunk N of
// the high split.  Mirrors apply_series (maps_f64.cpp:48-96) plus the
// gamma-dagger fold of the top coefficient (maps_f64.cpp:337-347).
template <class DF>
__device__ __forceinline__ double premap(const MapConsts& mc, const DF& D,
                                         int64_t j, double top) {
  const int64_t N = mc.N;
  const double Nd = double(N);
  const int fam = (mc.mode == kModeLow) ? 0 : 2;
  const int lam = mc.lambda;
  double acc = 0.0;
  RowLoopDown<kMaxLambda>::run([&](auto rc) {
    constexpr int r = decltype(rc)::value;
    if (r < lam) {
      int64_t k = j - r;
      if (k < 0) k += N;
      acc += D(k) * coef_r<r>(fam, double(k), Nd, mc.cpre[r]);
    }
  });
  if (mc.mode == kModeHigh && top != 0.0 && j < mc.nfold + lam) {
    // out[(k + r) mod N] += top * fold[k] * gamma_r(k), k < nfold
    RowLoop<kMaxLambda>::run([&](auto rc) {
      constexpr int r = decltype(rc)::value;
      if (r < lam) {
        int64_t k = j - r;
        if (k < 0) k += N;
        if (k < mc.nfold) acc += top * mc.fold[k] * coef_r<r>(2, double(k), Nd, mc.cpre[r]);
      }
    });
  }
  return acc;
}

// premap of both operands at once (D2(i) = (digit of u, digit of v)): the
// series coefficients are computed once for the pair.  Same values as two
// premap calls (a fold term with top = 0 adds an exact zero).
template <class DF2>
__device__ __forceinline__ double2 premap2(const MapConsts& mc, const DF2& D2, int64_t j,
                                           double topu, double topv) {
  const int64_t N = mc.N;
  const double Nd = double(N);
  const int fam = (mc.mode == kModeLow) ? 0 : 2;
  const int lam = mc.lambda;
  // k = j - r (+ N) as an exact double from one conversion of j
  const double jd = double(j);
  double au = 0.0, av = 0.0;
  RowLoopDown<kMaxLambda>::run([&](auto rc) {
    constexpr int r = decltype(rc)::value;
    if (r < lam) {
      int64_t k = j - r;
      const bool wrap = k < 0;
      if (wrap) k += N;
      const double cf = coef_r<r>(fam, jd - double(r) + (wrap ? Nd : 0.0), Nd, mc.cpre[r]);
      const double2 d = D2(k);
      au += d.x * cf;
      av += d.y * cf;
    }
  });
  if (mc.mode == kModeHigh && j < mc.nfold + lam) {
    RowLoop<kMaxLambda>::run([&](auto rc) {
      constexpr int r = decltype(rc)::value;
      if (r < lam) {
        int64_t k = j - r;
        if (k < 0) k += N;
        if (k < mc.nfold) {
          const double g = mc.fold[k] * coef_r<r>(2, double(k), Nd, mc.cpre[r]);
          if (topu != 0.0) au += topu * g;
          if (topv != 0.0) av += topv * g;
        }
      }
    });
  }
  return make_double2(au, av);
}

// Root-channel value of a high-split operand (maps_f64.cpp:319-328):
// theta = sum_d in[N - d] * inv_root^d over the first nroot terms.
template <class DF>
__device__ __forceinline__ double root_channel(const MapConsts& mc,
                                               const DF& D, double top) {
  double acc = 0.0;
  for (int d = 0; d < mc.nroot && d <= mc.N; ++d) {
    double x = (d == 0) ? top : D(mc.N - d);
    acc += x * mc.ipow[d];
  }
  return acc;
}

// ----------------------------------------------------------------------------
// Post-map.  W(j) returns convolution coefficient j (0 <= j < N).
// flat(j) = sum_r W(j - r) * post_r(j - r) for the r keeping j - r in [0, N)
// (apply_series_flat, maps_f64.cpp:175-187).
template <class WF>
__device__ __forceinline__ double post_flat(const MapConsts& mc, const WF& W,
                                            int64_t j) {
  const int64_t N = mc.N;
  const double Nd = double(N);
  const int fam = (mc.mode == kModeLow) ? 1 : 3;
  const int lam = mc.lambda;
  const double jd = double(j);  // k = j - r as an exact double, one conversion
  double acc = 0.0;
  RowLoopDown<kMaxLambda>::run([&](auto rc) {
    constexpr int r = decltype(rc)::value;
    const int64_t k = j - r;
    if (r < lam && k >= 0 && k < N) acc += W(k) * coef_r<r>(fam, jd - double(r), Nd, mc.cpost[r]);
  });
  return acc;
}

// beta* value at index i < N (beta_star_view_f64, maps_f64.cpp:269-281),
// returned pre-multiplied by 2^b.
template <class WF>
__device__ __forceinline__ double postmap_low(const MapConsts& mc, const WF& W,
                                              int64_t i) {
  const int64_t N = mc.N;
  double v = post_flat(mc, W, i);
  if (i <= mc.lambda - 2) v += post_flat(mc, W, i + N);
  if (i >= 1 && i <= mc.lambda - 1) v -= post_flat(mc, W, i + N - 1) * mc.step;
  return v * mc.scale_out;
}

// Folded buffer of delta-dagger before differencing (maps_f64.cpp:355-362).
template <class WF>
__device__ __forceinline__ double high_buf(const MapConsts& mc, const WF& W,
                                           int64_t i) {
  const int64_t N = mc.N;
  double v = post_flat(mc, W, i);
  for (int64_t j = N + mc.lambda - 2; j >= N; --j) {
    int64_t o = i - (j - N);
    if (o >= 0 && o < mc.nfold) v += post_flat(mc, W, j) * mc.fold[o];
  }
  return v;
}

// psi of delta-dagger (maps_f64.cpp:363-371); aux = theta_u * theta_v.
template <class WF>
__device__ __forceinline__ double high_psi(const MapConsts& mc, const WF& W,
                                           double aux) {
  double hrho = 0.0;
  for (int d = 1; d <= mc.nhrho && d <= mc.N; ++d)
    hrho += high_buf(mc, W, mc.N - d) * mc.ipow[d];
  return (aux - hrho * mc.root_neg_n) / mc.cofactor_scaled;
}

// delta-dagger value at i in [0, N], pre-multiplied by 2^b
// (maps_f64.cpp:372-383).
template <class WF>
__device__ __forceinline__ double postmap_high(const MapConsts& mc,
                                               const WF& W, int64_t i,
                                               double psi) {
  const int64_t N = mc.N;
  double v;
  if (i == N) {
    v = psi - high_buf(mc, W, N - 1) * mc.step;
  } else if (i == 0) {
    v = high_buf(mc, W, 0);
  } else {
    v = high_buf(mc, W, i) - high_buf(mc, W, i - 1) * mc.step;
  }
  if (i < mc.nfold) v -= psi * mc.fold[i];
  return v * mc.scale_out;
}

// ----------------------------------------------------------------------------
// Rounding with the reference tripwire (products_f64.cpp:16-27): a value is
// refused when |x| >= 2^53 (or NaN) or when it sits farther than a quarter
// from the nearest integer.  Returns the rounded integer.
struct RoundAcc {
  double max_err = 0.0;
  double max_abs = 0.0;
  uint32_t flags = 0;
  __device__ __forceinline__ long long round(double x) {
    double ax = fabs(x);
    if (ax < 2251799813685248.0) {
      // |x| < 2^51: adding 1.5 * 2^52 rounds x to the nearest integer (ties
      // to even, as rint) and leaves it in the low mantissa bits -- no
      // FRND / F2I on the quarter-rate conversion path
      const double t = x + 6755399441055744.0;
      const double r = t - 6755399441055744.0;
      const double e = fabs(x - r);
      max_err = fmax(max_err, e);
      max_abs = fmax(max_abs, ax);
      return __double_as_longlong(t) - 0x4338000000000000ll;
    }
    return round_wide(x, ax);
  }
  // The accumulated flags: the residual tripwire (products_f64.cpp:22) is
  // settled once from the running maximum instead of per coefficient.
  __device__ __forceinline__ uint32_t all_flags() const {
    return flags | (max_err > 0.25 ? uint32_t(kFlagTripwire) : 0u);
  }
  __device__ __forceinline__ long long round_wide(double x, double ax) {
    if (!(ax < 9007199254740992.0)) {
      flags |= kFlagOverflow;
      max_abs = fmax(max_abs, isnan(ax) ? 1e308 : ax);
      return 0;
    }
    double r = rint(x);
    double e = fabs(x - r);
    max_err = fmax(max_err, e);
    max_abs = fmax(max_abs, ax);
    if (e > 0.25) flags |= kFlagTripwire;
    return (long long)r;
  }
};

// Warp maximum of a non-negative double, exact, with two REDUX: the high
// words first, then the low words of the lanes that hold the maximal high word.
__device__ __forceinline__ double warp_max_nonneg(double x) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
  const uint32_t hi = uint32_t(b >> 32), lo = uint32_t(b);
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  return __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
}

__device__ __forceinline__ void status_merge(DevStatus* st, double max_err,
                                             double max_abs, uint32_t flags) {
  atomicMax(&st->max_err_bits, (unsigned long long)__double_as_longlong(max_err));
  atomicMax(&st->max_abs_bits, (unsigned long long)__double_as_longlong(max_abs));
  if (flags) atomicOr(&st->flags, flags);
}

// ----------------------------------------------------------------------------
// Recombination lanes.  Value V = sum_k e_k 2^{k b}; lane m collects the e_k
// whose bit offset falls in limb m: lane_m = sum e_k << (k b - 64 m), a
// signed 128-bit quantity (SignedAccumulator, products_f64.cpp:36-66).
template <class EF>
__device__ __forceinline__ __int128 lane_value(const EF& E, int64_t m, int b,
                                               int64_t K) {
  if (m < 0) return 0;
  int64_t klo = (64 * m + b - 1) / b;
  int64_t khi = (64 * m + 64 + b - 1) / b;  // exclusive
  if (khi > K) khi = K;
  __int128 acc = 0;
  for (int64_t k = klo; k < khi; ++k) {
    int sh = int(k * b - 64 * m);
    acc += (__int128)E(k) << sh;
  }
  return acc;
}

// Transfer function of limb m with s = lo(lane_m) + hi(lane_{m-1}).
// f(c) = floor((s + c) / 2^64) for c in {-1, 0, 1}.
__device__ __forceinline__ uint32_t limb_tf(__int128 s, uint32_t& flags) {
  long long hi = (long long)(s >> 64);
  unsigned long long lo = (unsigned long long)s;
  int fm = int(hi) - (lo == 0 ? 1 : 0);
  int f0 = int(hi);
  int fp = int(hi) + (lo == ~0ull ? 1 : 0);
  if (hi < -1 || hi > 1 || fm < -1 || fp > 1) {
    flags |= kFlagCarryRange;
    fm = f0 = fp = 0;
  }
  return uint32_t(fm + 1) | (uint32_t(f0 + 1) << 8) | (uint32_t(fp + 1) << 16);
}

// High product range bookkeeping (products_f64.cpp:167-169): w must lie in
// [0, 2^n].  Limb m of w is split into the bits below n, bit n, and above n.
__device__ __forceinline__ void high_classify(uint64_t x, int64_t m, int64_t n,
                                              uint32_t& topbit,
                                              uint32_t& lownz,
                                              uint32_t& flags) {
  const int64_t bit0 = 64 * m;
  uint64_t below = 0, atn = 0, above = 0;
  if (bit0 + 64 <= n) {
    below = x;
  } else if (bit0 > n) {
    above = x;
  } else {
    const int o = int(n - bit0);  // 0..63
    below = o ? (x & ((1ull << o) - 1)) : 0;
    atn = (x >> o) & 1ull;
    above = (o == 63) ? 0 : (x >> (o + 1));
  }
  if (below) lownz = 1;
  if (atn) topbit = 1;
  if (above) flags |= kFlagHighRange;
}
__device__ __forceinline__ uint64_t high_mask(int64_t m, int64_t OL,
                                              int64_t n) {
  if (m != OL - 1) return ~0ull;
  const int r = int((n + 1) & 63);
  return r ? ((1ull << r) - 1) : ~0ull;
}

// ----------------------------------------------------------------------------
// Block-wide exclusive scan of transfer functions (blockDim % 32 == 0).
// Returns the exclusive prefix of this thread; *agg gets the block total.
__device__ __forceinline__ uint32_t block_scan_tf(uint32_t f, uint32_t* sw,
                                                  uint32_t* agg) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  uint32_t inc = f;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    uint32_t o = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc = tf_compose(o, inc);
  }
  uint32_t excl = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) excl = kTfIdentity;
  __syncthreads();
  if (lane == 31) sw[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t v = lane < nw ? sw[lane] : kTfIdentity;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      uint32_t o = __shfl_up_sync(0xffffffffu, v, off);
      if (lane >= off) v = tf_compose(o, v);
    }
    sw[lane] = v;
  }
  __syncthreads();
  uint32_t wex = warp > 0 ? sw[warp - 1] : kTfIdentity;
  *agg = sw[nw - 1];
  __syncthreads();
  return tf_compose(wex, excl);
}

// ----------------------------------------------------------------------------
// Kill / generate / propagate codes of the balanced split's carry chains
// (carries are 0 or 1 there): 0 = K (carry out 0), 1 = G (carry out 1),
// 2 = P (carry out = carry in); two operands packed in bits [0,2) and [2,4).
// Composition "f then g" keeps g unless g propagates; applying f to carries
// c (codes 0 / 1 per operand) is kgp_compose(c, f).
constexpr uint32_t kKgpIdentity = 2u | (2u << 2);
__device__ __forceinline__ uint32_t kgp_compose(uint32_t f, uint32_t g) {
  const uint32_t pm = (g >> 1) & ~g & 0x5u;  // fields of g equal to P (binary 10)
  const uint32_t M = pm | (pm << 1);
  return (g & ~M) | (f & M);
}

__device__ __forceinline__ uint32_t block_scan_kgp(uint32_t f, uint32_t* sw, uint32_t* agg) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  uint32_t inc = f;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc = kgp_compose(o, inc);
  }
  uint32_t excl = __shfl_up_sync(0xffffffffu, inc, 1);
  if (lane == 0) excl = kKgpIdentity;
  __syncthreads();
  if (lane == 31) sw[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t v = lane < nw ? sw[lane] : kKgpIdentity;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, v, off);
      if (lane >= off) v = kgp_compose(o, v);
    }
    sw[lane] = v;
  }
  __syncthreads();
  const uint32_t wex = warp > 0 ? sw[warp - 1] : kKgpIdentity;
  *agg = sw[nw - 1];
  __syncthreads();
  return kgp_compose(wex, excl);
}

// Warp-parallel decoupled look-back (called by all 32 lanes of one warp):
// each round reads the state words of the 32 nearest unresolved
// predecessors at once, composes their aggregates with a warp reduction and
// stops at the nearest inclusive prefix or constant aggregate.  carry0 is the carry into block 0.
// Returns the carry into block blk (same value in every lane) and publishes
// this block's inclusive carry.
__device__ __forceinline__ int lookback_warp(unsigned long long* state,
                                             uint32_t blk, uint32_t agg,
                                             uint32_t epoch, int carry0,
                                             bool published = false) {
  const int lane = threadIdx.x & 31;
  const unsigned long long ep = (unsigned long long)epoch << 32;
  int carry_in = carry0;
  if (blk != 0) {
    if (lane == 0 && !published)
      *(volatile unsigned long long*)(state + blk) = ep | (1ull << 30) | agg;
    uint32_t E = kTfIdentity;
    int64_t base = int64_t(blk) - 1;
    while (true) {
      const int64_t j = base - lane;
      unsigned long long w = 0;
      if (j >= 0) w = *(volatile unsigned long long*)(state + j);
      const bool valid = (j >= 0) && ((w >> 32) == epoch) && (((w >> 30) & 3u) != 0);
      // the walk stops at an inclusive prefix or at an aggregate that is a
      // constant function (its carry-out does not depend on its carry-in --
      // almost every block's), so it rarely goes past the nearest predecessor
      const uint32_t wf = uint32_t(w & 0xFFFFFFu);
      const bool cst = valid && (((w >> 30) & 3u) == 1) && ((wf & 0xFFu) == ((wf >> 8) & 0xFFu)) &&
                       ((wf & 0xFFu) == (wf >> 16));
      const bool incl = valid && ((((w >> 30) & 3u) == 2) || cst);
      if (cst) w = (w & ~0xFFFFFFull) | (wf & 0xFFu);  // its carry-out + 1, like an inclusive word
      const uint32_t bi = __ballot_sync(0xffffffffu, incl);
      const uint32_t bv = __ballot_sync(0xffffffffu, valid);
      const int first = bi ? (__ffs(bi) - 1) : 32;
      const uint32_t need = (first == 32) ? 0xffffffffu : ((1u << first) - 1u);
      if ((bv & need) != need) continue;  // a nearer predecessor is not ready
      // compose aggregates of lanes [0, first): f_0 o f_1 o ... o f_{first-1}
      uint32_t f = (lane < first) ? uint32_t(w & 0xFFFFFFu) : kTfIdentity;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_down_sync(0xffffffffu, f, off);
        if (lane + off < 32) f = tf_compose(o, f);
      }
      f = __shfl_sync(0xffffffffu, f, 0);
      E = tf_compose(f, E);
      if (first < 32) {
        const int v = int(__shfl_sync(0xffffffffu, uint32_t(w & 0xFFFFFFu), first)) - 1;
        carry_in = tf_apply(E, v);
        break;
      }
      base -= 32;
    }
  }
  if (lane == 0) {
    const int out = tf_apply(agg, carry_in);
    *(volatile unsigned long long*)(state + blk) = ep | (2ull << 30) | uint64_t(out + 1);
  }
  return carry_in;
}

}  // namespace tmg
