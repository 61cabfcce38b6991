// Post-map, rounding and carry propagation as two kernels without
// inter-block waiting.
//
//   k_carry_lanes  every block owns 256 x PT consecutive limbs (PT = 2 or 4
//                  by the window size) and the coefficients whose bit
//                  offsets k b land in them.  The block post-maps them (beta*
//                  low, delta+ high; nothing for the full product) and rounds
//                  them with the reference's tripwire, one coefficient per
//                  thread and pass; each thread then forms the signed 128-bit
//                  lanes lane_m = sum e_k << (k b - 64 m) of its PT limbs and
//                  the limb sums s_m = lo(lane_m) + hi(lane_{m-1}).  A block
//                  scan of the limbs' carry transfer functions gives every
//                  limb for a zero carry into the block, written to the
//                  output (high: to t); the block's composed function goes
//                  to aggs[blk].
//   k_carry_patch  one warp per block: the block's carry-in (the composition
//                  of the preceding blocks' functions) is added to its first
//                  limbs, up to the first that does not wrap (usually one
//                  limb), then the range checks and the high product's
//                  stopping-limb nominations that read those limbs.
//
// Compared with the single-pass look-back kernel (k_carry), no block ever
// waits on another: the lanes kernel runs at full occupancy and its
// aggregate is final when it is written.
//
// The post-map runs in gather form with the operation order of post_flat:
// output j sums its rows r = lambda-1 .. 0 with the same fused
// multiply-adds, so the values are bit-identical to the generic path.  The
// few outputs that also see the wrap of the cyclic maps (low: j <= lambda - 1;
// high: i below the fold, k = N) go through the generic helpers.
//
// Reference: products_f64.cpp:29-102 (SignedAccumulator, round_accumulate),
// maps_f64.cpp:140-188, 269-281, 350-384 (beta*, delta+).
#include "kernels.cuh"

namespace tmg {

namespace {

constexpr int kT = kC2Threads;

// First coefficient of lane m, ceil(64 m / b), clamped to K.  The host
// takes this path only when every bit offset fits in 32 bits
// (64 ML + 64 < 2^32), so a 32-bit reciprocal division (FastDiv) replaces
// the 64-bit one.
__device__ __forceinline__ int64_t kfirst(int64_t m, const FastDiv& fb, int64_t K) {
  const uint32_t num = uint32_t(64 * m) + fb.d - 1u;
  const int64_t k = int64_t(fdiv(num, fb));
  return k < K ? k : K;
}

// acc += e << sh for 0 <= sh < 64 on a signed 128-bit (lo, hi) pair.
__device__ __forceinline__ void add_shifted(unsigned long long& lo, long long& hi, long long e,
                                            uint32_t sh) {
  const unsigned long long l = (unsigned long long)e << sh;
  const long long h = (e >> 1) >> (63 - sh);  // arithmetic; sh = 0 gives the sign word
  const unsigned long long nlo = lo + l;
  hi += h + (nlo < lo ? 1 : 0);
  lo = nlo;
}

// Lane m = sum_{k in lane m} e_k << (k b - 64 m) from se[k - kbase].
__device__ __forceinline__ void lane_of(const long long* __restrict__ se, int64_t kbase,
                                        int64_t m, int64_t ka, int64_t kb, int b,
                                        unsigned long long& lo, long long& hi) {
  lo = 0;
  hi = 0;
  const int n = int(kb - ka);
  const long long* p = se + (ka - kbase);
  uint32_t sh = uint32_t(ka) * uint32_t(b) - 64u * uint32_t(m);  // < 64 (mod 2^32 exact)
  if (n <= 8) {
    // at most ceil(64 / b) + 1 terms: unrolled and predicated (b >= 9)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i < n) add_shifted(lo, hi, p[i], sh + uint32_t(i * b));
    }
  } else {
    for (int i = 0; i < n; ++i) {
      add_shifted(lo, hi, p[i], sh);
      sh += uint32_t(b);
    }
  }
}

// Rounded coefficients e_k, k in [kbase, kend), of the whole block into
// se[k - kbase]: one coefficient per thread and pass (gather form), so the
// work is spread evenly over the block.  Output j of the flat post-map sums
// its rows as acc = fma(w_{j-r}, P_r(j-r) c_r, acc) for r = lambda-1 .. 1 and
// adds w_j last (post_flat's order, bit-identical values).  The high product's differencing
// x_k = hbuf(k) - hbuf(k-1) step reads hbuf from shared memory (shb), written
// in a first pass.  The wrap outputs go through the generic helpers as before.
template <int LAM>
__device__ __forceinline__ void coeffs_block(const CarryArgs& a, const double* __restrict__ sww,
                                             int64_t wlo, int64_t nw, int64_t kbase,
                                             int64_t kend, long long* __restrict__ se,
                                             double* __restrict__ shb, RoundAcc& ra, double psi,
                                             uint32_t& flags, int tid) {
  const MapConsts& mc = a.mc;
  auto WS = [&](int64_t j) -> double {
    const int64_t o = j - wlo;
    return (o >= 0 && o < nw) ? sww[o] : __ldg(a.w + j);
  };
  if constexpr (LAM == 0) {
    // no post-map: each coefficient is read once, straight from global
    // memory (four loads in flight per thread)
    const double* wk = a.w + kbase;
    const int32_t nk = int32_t(kend - kbase);
    int32_t q = tid;
    for (; q + 3 * kT < nk; q += 4 * kT) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(wk + q + u * kT);
#pragma unroll
      for (int u = 0; u < 4; ++u) se[q + u * kT] = ra.round(v[u]);
    }
    for (; q < nk; q += kT) se[q] = ra.round(__ldg(wk + q));
  } else {
    // Blocks whose post-map inputs all lie in [0, N) away from the wrap
    // outputs (block-uniform) take the same arithmetic without bound checks,
    // 32-bit indices and exact FP64 index conversions.
    const int64_t N0 = mc.N;
    const int64_t hs0 = int64_t(mc.nfold) + LAM - 2;
    const bool lowm = mc.mode == kModeLow;
    const bool interior = kbase >= LAM + 1 && kend + 1 <= N0 && kend - wlo < (int64_t(1) << 31) &&
                          (lowm || kbase - 1 >= hs0);
    if (interior) {
      const double st = lowm ? double(N0) : -double(N0);
      const double step = mc.step, sc = mc.scale_out;
      double cr[LAM];
#pragma unroll
      for (int r = 0; r < LAM; ++r) cr[r] = mc.cpost[r];
      const double* wb = sww - wlo;  // wb[i] = w_i inside the window
      const uint32_t kb32 = uint32_t(kbase);
      auto pfd = [&](uint32_t j) -> double {
        const double jd = __hiloint2double(0x43300000, int(j)) - 4503599627370496.0;
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
          acc = fma(wb[j - r], p * cr[r], acc);
        }
        return acc + wb[j];
      };
      const uint32_t nk = uint32_t(kend - kbase);
      if (lowm) {
        for (uint32_t q = tid; q < nk; q += kT) se[q] = ra.round(pfd(kb32 + q + 1) * sc);
      } else {
        for (uint32_t q = tid; q < nk + 1; q += kT) shb[q] = pfd(kb32 + q - 1);
        __syncthreads();
        for (uint32_t q = tid; q < nk; q += kT) se[q] = ra.round((shb[q + 1] - shb[q] * step) * sc);
      }
      return;
    }
    const int b = mc.b;
    const int64_t N = mc.N;
    const bool low = mc.mode == kModeLow;
    const double Nd = double(N);
    const double st = low ? Nd : -Nd;  // beta: k + i N, delta: k - i N
    const double step = mc.step, sc = mc.scale_out;
    double cr[LAM];
#pragma unroll
    for (int r = 0; r < LAM; ++r) cr[r] = mc.cpost[r];
    // flat post-map output j (inputs outside [0, N) contribute nothing)
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
          acc = fma(sww[i - wlo], p * cr[r], acc);
        }
      }
      if (j >= 0 && j < N) acc = acc + sww[j - wlo];
      return acc;
    };
    if (low) {
      for (int64_t k = kbase + tid; k < kend; k += kT) {
        const int64_t i = k + 1;
        const double x = (i <= LAM - 1) ? postmap_low(mc, WS, i) : pf(i) * sc;
        long long e = ra.round(x);
        if (k == 0) {
          const long long c0v = ra.round(postmap_low(mc, WS, 0));
          if (c0v & ((1ll << b) - 1)) flags |= kFlagLowNotDivisible;
          e += (c0v >> b);
        }
        se[k - kbase] = e;
      }
    } else {
      const int64_t hslow = int64_t(mc.nfold) + LAM - 2;  // hbuf(i) = post_flat(i) from here on
      // shb[i - kbase + 1] = hbuf(i) for i in [kbase - 1, kend), zero outside [0, N)
      for (int64_t i = kbase - 1 + tid; i < kend; i += kT) {
        double hb = 0.0;
        if (i >= 0 && i < N) hb = (i < hslow) ? high_buf(mc, WS, i) : pf(i);
        shb[i - kbase + 1] = hb;
      }
      __syncthreads();
      for (int64_t k = kbase + tid; k < kend; k += kT) {
        const double hp = shb[k - kbase];
        double v = (k == N) ? psi - hp * step : shb[k - kbase + 1] - hp * step;
        if (k < mc.nfold) v -= psi * mc.fold[k];
        se[k - kbase] = ra.round(v * sc);
      }
    }
  }
}

// High product: limb m of t feeds w0_{m-q} (bits r..63) and w0_{m-q-1}
// (bits 0..r-1) of w0 = t >> s, q = s / 64, r = s % 64; a limb nominates the
// w0 limbs its bits prove not all ones (the first such limb stops the
// rounding increment of k_high_round), and the limbs below bit s - 1 feed
// the sticky bit.
struct HighLimbs {
  int64_t hq, WL, sb;
  int hr;
  __device__ explicit HighLimbs(const CarryArgs& a)
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

template <int LAM, int kPT>
__global__ void __launch_bounds__(kT, 4) k_carry_lanes(CarryArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int64_t kLimbs = int64_t(kT) * kPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t sw[32];
  __shared__ long long s_hi[kT];
  __shared__ double s_psi;
  __shared__ uint32_t s_flags;
  __shared__ double2 s_red[kT / 32];
  const int tid = threadIdx.x;
  const MapConsts& mc = a.mc;
  const int b = mc.b;
  const int64_t K = a.K;
  const int64_t blk = blockIdx.x;
  const int64_t ms = blk * kLimbs;
  const int64_t me = min(a.ML, ms + kLimbs);
  const int64_t kbase = kfirst(ms > 0 ? ms - 1 : 0, a.fb, K);
  const int64_t kend = kfirst(me, a.fb, K);
  // staged convolution window (post-map neighbourhood: lambda below, one above)
  // (16-byte aligned ends for the bulk copy; w holds L >= nwt + 1 values
  // when nwt is odd, since L is even)
  const int64_t nwt = (mc.mode == kModeFull) ? K : mc.N;
  const int64_t wlo = max(int64_t(0), kbase - LAM - 1) & ~int64_t(1);
  const int64_t whi = (min(nwt, kend + 2) + 1) & ~int64_t(1);
  // (the full product reads its coefficients once: no window)
  const int64_t nw = (LAM > 0 && whi > wlo) ? whi - wlo : 0;
  double* sww = reinterpret_cast<double*>(smem_raw);
  // the high product's folded buffer hbuf takes the slot after the staged
  // window, and its rounded coefficients overwrite the window, which is dead
  // once hbuf is formed (coeffs_block separates the two by a barrier): no
  // shared memory beyond the low product's
  const bool hmode = mc.mode == kModeHigh;
  long long* se = hmode ? reinterpret_cast<long long*>(sww)
                        : reinterpret_cast<long long*>(sww + (nw + 1));
  // the window arrives by one bulk copy (TMA engine) on an mbarrier, issued
  // before the block's set-up so the two overlap
  __shared__ __align__(8) uint64_t s_mbar;
  if (tid == 0 && nw > 0) {
    mbar_init(&s_mbar, 1);
    mbar_expect_tx(&s_mbar, uint32_t(nw * 8));
    bulk_g2s(sww, a.w + wlo, uint32_t(nw * 8), &s_mbar);
  }
  __shared__ uint32_t s_first, s_hmin, s_sticky;
  if (tid == 0) {
    s_flags = 0;
    s_first = 0xffffffffu;
    s_hmin = 0xffffffffu;
    s_sticky = 0;
    // psi enters only x_N and the fold region k < nfold (delta+,
    // maps_f64.cpp:363-383): the first and the last block
    const bool need_psi = mc.mode == kModeHigh && (kbase < mc.nfold || kend > mc.N);
    s_psi = need_psi ? high_psi(mc, [&](int64_t j) { return __ldg(a.w + j); }, a.aux[0]) : 0.0;
  }
  __syncthreads();
  if (nw > 0) mbar_wait(&s_mbar, 0);
  RoundAcc ra;
  uint32_t flags = 0;
  const int64_t m0 = ms + int64_t(tid) * kPT;
  // the block's coefficients (those of lane ms - 1 included)
  double* shb = sww + (nw + 1);
  coeffs_block<LAM>(a, sww, wlo, nw, kbase, kend, se, shb, ra, s_psi, flags, tid);
  __syncthreads();
  // lanes of the thread's limbs
  unsigned long long lo[kPT];
  long long hi[kPT];
  {
    int64_t ka = kfirst(m0, a.fb, K);
#pragma unroll
    for (int q = 0; q < kPT; ++q) {
      const int64_t m = m0 + q;
      lo[q] = 0;
      hi[q] = 0;
      if (m < me) {
        const int64_t kb = kfirst(m + 1, a.fb, K);
        lane_of(se, kbase, m, ka, kb, b, lo[q], hi[q]);
        ka = kb;
      }
    }
  }
  long long hin = 0;  // hi(lane_{m0 - 1})
  if (tid == 0 && ms > 0) {
    unsigned long long l0;
    lane_of(se, kbase, ms - 1, kbase, kfirst(ms, a.fb, K), b, l0, hin);
  }
  s_hi[tid] = hi[kPT - 1];
  __syncthreads();
  if (tid > 0) hin = s_hi[tid - 1];
  uint32_t f = kTfIdentity;
  uint32_t tfq[kPT];
#pragma unroll
  for (int q = 0; q < kPT; ++q) {
    const int64_t m = m0 + q;
    tfq[q] = kTfIdentity;
    if (m < me) {
      const __int128 s = (__int128)lo[q] + (__int128)(q == 0 ? hin : hi[q - 1]);
      tfq[q] = limb_tf(s, flags);
      f = tf_compose(f, tfq[q]);
      lo[q] = (unsigned long long)s;  // the low word of s for the limbs below
    }
  }
  uint32_t agg;
  const uint32_t ex = block_scan_tf(f, sw, &agg);
  if (tid == 0) a.aggs[blk] = agg;
  // The limbs for a zero carry into the block (the limb is lo(s_m + c), the
  // carry the limb's transfer function of c); k_carry_patch adds the
  // carry-in of the blocks where it is not zero.  The full product's limbs
  // at and above out_limbs, and the top carry of the full and the high
  // product, go to scratch for the range checks.
  {
    int c = tf_apply(ex, 0);
    const int64_t OL = a.out_limbs;
    uint64_t* tail = hmode ? a.tbuf : reinterpret_cast<uint64_t*>(a.sbuf);
    uint32_t first = 0xffffffffu;
#pragma unroll
    for (int q = 0; q < kPT; ++q) {
      const int64_t m = m0 + q;
      if (m < me) {
        const uint64_t x = lo[q] + uint64_t(int64_t(c));
        c = tf_apply(tfq[q], c);
        if (hmode) {
          tail[m] = x;
          lo[q] = x;
          // a carry-in changes no limb above the first one that is neither
          // 0 nor all ones
          if (x + 1 > 1 && first == 0xffffffffu) first = uint32_t(m - ms);
        } else if (m < OL) {
          a.out[m] = (mc.mode == kModeLow && m == OL - 1 && (a.n & 63)) ? (x & ((1ull << (a.n & 63)) - 1))
                                                                         : x;
        } else {
          tail[m] = x;
        }
        if (m == a.ML - 1 && mc.mode != kModeLow) tail[a.ML] = uint64_t(int64_t(c));
      }
    }
    if (hmode && first != 0xffffffffu) atomicMin(&s_first, first);
  }
  flags |= ra.all_flags();
  {
    const double e = warp_max_nonneg(ra.max_err), m = warp_max_nonneg(ra.max_abs);
    if ((tid & 31) == 0) s_red[tid >> 5] = make_double2(e, m);
  }
  if (flags) atomicOr(&s_flags, flags);
  // the last block to finish turns the per-block functions into each
  // block's carry-in (one exclusive scan instead of a prefix per block);
  // without lanes_cins, k_carry_patch composes them itself
  __shared__ uint32_t s_last;
  if (tid == 0) {
    s_last = 0;
    if (a.lanes_cins) {
      __threadfence();
      s_last = (atomicAdd(a.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
    }
  }
  __syncthreads();
  if (hmode) {
    // nominations and sticky bits of the limbs no carry-in can change (all
    // of block 0's, which has none); k_carry_patch sees the others
    const HighLimbs hl(a);
    const int64_t mfix = blk == 0 ? ms : ms + int64_t(s_first) + 1;
    uint32_t hmin = 0xffffffffu, sticky = 0;
#pragma unroll
    for (int q = 0; q < kPT; ++q) {
      const int64_t m = m0 + q;
      if (m < me && m >= mfix) hl.see(m, lo[q], hmin, sticky);
    }
    // w0's top limb has zero fill above bit 64 - r: never all ones
    if (hl.hr != 0 && blk == 0 && tid == 0 && hl.WL > 0) hmin = min(hmin, uint32_t(hl.WL - 1));
    hmin = __reduce_min_sync(0xffffffffu, hmin);
    sticky = __reduce_or_sync(0xffffffffu, sticky);
    if ((tid & 31) == 0) {
      if (hmin != 0xffffffffu) atomicMin(&s_hmin, hmin);
      if (sticky) s_sticky = 1;
    }
    __syncthreads();
    if (tid == 0) {
      if (s_hmin != 0xffffffffu) atomicMin(a.hstop, s_hmin);
      if (s_sticky) atomicOr(&a.status->high_sticky, 1u);
    }
  }
  if (tid == 0) {
    // one status update per block
    double e = 0.0, m = 0.0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) {
      e = fmax(e, s_red[w].x);
      m = fmax(m, s_red[w].y);
    }
    status_merge(a.status, e, m, s_flags);
  }
  if (s_last) {
    __threadfence();
    const uint32_t B = gridDim.x;
    const uint32_t Q = (B + kT - 1) / kT;
    const uint32_t i0 = uint32_t(tid) * Q, i1 = min(B, i0 + Q);
    uint32_t g = kTfIdentity;
    for (uint32_t i = i0; i < i1; ++i) g = tf_compose(g, __ldcg(a.aggs + i));
    uint32_t tot;
    uint32_t ex = block_scan_tf(g, sw, &tot);
    for (uint32_t i = i0; i < i1; ++i) {
      a.cins[i] = tf_apply(ex, 0);
      ex = tf_compose(ex, __ldcg(a.aggs + i));
    }
    if (tid == 0) *a.ticket = 0;
  }
}

// Single pass: k_carry_lanes with the block's carry-in taken by a
// warp-parallel decoupled look-back (lookback_warp) between its block scan
// and its stores, so every limb is written once with its final value and no
// second kernel patches carry-ins.  A block's aggregate is published right
// after its scan and is almost always a constant function (a carry-in
// changes a block's carry-out only if all its limb sums sit at a wrap
// boundary), so the look-back usually reads one predecessor's aggregate.
// Blocks are dispatched in index order (predecessors are resident or done);
// the look-back words carry a generation that the product's k_zstat
// advances in device memory, so no state is reset between launches and
// replayed CUDA graphs stay valid.  The checks that need final limbs
// (the full product's range, the high product's nominations, sticky bit
// and sign) run here on the block's own limbs.
template <int LAM, int kPT>
__global__ void __launch_bounds__(kT, 4) k_carry_lb(CarryArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int64_t kLimbs = int64_t(kT) * kPT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t sw[32];
  __shared__ long long s_hi[kT];
  __shared__ double s_psi;
  __shared__ uint32_t s_flags, s_gen, s_hmin, s_sticky;
  __shared__ int s_cin;
  __shared__ double2 s_red[kT / 32];
  __shared__ __align__(8) uint64_t s_mbar;
  const int tid = threadIdx.x;
  const MapConsts& mc = a.mc;
  const int b = mc.b;
  const int64_t K = a.K;
  if (tid == 0) s_gen = *a.gen;
  const uint32_t vblk = blockIdx.x;
  const int64_t blk = vblk;
  const int64_t ms = blk * kLimbs;
  const int64_t me = min(a.ML, ms + kLimbs);
  const int64_t kbase = kfirst(ms > 0 ? ms - 1 : 0, a.fb, K);
  const int64_t kend = kfirst(me, a.fb, K);
  const int64_t nwt = (mc.mode == kModeFull) ? K : mc.N;
  const int64_t wlo = max(int64_t(0), kbase - LAM - 1) & ~int64_t(1);
  const int64_t whi = (min(nwt, kend + 2) + 1) & ~int64_t(1);
  const int64_t nw = (LAM > 0 && whi > wlo) ? whi - wlo : 0;
  double* sww = reinterpret_cast<double*>(smem_raw);
  const bool hmode = mc.mode == kModeHigh;
  long long* se = hmode ? reinterpret_cast<long long*>(sww)
                        : reinterpret_cast<long long*>(sww + (nw + 1));
  if (tid == 0 && nw > 0) {
    mbar_init(&s_mbar, 1);
    mbar_expect_tx(&s_mbar, uint32_t(nw * 8));
    bulk_g2s(sww, a.w + wlo, uint32_t(nw * 8), &s_mbar);
  }
  if (tid == 0) {
    s_flags = 0;
    s_hmin = 0xffffffffu;
    s_sticky = 0;
    const bool need_psi = mc.mode == kModeHigh && (kbase < mc.nfold || kend > mc.N);
    s_psi = need_psi ? high_psi(mc, [&](int64_t j) { return __ldg(a.w + j); }, a.aux[0]) : 0.0;
  }
  __syncthreads();
  if (nw > 0) mbar_wait(&s_mbar, 0);
  RoundAcc ra;
  uint32_t flags = 0;
  const int64_t m0 = ms + int64_t(tid) * kPT;
  double* shb = sww + (nw + 1);
  coeffs_block<LAM>(a, sww, wlo, nw, kbase, kend, se, shb, ra, s_psi, flags, tid);
  __syncthreads();
  unsigned long long lo[kPT];
  long long hi[kPT];
  {
    int64_t ka = kfirst(m0, a.fb, K);
#pragma unroll
    for (int q = 0; q < kPT; ++q) {
      const int64_t m = m0 + q;
      lo[q] = 0;
      hi[q] = 0;
      if (m < me) {
        const int64_t kb = kfirst(m + 1, a.fb, K);
        lane_of(se, kbase, m, ka, kb, b, lo[q], hi[q]);
        ka = kb;
      }
    }
  }
  long long hin = 0;  // hi(lane_{m0 - 1})
  if (tid == 0 && ms > 0) {
    unsigned long long l0;
    lane_of(se, kbase, ms - 1, kbase, kfirst(ms, a.fb, K), b, l0, hin);
  }
  s_hi[tid] = hi[kPT - 1];
  __syncthreads();
  if (tid > 0) hin = s_hi[tid - 1];
  uint32_t f = kTfIdentity;
  uint32_t tfq[kPT];
#pragma unroll
  for (int q = 0; q < kPT; ++q) {
    const int64_t m = m0 + q;
    tfq[q] = kTfIdentity;
    if (m < me) {
      const __int128 sm = (__int128)lo[q] + (__int128)(q == 0 ? hin : hi[q - 1]);
      tfq[q] = limb_tf(sm, flags);
      f = tf_compose(f, tfq[q]);
      lo[q] = (unsigned long long)sm;
    }
  }
  uint32_t agg;
  const uint32_t ex = block_scan_tf(f, sw, &agg);
  // publish the aggregate first, so that successors' look-backs can start
  if (tid == 0 && vblk != 0)
    *(volatile unsigned long long*)(a.scan.state + vblk) =
        (static_cast<unsigned long long>(s_gen) << 32) | (1ull << 30) | agg;
  const int64_t OL = a.out_limbs;
  const bool full = mc.mode == kModeFull, low = mc.mode == kModeLow;
  const int hb = int((2 * a.n) & 63);
  auto store = [&](int64_t m, uint64_t x) {
    if (hmode) {
      a.tbuf[m] = x;
    } else if (m < OL) {
      a.out[m] = (low && m == OL - 1 && (a.n & 63)) ? (x & ((1ull << (a.n & 63)) - 1)) : x;
    }
  };
  // the limbs for a zero carry into the block go out before the look-back
  // (whose wait then overlaps their drain); the threads whose carry-in
  // differs once the block's carry-in is known store again (with a nonzero
  // carry-in: the first thread, and the few behind a run of wrapping limbs)
  const int c0 = tf_apply(ex, 0);
  {
    int c = c0;
#pragma unroll
    for (int q = 0; q < kPT; ++q) {
      const int64_t m = m0 + q;
      if (m < me) {
        store(m, lo[q] + uint64_t(int64_t(c)));
        c = tf_apply(tfq[q], c);
      }
    }
  }
  if (tid < 32) {
    const int cin = lookback_warp(a.scan.state, vblk, agg, s_gen, 0, true);
    if (tid == 0) s_cin = cin;
  }
  __syncthreads();
  int c = tf_apply(ex, s_cin);
  const bool restore = c != c0;
#pragma unroll
  for (int q = 0; q < kPT; ++q) {
    const int64_t m = m0 + q;
    if (m < me) {
      const uint64_t x = lo[q] + uint64_t(int64_t(c));
      c = tf_apply(tfq[q], c);
      lo[q] = x;
      if (restore) store(m, x);
      if (full && m >= OL - 1 && (m == OL - 1 ? (hb && (x >> hb)) : x != 0)) flags |= kFlagFullOverflow;
      // sign of the recombined value: the carry out of the top limb
      if (m == a.ML - 1 && c < 0) flags |= full ? uint32_t(kFlagNegative) : hmode ? uint32_t(kFlagHighRange) : 0u;
    }
  }
  flags |= ra.all_flags();
  {
    const double e = warp_max_nonneg(ra.max_err), mx = warp_max_nonneg(ra.max_abs);
    if ((tid & 31) == 0) s_red[tid >> 5] = make_double2(e, mx);
  }
  if (hmode) {
    const HighLimbs hl(a);
    uint32_t hmin = 0xffffffffu, sticky = 0;
#pragma unroll
    for (int q = 0; q < kPT; ++q) {
      const int64_t m = m0 + q;
      if (m < me) hl.see(m, lo[q], hmin, sticky);
    }
    // w0's top limb has zero fill above bit 64 - r: never all ones
    if (hl.hr != 0 && blk == 0 && tid == 0 && hl.WL > 0) hmin = min(hmin, uint32_t(hl.WL - 1));
    hmin = __reduce_min_sync(0xffffffffu, hmin);
    sticky = __reduce_or_sync(0xffffffffu, sticky);
    if ((tid & 31) == 0) {
      if (hmin != 0xffffffffu) atomicMin(&s_hmin, hmin);
      if (sticky) s_sticky = 1;
    }
  }
  if (flags) atomicOr(&s_flags, flags);
  __syncthreads();
  if (tid == 0) {
    if (hmode) {
      if (s_hmin != 0xffffffffu) atomicMin(a.hstop, s_hmin);
      if (s_sticky) atomicOr(&a.status->high_sticky, 1u);
    }
    double e = 0.0, mx = 0.0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) {
      e = fmax(e, s_red[w].x);
      mx = fmax(mx, s_red[w].y);
    }
    status_merge(a.status, e, mx, s_flags);
  }
}

}  // namespace

// k_carry_lanes wrote every limb for a zero carry into its block.  A
// carry-in d = +-1 adds d to a block's limbs from its first limb up to and
// including the first one that does not wrap (old value != ~0 for d = 1,
// != 0 for d = -1).  One warp per block finds that limb 32 limbs at a time
// (a ballot) and updates the limbs below it.  The update stops at the block
// end, since the next block's own carry-in already counts a carry through
// this block.  Then the checks that read the final limbs: the full
// product's range (bits above 2n, carry out of the top limb), and the high
// product's nominations and sticky bits of the limbs k_carry_lanes left out
// (up to the first one that is neither 0 nor all ones) and its range.
template <int kPT>
__global__ void __launch_bounds__(kC2Threads) k_carry_patch(CarryArgs a) {
  pdl_trigger();
  pdl_wait();
  const int64_t kLimbs = a.blk_limbs ? a.blk_limbs : int64_t(kT) * kPT;
  const int64_t nblk = (a.ML + kLimbs - 1) / kLimbs;
  const int64_t blk = (int64_t(blockIdx.x) * kT + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  int d;
  if (a.lanes_cins) {
    if (blk >= nblk) return;
    d = __ldcg(a.cins + blk);
  } else {
    // carry-in: the composition of the preceding blocks' functions, the
    // CTA's prefix by a block scan, then the warp's own few
    __shared__ uint32_t sw[32];
    const uint32_t b0 = blockIdx.x * (kT / 32);
    const uint32_t Q = (b0 + kT - 1) / kT;
    const uint32_t i0 = min(b0, uint32_t(threadIdx.x) * Q), i1 = min(b0, i0 + Q);
    uint32_t g = kTfIdentity;
    for (uint32_t i = i0; i < i1; ++i) g = tf_compose(g, __ldcg(a.aggs + i));
    uint32_t pre;
    (void)block_scan_tf(g, sw, &pre);
    if (blk >= nblk) return;
    for (uint32_t i = b0; i < uint32_t(blk); ++i) pre = tf_compose(pre, __ldcg(a.aggs + i));
    d = tf_apply(pre, 0);
  }
  const int mode = a.mc.mode;
  const bool full = mode == kModeFull, low = mode == kModeLow, high = mode == kModeHigh;
  // full, low: limbs below out_limbs are in the output, the rest (full) in
  // scratch; high: all in tbuf
  const int64_t OL = a.out_limbs, OLx = high ? 0 : OL;
  uint64_t* tail = high ? a.tbuf : reinterpret_cast<uint64_t*>(a.sbuf);
  const int64_t ms = blk * kLimbs, me = min(a.ML, ms + kLimbs);
  auto at = [&](int64_t m) -> uint64_t* { return m < OLx ? a.out + m : tail + m; };
  // high: the limbs [ms, mhi] are those k_carry_lanes did not see
  const bool hsee = high && blk > 0;
  int64_t stop = ms, mhi = me - 1;  // limbs [ms, stop) get d
  if (d != 0 || hsee) {
    stop = me;
    bool have_stop = d == 0;
    const uint64_t wraps = d > 0 ? ~0ull : 0ull;
    // 4 x 32 limbs in flight per step: a run of wrapping limbs (the full
    // product's zero limbs above the value) costs few round trips
    for (int64_t base = ms; base < me; base += 128) {
      uint64_t x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t m = base + 32 * u + lane;
        x[u] = m < me ? *at(m) : wraps;
      }
      bool done = false;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (!have_stop) {
          const unsigned bal = __ballot_sync(0xffffffffu, x[u] != wraps);
          if (bal) {
            stop = base + 32 * u + __ffs(bal);
            have_stop = true;
          }
        }
        if (hsee) {
          const unsigned bal = __ballot_sync(0xffffffffu, x[u] + 1 > 1 && base + 32 * u + lane < me);
          if (bal) {
            mhi = base + 32 * u + __ffs(bal) - 1;
            done = true;
            break;
          }
        } else if (have_stop) {
          done = true;
          break;
        }
      }
      if (done) break;
    }
    if (d != 0) {
      const int lowbits = int(a.n & 63);
      for (int64_t m = ms + lane; m < stop; m += 32) {
        if (low && m >= OL) break;
        uint64_t* p = at(m);
        const uint64_t x = *p + uint64_t(int64_t(d));
        *p = (low && m == OL - 1 && lowbits) ? (x & ((1ull << lowbits) - 1)) : x;  // u v mod 2^n
      }
      __syncwarp();
    }
  }
  if (high) {
    uint32_t flags = 0, hmin = 0xffffffffu, sticky = 0;
    if (hsee) {
      const HighLimbs hl(a);
      for (int64_t m = ms + lane; m <= mhi; m += 32) hl.see(m, tail[m], hmin, sticky);
      hmin = __reduce_min_sync(0xffffffffu, hmin);
      sticky = __reduce_or_sync(0xffffffffu, sticky);
    }
    if (blk == nblk - 1 && lane == 0) {
      const int dend = (d != 0 && stop == me) ? d : 0;
      if (int64_t(tail[a.ML]) + dend < 0) flags |= kFlagHighRange;  // sign of t
    }
    if (lane == 0) {
      if (hmin < __ldcg(a.hstop)) atomicMin(a.hstop, hmin);
      if (sticky) atomicOr(&a.status->high_sticky, 1u);
      if (flags) atomicOr(&a.status->flags, flags);
    }
    return;
  }
  if (!full || me <= OL - 1) return;
  uint32_t flags = 0;
  const int hb = int((2 * a.n) & 63);
  for (int64_t m0 = max(ms, OL - 1) + lane; m0 < me; m0 += 256) {
    uint64_t x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = m0 + 32 * u < me ? *at(m0 + 32 * u) : 0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (m0 + 32 * u == OL - 1 ? (hb && (x[u] >> hb)) : x[u] != 0) flags |= kFlagFullOverflow;
  }
  if (blk == nblk - 1 && lane == 0) {
    // sign of the recombined value: the carry out of the top limb
    const int dend = (d != 0 && stop == me) ? d : 0;
    if (int64_t(tail[a.ML]) + dend < 0) flags |= kFlagNegative;
  }
  flags = __reduce_or_sync(0xffffffffu, flags);
  if (lane == 0 && flags) atomicOr(&a.status->flags, flags);
}

size_t carry2_smem(int b, int lam, int pt, bool /*hbuf: shares the coefficient slot*/) {
  const int64_t nk = (64 * int64_t(kC2Threads * pt + 1) + b - 1) / b + 4;
  if (lam == 0) return size_t(nk + 4) * 8 + 64;  // no staged window
  return size_t(nk + lam + 8) * 8 + size_t(nk + 4) * 8 + 64;
}

template <int PT>
CarryLanesFn lanes_pt(int lam) {
  switch (lam) {
    case 0: return k_carry_lanes<0, PT>;
    case 1: return k_carry_lanes<1, PT>;
    case 2: return k_carry_lanes<2, PT>;
    case 3: return k_carry_lanes<3, PT>;
    case 4: return k_carry_lanes<4, PT>;
    case 5: return k_carry_lanes<5, PT>;
    case 6: return k_carry_lanes<6, PT>;
    case 7: return k_carry_lanes<7, PT>;
    default: return k_carry_lanes<8, PT>;
  }
}

CarryLanesFn carry_lanes_kernel(int lam, int pt) {
  return pt == 4 ? lanes_pt<4>(lam) : pt == 2 ? lanes_pt<2>(lam) : nullptr;
}

template <int PT>
CarryLanesFn lb_pt(int lam) {
  switch (lam) {
    case 0: return k_carry_lb<0, PT>;
    case 4: return k_carry_lb<4, PT>;
    case 5: return k_carry_lb<5, PT>;
    default: return nullptr;
  }
}
CarryLanesFn carry_lb_kernel(int lam, int pt) {
  return pt == 4 ? lb_pt<4>(lam) : pt == 2 ? lb_pt<2>(lam) : lb_pt<1>(lam);
}
CarryLanesFn carry_patch_kernel(int pt) { return pt == 4 ? k_carry_patch<4> : k_carry_patch<2>; }

}  // namespace tmg
