// Fused single-CTA product kernel for transform lengths that fit in shared
// memory (L <= kSmallMaxL).  One CTA computes one whole product:
//   limbs -> balanced chunks (block carry scan) -> pre-map -> forward FFT of
//   z = a + i c -> spectral product -> half-length inverse FFT -> post-map ->
//   rounding tripwire -> recombination with a block carry scan -> limbs.
// A grid of CTAs runs a batch of independent products of the same size in
// one launch (the batched configuration).
//
// Reference path: products_f64.cpp:106-171 end to end.
#include "kernels.cuh"
#include "fft_ct.cuh"

#include <type_traits>

namespace tmg {

namespace {

__device__ __forceinline__ uint64_t window_smem(const uint64_t* limbs,
                                                int64_t nlimbs, int64_t pos,
                                                int b) {
  const uint64_t mask = (b >= 64) ? ~0ull : ((1ull << b) - 1);
  int64_t idx = pos >> 6;
  uint32_t sh = uint32_t(pos & 63);
  uint64_t lo = (idx >= 0 && idx < nlimbs) ? limbs[idx] : 0;
  uint64_t hi = (idx + 1 >= 0 && idx + 1 < nlimbs) ? limbs[idx + 1] : 0;
  uint64_t w = (sh == 0) ? lo : ((lo >> sh) | (hi << (64 - sh)));
  return w & mask;
}

constexpr int kMaxPer = 18;  // values per thread held across a barrier
constexpr uint32_t kPreShift = kMaxLambda;  // > lambda - 1: digit slots above the pre-map outputs

// Whole transform of length SC::R in shared memory (padded natural layout)
// with a compile-time radix schedule: every stage's butterflies spread over
// NTHR threads (NB per thread), stage twiddles omega^{j q step} from the
// two-level table (step = (R / (NS RAD)) * stride), the register block sized
// for this schedule only.  Same arithmetic as the generic stages.
template <bool INV, class SC, int S, int NTHR, int P>
__device__ __forceinline__ void small_ct_stages(double2 (&x)[P], double2* __restrict__ buf,
                                                const TwSmem& tw, uint32_t stride, int tid) {
  constexpr int RAD = SC::rad(S);
  constexpr uint32_t NS = SC::ns(S);
  constexpr uint32_t R = SC::R;
  constexpr uint32_t nbf = R / RAD;
  constexpr int NB = int((nbf + NTHR - 1) / NTHR);
  static_assert(NB * RAD <= P, "register block");
  constexpr uint32_t step = R / (NS * uint32_t(RAD));
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const uint32_t bf = uint32_t(tid) + uint32_t(i) * NTHR;
    if (nbf % NTHR == 0 || bf < nbf) {
#pragma unroll
      for (int q = 0; q < RAD; ++q) x[i * RAD + q] = buf[padidx(bf + q * nbf)];
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const uint32_t bf = uint32_t(tid) + uint32_t(i) * NTHR;
    if (nbf % NTHR == 0 || bf < nbf) {
      const uint32_t tq = bf / NS, j = bf - tq * NS;
      double2* xv = x + i * RAD;
      if (NS > 1 && j != 0) {
#pragma unroll
        for (int q = 1; q < RAD; ++q) {
          const double2 w = tw.get(j * uint32_t(q) * step * stride);
          xv[q] = INV ? cmulc(xv[q], w) : cmul(xv[q], w);
        }
      }
      dft<RAD, INV>(xv);
      const uint32_t ob = tq * NS * RAD + j;
#pragma unroll
      for (int q = 0; q < RAD; ++q) buf[padidx(ob + q * NS)] = xv[q];
    }
  }
  __syncthreads();
  if constexpr (S + 1 < SC::nst) small_ct_stages<INV, SC, S + 1, NTHR, P>(x, buf, tw, stride, tid);
}

}  // namespace

template <int MAXT, int MINB, class SCF = void, class SCI = void>
__device__ __forceinline__ void small_product_body(const SmallArgs& a);

// Two instantiations: up to 512 threads at 128 registers (one CTA per SM),
// and up to 384 threads at <= 85 registers so that two CTAs share an SM --
// products of L <= 6144 (config 4's 2^16-bit batch) are latency-bound at one
// 10-warp CTA per SM.
__global__ void __launch_bounds__(512, 1)
k_small_product(const __grid_constant__ SmallArgs a) {
  small_product_body<512, 1>(a);
}
__global__ void __launch_bounds__(384, 2)
k_small_product_2(const __grid_constant__ SmallArgs a) {
  small_product_body<384, 2>(a);
}
// The full product of BASELINE config 4's size (2^16 bits, L = 6144 =
// 8 x 8 x 8 x 12, inverse 3072 = 8 x 8 x 4 x 12) with compile-time
// schedules at one 768-thread CTA per SM (4096 products: 1.45 -> 1.07 ms).
__global__ void __launch_bounds__(768, 1)
k_small_6144(const __grid_constant__ SmallArgs a) {
  small_product_body<768, 1, Sched<8, 8, 8, 12>, Sched<8, 8, 4, 12>>(a);
}

// The truncated products of BASELINE config 4 (2^16 bits, L = 5120 =
// 16 x 16 x 5 x 4, inverse 2560 = 16 x 16 x 10) with compile-time schedules
// at two 384-thread CTAs per SM.
__global__ void __launch_bounds__(384, 2)
k_small_5120(const __grid_constant__ SmallArgs a) {
  small_product_body<384, 2, Sched<16, 16, 5, 4>, Sched<16, 16, 10>>(a);
}

// Batches of products just above the single-product cutoff (L <= 12288, the
// 2^17-bit range): one CTA per product at up to 768 threads.
__global__ void __launch_bounds__(kSmallBatchMaxThreads, 1)
k_small_product_big(const __grid_constant__ SmallArgs a) {
  small_product_body<kSmallBatchMaxThreads, 1>(a);
}

// Convolution coefficient j from the inverse transform in shared memory:
// y_m = w_{2m} + i w_{2m+1}, times the convolution's 1 / (4 L).
struct SmallW {
  const double2* buf;
  double scale, scale_lo;
  __device__ __forceinline__ double operator()(int64_t j) const {
    const double2 y = buf[padidx(uint32_t(j >> 1))];
    return mul_hl((j & 1) ? y.y : y.x, scale, scale_lo);
  }
};

// The post-map values next to the wraps of the cyclic maps (low: i below
// lambda; high: the fold region) go through the generic helpers, out of
// line: inlined into the unrolled per-thread loop they made the kernel
// about 1 MB of code, and it stalled on instruction fetch.
__device__ __noinline__ double small_postmap_low_slow(const MapConsts& mc, SmallW W, int64_t i) {
  return postmap_low(mc, W, i);
}
__device__ __noinline__ double small_high_buf_slow(const MapConsts& mc, SmallW W, int64_t i) {
  return high_buf(mc, W, i);
}

// post_flat(mc, W, i) for lambda - 1 <= i < N (no term leaves [0, N)): the
// same operation order.
__device__ __forceinline__ double small_post_flat_in(const MapConsts& mc, const SmallW& W, int64_t i) {
  const double Nd = double(mc.N);
  const int fam = (mc.mode == kModeLow) ? 1 : 3;
  const int lam = mc.lambda;
  const double jd = double(i);
  double acc = 0.0;
  RowLoopDown<kMaxLambda>::run([&](auto rc) {
    constexpr int r = decltype(rc)::value;
    if constexpr (r > 0) {
      if (r < lam) acc += W(i - r) * coef_r<r>(fam, jd - double(r), Nd, mc.cpost[r]);
    }
  });
  return acc + W(i);
}

template <int MAXT, int MINB, class SCF, class SCI>
__device__ __forceinline__ void small_product_body(const SmallArgs& a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int64_t L = a.L;
  const MapConsts& mc = a.mc;
  const int b = mc.b;
  const int64_t N = mc.N;

  double2* buf = reinterpret_cast<double2*>(smem_raw);
  // the transform, plus kPreShift slots: the truncated products' digits sit
  // kPreShift slots up (see the pre-map below)
  uint64_t* ul = reinterpret_cast<uint64_t*>(buf + padded_len(uint32_t(L) + kPreShift + 1));
  uint64_t* vl = ul + a.nlimbs;
  uint32_t* sw = reinterpret_cast<uint32_t*>(vl + a.nlimbs);  // 32 words
  double* sd = reinterpret_cast<double*>(sw + 32);             // scalars
  double2* stw = reinterpret_cast<double2*>(sd + 8);            // twiddles
  const TwSmem tw = load_tw_smem(stw, a.fwd, tid, nthr);

  const uint64_t* gu = a.u + int64_t(blockIdx.x) * a.nlimbs;
  const uint64_t* gv = a.v + int64_t(blockIdx.x) * a.nlimbs;
  uint64_t* gout = a.out + int64_t(blockIdx.x) * a.out_limbs;

  // 1. operand limbs -> smem; operand range check (bits at/after n).
  uint32_t flags = 0;
  for (int64_t i = tid; i < a.nlimbs; i += nthr) {
    uint64_t x = __ldg(gu + i), y = __ldg(gv + i);
    ul[i] = x;
    vl[i] = y;
    if (i == a.nlimbs - 1 && (a.n & 63)) {
      uint64_t hm = ~0ull << (a.n & 63);
      if ((x & hm) | (y & hm)) flags |= kFlagInputRange;
    }
  }
  __syncthreads();

  // 2. balanced split: chunk windows, carry scan over the block.
  const int64_t count = a.count;
  const int64_t cpt = (count + nthr - 1) / nthr;
  const int64_t c0 = int64_t(tid) * cpt;
  const int64_t c1 = min(count, c0 + cpt);
  uint32_t fu = kTfIdentity, fv = kTfIdentity;
  for (int64_t j = c0; j < c1 && j < count - 1; ++j) {
    uint64_t wu = window_smem(ul, a.nlimbs, j * b - a.lead, b);
    uint64_t wv = window_smem(vl, a.nlimbs, j * b - a.lead, b);
    fu = tf_compose(fu, mc.balanced ? split_tf(wu, b) : tf_const(0));
    fv = tf_compose(fv, mc.balanced ? split_tf(wv, b) : tf_const(0));
  }
  uint32_t aggu, aggv;
  uint32_t exu = block_scan_tf(fu, sw, &aggu);
  uint32_t exv = block_scan_tf(fv, sw, &aggv);
  {
    int cu = tf_apply(exu, 0), cv = tf_apply(exv, 0);
    for (int64_t j = c0; j < c1; ++j) {
      uint64_t wu = window_smem(ul, a.nlimbs, j * b - a.lead, b);
      uint64_t wv = window_smem(vl, a.nlimbs, j * b - a.lead, b);
      bool top = (j == count - 1);
      double du = double(split_digit(wu, cu, b, top || !mc.balanced));
      double dv = double(split_digit(wv, cv, b, top || !mc.balanced));
      cu = mc.balanced ? tf_apply(split_tf(wu, b), cu) : 0;
      cv = mc.balanced ? tf_apply(split_tf(wv, b), cv) : 0;
      if (j < L + (mc.mode != kModeFull ? 1 : 0))
        buf[padidx(uint32_t(j + (mc.mode != kModeFull ? kPreShift : 0)))] = make_double2(du, dv);
      if (mc.mode == kModeHigh && top) {
        sd[0] = du;
        sd[1] = dv;
      }
    }
    // zero padding of the full product (chunks N..2N-1)
    for (int64_t j = count + tid; j < L; j += nthr)
      buf[padidx(uint32_t(j))] = make_double2(0.0, 0.0);
  }
  __syncthreads();

  // 3. pre-map (low: alpha*, high: gamma+ and root channel).
  if (mc.mode != kModeFull) {
    if (mc.mode == kModeHigh && tid == 0) {
      double tu = sd[0], tv = sd[1];
      auto Du = [&](int64_t i) { return buf[padidx(uint32_t(i + kPreShift))].x; };
      auto Dv = [&](int64_t i) { return buf[padidx(uint32_t(i + kPreShift))].y; };
      sd[2] = root_channel(mc, Du, tu) * root_channel(mc, Dv, tv);
    }
    const double tu = (mc.mode == kModeHigh) ? sd[0] : 0.0;
    const double tv = (mc.mode == kModeHigh) ? sd[1] : 0.0;
    // Digit i sits at slot i + kPreShift and z_j goes to slot j: output j
    // reads slots j + 1 .. j + kPreShift (its cyclic wrap reads digits at or
    // above N, which no output overwrites), so one pass of nthr outputs can
    // write after a single barrier without clobbering what a later pass
    // reads -- and no thread holds more than one output across it.
    auto D2 = [&](int64_t i) { return buf[padidx(uint32_t(i + kPreShift))]; };
    for (int64_t j0 = 0; j0 < N; j0 += nthr) {
      const int64_t j = j0 + tid;
      const double2 z = (j < N) ? premap2(mc, D2, j, tu, tv) : make_double2(0.0, 0.0);
      __syncthreads();
      if (j < N) buf[padidx(uint32_t(j))] = z;
    }
    __syncthreads();
  }

  // 4. forward FFT of z = a + i c, length L.
  LayRows lay1{1u, 0u};
  if constexpr (std::is_void<SCF>::value) {
    fft_smem<false>(buf, lay1, a.fwd, tw, tid, nthr);
  } else {
    double2 xf[16];
    small_ct_stages<false, SCF, 0, MAXT, 16>(xf, buf, tw, 1u, tid);
  }

  // 5. spectral product: W_k = (Z_k + conj Z_-k)(Z_k - conj Z_-k)/(4i L),
  //    then Y_k = (W_k + W_{k+L/2}) + i e^{2 pi i k/L}(W_k - W_{k+L/2}).
  const uint32_t H = uint32_t(L / 2);
  for (uint32_t k = tid; k <= H; k += nthr) {
    uint32_t k2 = (k == 0) ? 0 : uint32_t(L) - k;
    double2 z1 = buf[padidx(k)], z2 = buf[padidx(k2)];
    double2 p = make_double2(z1.x + z2.x, z1.y - z2.y);
    double2 q = make_double2(z1.x - z2.x, z1.y + z2.y);
    double2 pq = cmul(p, q);
    double2 w = make_double2(pq.y, -pq.x);  // -i * pq; 1/(4L) after the inverse (W below)
    buf[padidx(k)] = w;
    if (k2 != k) buf[padidx(k2)] = cconj(w);
  }
  __syncthreads();
  for (uint32_t k = tid; k < H; k += nthr) {
    double2 w1 = buf[padidx(k)], w2 = buf[padidx(k + H)];
    double2 e = cadd(w1, w2);
    double2 o = cmulc(csub(w1, w2), tw.get(k));  // * e^{+2 pi i k/L}
    buf[padidx(k)] = make_double2(e.x - o.y, e.y + o.x);
  }
  __syncthreads();

  // 6. inverse FFT of length L/2: y_m = w_{2m} + i w_{2m+1}.
  if constexpr (std::is_void<SCI>::value) {
    fft_smem<true>(buf, lay1, a.inv, tw, tid, nthr);
  } else {
    double2 xi[16];
    small_ct_stages<true, SCI, 0, MAXT, 16>(xi, buf, tw, 2u, tid);
  }

  // 7. post-map and rounding.
  // the convolution's 1/(4L) is applied to the inverse transform's outputs
  // (CoefSink, k_multipass.cu, says why)
  const SmallW W{buf, a.scale, a.scale_lo};
  const int64_t M = (mc.mode == kModeFull) ? L : (mc.mode == kModeLow ? N : N + 1);
  double psi = 0.0;
  if (mc.mode == kModeHigh) {
    // once per product (maps_f64.cpp:363-371), shared through sd[3]
    if (tid == 0) sd[3] = high_psi(mc, W, sd[2]);
    __syncthreads();
    psi = sd[3];
  }
  RoundAcc ra;
  long long cv[kMaxPer];
  // full / low: strided elements; high: kMaxPer consecutive elements per
  // thread so the folded buffer hbuf(i - 1) of x_i is the previous hbuf(i)
  const bool runs = mc.mode == kModeHigh;
  auto elem = [&](int k) -> int64_t {
    return runs ? int64_t(tid) * kMaxPer + k : tid + int64_t(k) * nthr;
  };
  double hprev = 0.0;
  if (runs && int64_t(tid) * kMaxPer < M) {
    const int64_t i0 = int64_t(tid) * kMaxPer;
    hprev = (i0 >= 1 && i0 - 1 < N) ? small_high_buf_slow(mc, W, i0 - 1) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < kMaxPer; ++k) {
    const int64_t i = elem(k);
    if (i < M) {
      double x;
      if (mc.mode == kModeFull) {
        x = W(i);
      } else if (mc.mode == kModeLow) {
        x = (i >= mc.lambda) ? small_post_flat_in(mc, W, i) * mc.scale_out : small_postmap_low_slow(mc, W, i);
      } else {
        // postmap_high (maps_f64.cpp:372-383) with hbuf(i - 1) carried over;
        // hbuf(i) = post_flat(i) from nfold + lambda - 2 on
        const double hk = (i >= N) ? 0.0
                          : (i >= int64_t(mc.nfold) + mc.lambda - 2 && i >= mc.lambda - 1)
                              ? small_post_flat_in(mc, W, i)
                              : small_high_buf_slow(mc, W, i);
        double v;
        if (i == N) v = psi - hprev * mc.step;
        else if (i == 0) v = hk;
        else v = hk - hprev * mc.step;
        if (i < mc.nfold) v -= psi * mc.fold[i];
        x = v * mc.scale_out;
        hprev = hk;
      }
      cv[k] = ra.round(x);
    }
  }
  __syncthreads();
  long long* cb = reinterpret_cast<long long*>(buf);
#pragma unroll
  for (int k = 0; k < kMaxPer; ++k) {
    const int64_t i = elem(k);
    if (i < M) cb[i] = cv[k];
  }
  flags |= ra.all_flags();
  // block max of errors
  {
    const double e = warp_max_nonneg(ra.max_err), m = warp_max_nonneg(ra.max_abs);
    if ((tid & 31) == 0) status_merge(a.status, e, m, 0);
  }
  __syncthreads();

  // 8. recombination e_k at bit k*b, k < K.
  const int64_t K = a.K;
  long long c0v = cb[0];
  if (mc.mode == kModeLow && tid == 0) {
    if (c0v & ((1ll << b) - 1)) flags |= kFlagLowNotDivisible;
  }
  auto E = [&](int64_t k) -> long long {
    if (mc.mode == kModeLow) {
      long long e = cb[k + 1];
      if (k == 0) e += (c0v >> b);
      return e;
    }
    return cb[k];
  };
  uint64_t* vlimb = reinterpret_cast<uint64_t*>(cb + M + 1);
  const int64_t ML = a.ML;
  const int64_t lpt = (ML + nthr - 1) / nthr;
  const int64_t m0 = int64_t(tid) * lpt;
  const int64_t m1 = min(ML, m0 + lpt);
  const int64_t s_sh = a.shift_s;
  {
    auto lane = [&](int64_t m) -> __int128 { return lane_value(E, m, b, K); };
    uint32_t f = kTfIdentity;
    __int128 prev = lane(m0 - 1);
    for (int64_t m = m0; m < m1; ++m) {
      __int128 cur = lane(m);
      __int128 s = (__int128)(unsigned long long)cur + (prev >> 64);
      f = tf_compose(f, limb_tf(s, flags));
      prev = cur;
    }
    uint32_t agg;
    uint32_t ex = block_scan_tf(f, sw, &agg);
    int c = tf_apply(ex, 0);
    prev = lane(m0 - 1);
    for (int64_t m = m0; m < m1; ++m) {
      __int128 cur = lane(m);
      __int128 s = (__int128)(unsigned long long)cur + (prev >> 64);
      uint32_t tfm = limb_tf(s, flags);
      vlimb[m] = (unsigned long long)(s + c);
      c = tf_apply(tfm, c);
      prev = cur;
    }
    if (m1 == ML && m0 < m1) sd[4] = double(c);  // sign of V
    __syncthreads();
  }
  const int sign = int(sd[4]);
  // 9. outputs and range checks.
  const int64_t OL = a.out_limbs;
  uint32_t topbit = 0, lownz = 0;
  if (mc.mode == kModeFull) {
    if (tid == 0 && sign < 0) flags |= kFlagNegative;
    const int64_t nb2 = 2 * a.n;  // product bits
    for (int64_t m = tid; m < ML; m += nthr) {
      uint64_t x = vlimb[m];
      if (m < OL) {
        if (m == OL - 1 && (nb2 & 63) && (x >> (nb2 & 63))) flags |= kFlagFullOverflow;
        gout[m] = x;
      } else if (x) {
        flags |= kFlagFullOverflow;
      }
    }
    for (int64_t m = ML + tid; m < OL; m += nthr) gout[m] = 0;
  } else if (mc.mode == kModeLow) {
    for (int64_t m = tid; m < OL; m += nthr) {
      uint64_t x = m < ML ? vlimb[m] : 0;
      if (m == OL - 1 && (a.n & 63)) x &= (1ull << (a.n & 63)) - 1;
      gout[m] = x;
    }
  } else {
    // w = round_even(V / 2^s) = (V >> s) + inc (products_f64.cpp:162-166);
    // inc ripples through all-ones limbs of V >> s (block carry scan)
    if (tid == 0) {
      if (sign < 0) flags |= kFlagHighRange;
      const int64_t sb = s_sh - 1;
      uint32_t sticky = 0;
      for (int64_t m = 0; 64 * m < sb && m < ML; ++m) {
        uint64_t x = vlimb[m];
        if (64 * m + 64 > sb) x &= (1ull << (sb - 64 * m)) - 1;
        if (x) { sticky = 1; break; }
      }
      const int bs1 = int((vlimb[sb >> 6] >> (sb & 63)) & 1);
      const int bs = int(((s_sh >> 6) < ML ? vlimb[s_sh >> 6] : 0ull) >> (s_sh & 63) & 1);
      sw[3] = uint32_t(bs1 & int(sticky | uint32_t(bs)));
    }
    __syncthreads();
    const int inc = int(sw[3]);
    __syncthreads();
    const int64_t q = s_sh >> 6;
    const int r = int(s_sh & 63);
    const int64_t WL = ML - q;
    const int64_t wpt = (WL + nthr - 1) / nthr;
    const int64_t w0 = int64_t(tid) * wpt, w1 = min(WL, w0 + wpt);
    auto wlimb = [&](int64_t m) -> uint64_t {
      uint64_t lo = vlimb[m + q];
      uint64_t hi = (m + q + 1 < ML) ? vlimb[m + q + 1] : (sign < 0 ? ~0ull : 0ull);
      return r ? ((lo >> r) | (hi << (64 - r))) : lo;
    };
    uint32_t f = kTfIdentity;
    for (int64_t m = w0; m < w1; ++m) f = tf_compose(f, wlimb(m) == ~0ull ? kTfIdentity : tf_const(0));
    uint32_t agg;
    uint32_t ex = block_scan_tf(f, sw, &agg);
    int c = tf_apply(ex, inc);
    for (int64_t m = w0; m < w1; ++m) {
      const uint64_t x0 = wlimb(m);
      const uint64_t x = x0 + uint64_t(c);
      c = (c && x0 == ~0ull) ? 1 : 0;
      high_classify(x, m, a.n, topbit, lownz, flags);
      if (m < OL) gout[m] = x & high_mask(m, OL, a.n);
    }
    for (int64_t m = WL + tid; m < OL; m += nthr) gout[m] = 0;
  }
  // block-combine flags; the high range test needs both bits of the block
  __syncthreads();
  if (tid == 0) { sw[0] = 0; sw[1] = 0; sw[2] = 0; }
  __syncthreads();
  if (topbit) atomicOr(&sw[0], 1u);
  if (lownz) atomicOr(&sw[1], 1u);
  if (flags) atomicOr(&sw[2], flags);
  __syncthreads();
  if (tid == 0) {
    uint32_t f = sw[2];
    if (sw[0] && sw[1]) f |= kFlagHighRange;
    if (a.pflags) a.pflags[blockIdx.x] = f;
    if (f) atomicOr(&a.status->flags, f);
  }
}

}  // namespace tmg
