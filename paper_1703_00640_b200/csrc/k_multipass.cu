// Multi-pass product pipeline for transform lengths beyond one CTA.
//
//   k_split_scan  carry-in bits of the balanced split (decoupled look-back)
//   k_f1          limbs -> chunks -> pre-map -> column DFTs over A, twiddle
//   k_col         generic in-place column pass (forward over B, inverse over B)
//   k_mid         row DFTs over C for a conjugate row pair, spectral product,
//                 half-length inverse row DFT, twiddle
//   k_ilast       inverse column DFTs over A -> convolution coefficients
//   k_carry       post-map, rounding tripwire, recombination lanes, carry
//                 propagation (decoupled look-back), output limbs
//
// Reference path: products_f64.cpp:106-171 with the FFTW convolution of
// convolution.cpp:175-195.
#include "kernels.cuh"

namespace tmg {

// ---------------------------------------------------------------------------
// Sequential reader of consecutive b-bit windows of u * 2^lead.
struct WindowReader {
  const uint64_t* limbs;
  int64_t nlimbs;
  int64_t idx;
  uint32_t sh;
  uint64_t cur, nxt;
  int b;
  uint64_t mask;
  __device__ __forceinline__ uint64_t load(int64_t i) const {
    return (i >= 0 && i < nlimbs) ? __ldg(limbs + i) : 0ull;
  }
  __device__ __forceinline__ void init(const uint64_t* l, int64_t nl,
                                       int64_t pos, int bb) {
    limbs = l;
    nlimbs = nl;
    b = bb;
    mask = (1ull << bb) - 1;
    idx = pos >> 6;
    sh = uint32_t(pos & 63);
    cur = load(idx);
    nxt = load(idx + 1);
  }
  __device__ __forceinline__ uint64_t next() {
    uint64_t w = sh ? ((cur >> sh) | (nxt << (64 - sh))) : cur;
    sh += b;
    if (sh >= 64) {
      sh -= 64;
      cur = nxt;
      ++idx;
      nxt = load(idx + 1);
    }
    return w & mask;
  }
};

__device__ __forceinline__ int cbit(const uint32_t* cb, int64_t j) {
  return int((__ldg(cb + (j >> 5)) >> (j & 31)) & 1u);
}

__device__ __forceinline__ double digit_at(const uint64_t* limbs,
                                           int64_t nlimbs, int b, int64_t lead,
                                           int64_t count, const uint32_t* cb,
                                           int64_t j) {
  uint64_t w = window_bits(limbs, nlimbs, j * b - lead, b);
  return double(split_digit(w, cbit(cb, j), b, j == count - 1));
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kSplitThreads)
k_split_scan(SplitScanArgs a) {
  __shared__ uint32_t sw[32];
  __shared__ uint32_t s_blk;
  __shared__ int s_cin;
  const bool isv = blockIdx.y == 1;
  const uint64_t* limbs = isv ? a.v : a.u;
  uint32_t* cbits = isv ? a.cbits_v : a.cbits_u;
  ScanState sc = isv ? a.scan_v : a.scan_u;
  const int tid = threadIdx.x;
  if (tid == 0) s_blk = uint32_t(atomicAdd(sc.ctr, 1ull));
  __syncthreads();
  const uint32_t blk = s_blk;
  const int64_t base = int64_t(blk) * (kSplitThreads * 32) + int64_t(tid) * 32;
  const int b = a.b;
  uint32_t f = kTfIdentity;
  uint64_t wv[32];
  {
    WindowReader rd;
    rd.init(limbs, a.nlimbs, base * b - a.lead, b);
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      wv[q] = rd.next();
      if (base + q < a.count - 1) f = tf_compose(f, split_tf(wv[q], b));
    }
  }
  uint32_t agg;
  uint32_t ex = block_scan_tf(f, sw, &agg);
  if (tid == 0) s_cin = lookback_carry(sc.state, blk, agg, sc.epoch, 0);
  __syncthreads();
  int c = tf_apply(ex, s_cin);
  uint32_t bits = 0;
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    bits |= uint32_t(c) << q;
    c = tf_apply(split_tf(wv[q], b), c);
  }
  if (base < a.count) cbits[base >> 5] = bits;
  if (blk == 0 && tid == 0 && (a.n & 63)) {
    uint64_t top = __ldg(limbs + a.nlimbs - 1);
    if (top >> (a.n & 63)) atomicOr(&a.status->flags, uint32_t(kFlagInputRange));
  }
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(sc.ctr + 1, 1ull) == gridDim.x - 1) {
      sc.ctr[0] = 0;
      sc.ctr[1] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// F1: split + pre-map + forward column DFT over A (rows j_a, chunk index
// j = j_a * ncols + col), twiddle omega_L^{col k_a}, store T[k_a][col].
__global__ void __launch_bounds__(512)
k_f1(F1Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const uint32_t c = 1u << a.logc;
  const uint32_t col0 = blockIdx.x * c;
  const uint32_t A = a.fft.R;
  const MapConsts& mc = a.mc;
  const int b = a.b;
  const int64_t N = mc.N;
  const int lam = (mc.mode == kModeFull) ? 1 : mc.lambda;
  LayCols lay{a.logc, c - 1};

  double topu = 0.0, topv = 0.0;
  if (mc.mode == kModeHigh && col0 < uint32_t(mc.nfold + mc.lambda)) {
    topu = digit_at(a.u, a.nlimbs, b, a.lead, a.count, a.cbits_u, N);
    topv = digit_at(a.v, a.nlimbs, b, a.lead, a.count, a.cbits_v, N);
  }
  if (mc.mode == kModeHigh && blockIdx.x == 0 && tid == 0) {
    auto Du = [&](int64_t i) {
      return digit_at(a.u, a.nlimbs, b, a.lead, a.count, a.cbits_u, i);
    };
    auto Dv = [&](int64_t i) {
      return digit_at(a.v, a.nlimbs, b, a.lead, a.count, a.cbits_v, i);
    };
    a.aux[0] = root_channel(mc, Du, topu) * root_channel(mc, Dv, topv);
  }

  // 1. inputs: one thread per row segment of c columns (plus lam-1 halo).
  for (uint32_t row = tid; row < A; row += nthr) {
    const int64_t j0 = int64_t(row) * a.ncols + col0;
    if (mc.mode == kModeFull) {
      if (j0 >= N) {
        for (uint32_t q = 0; q < c; ++q) sbuf[lay.idx(q, row)] = make_double2(0.0, 0.0);
        continue;
      }
      WindowReader ru, rv;
      ru.init(a.u, a.nlimbs, j0 * b, b);
      rv.init(a.v, a.nlimbs, j0 * b, b);
      
      for (uint32_t q = 0; q < c; ++q) {
        const int64_t j = j0 + q;
        uint64_t wu = ru.next(), wv = rv.next();
        double du = 0.0, dv = 0.0;
        if (j < N) {
          du = double(split_digit(wu, cbit(a.cbits_u, j), b, j == a.count - 1));
          dv = double(split_digit(wv, cbit(a.cbits_v, j), b, j == a.count - 1));
        }
        sbuf[lay.idx(q, row)] = make_double2(du, dv);


      }
      continue;
    }
    // low / high: digits of chunks j0 - (lam-1) .. j0 + c - 1
    const int64_t js = j0 - (lam - 1);
    double du[kMaxLambda + 64], dv[kMaxLambda + 64];  // c + lam - 1 <= 72
    const int cnt = int(c) + lam - 1;
    if (js >= 0) {
      WindowReader ru, rv;
      ru.init(a.u, a.nlimbs, js * b - a.lead, b);
      rv.init(a.v, a.nlimbs, js * b - a.lead, b);
      for (int q = 0; q < cnt; ++q) {
        const int64_t j = js + q;
        uint64_t wu = ru.next(), wv = rv.next();
        du[q] = double(split_digit(wu, cbit(a.cbits_u, j), b, j == a.count - 1));
        dv[q] = double(split_digit(wv, cbit(a.cbits_v, j), b, j == a.count - 1));
      }
    } else {
      for (int q = 0; q < cnt; ++q) {
        int64_t j = js + q;
        if (j < 0) j += N;
        du[q] = digit_at(a.u, a.nlimbs, b, a.lead, a.count, a.cbits_u, j);
        dv[q] = digit_at(a.v, a.nlimbs, b, a.lead, a.count, a.cbits_v, j);
      }
    }
    for (uint32_t q = 0; q < c; ++q) {
      const int64_t j = j0 + q;
      const int o = int(q) + lam - 1;  // position of chunk j in du/dv
      auto Du = [&](int64_t k) {
        int64_t d = j - k;
        if (d < 0) d += N;
        return du[o - int(d)];
      };
      auto Dv = [&](int64_t k) {
        int64_t d = j - k;
        if (d < 0) d += N;
        return dv[o - int(d)];
      };
      sbuf[lay.idx(q, row)] =
          make_double2(premap(mc, Du, j, topu), premap(mc, Dv, j, topv));
    }
  }
  __syncthreads();

  // 2. column DFTs
  fft_smem<false>(sbuf, lay, a.fft, tid, nthr);

  // 3. twiddle and store
  const uint32_t tot = A * c;
  for (uint32_t e = tid; e < tot; e += nthr) {
    const uint32_t ka = e >> a.logc, q = e & (c - 1);
    const uint32_t col = col0 + q;
    double2 z = sbuf[lay.idx(q, ka)];
    z = cmul(z, a.tw.get(col * ka));
    a.out[int64_t(ka) * a.ncols + col] = z;
  }
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t col_off(const ColGeom& g, int64_t outer,
                                           uint32_t row, uint32_t col) {
  return outer * g.os + int64_t(row) * g.rs + int64_t(col / g.cw) * g.cs +
         (col % g.cw);
}

__global__ void __launch_bounds__(512)
k_col(ColArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const uint32_t c = 1u << a.logc;
  const uint32_t col0 = blockIdx.x * c;
  const int64_t outer = blockIdx.y;
  const uint32_t R = a.fft.R;
  LayCols lay{a.logc, c - 1};
  const uint32_t tot = R * c;
  for (uint32_t e = tid; e < tot; e += nthr) {
    const uint32_t row = e >> a.logc, q = e & (c - 1);
    sbuf[lay.idx(q, row)] = a.data[col_off(a.g, outer, row, col0 + q)];
  }
  __syncthreads();
  if (a.inv) fft_smem<true>(sbuf, lay, a.fft, tid, nthr);
  else fft_smem<false>(sbuf, lay, a.fft, tid, nthr);
  for (uint32_t e = tid; e < tot; e += nthr) {
    const uint32_t k = e >> a.logc, q = e & (c - 1);
    const uint32_t col = col0 + q;
    double2 z = sbuf[lay.idx(q, k)];
    const uint32_t x = (uint32_t(outer) * a.to + col * a.tc) * k * a.tmul;
    if (x) {
      double2 w = a.tw.get(x);
      z = a.inv ? cmulc(z, w) : cmul(z, w);
    }
    a.data[col_off(a.g, outer, k, col)] = z;
  }
}

// ---------------------------------------------------------------------------
// Row pass: conjugate row pair (r, AB - r), r = k_a + A k_b.
__global__ void __launch_bounds__(512)
k_mid(MidArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const uint32_t AB = a.A * a.B;
  const uint32_t C = a.C, H = C / 2;
  const uint32_t r0 = blockIdx.x;
  const uint32_t r1 = (AB - r0) % AB;
  const uint32_t nrows = (r1 == r0) ? 1 : 2;
  const uint32_t rowstride = padded_len(C) + 4;
  LayRows lay{nrows, rowstride};
  const uint32_t rr[2] = {r0, r1};
  int64_t base[2];
  for (uint32_t i = 0; i < nrows; ++i) {
    const uint32_t r = rr[i];
    base[i] = (int64_t(r % a.A) * a.B + (r / a.A)) * int64_t(C);
  }
  for (uint32_t e = tid; e < nrows * C; e += nthr) {
    const uint32_t i = e >= C ? 1 : 0, k = e - i * C;
    sbuf[lay.idx(i, k)] = a.data[base[i] + k];
  }
  __syncthreads();
  fft_smem<false>(sbuf, lay, a.fwd, tid, nthr);

  // spectral product over the pair
  const uint32_t brw = (r0 != 0) ? 1u : 0u;  // borrow of -k when r != 0
  for (uint32_t k = tid; k < C; k += nthr) {
    const uint32_t kp = (C - k - brw) % C;   // partner column
    const uint32_t ip = (nrows == 2) ? 1u : 0u;
    if (nrows == 1 && kp < k) continue;      // self-paired row: once per pair
    double2 z1 = sbuf[lay.idx(0, k)], z2 = sbuf[lay.idx(ip, kp)];
    double2 p = make_double2(z1.x + z2.x, z1.y - z2.y);
    double2 q = make_double2(z1.x - z2.x, z1.y + z2.y);
    double2 pq = cmul(p, q);
    double2 w = make_double2(pq.y * a.scale, -pq.x * a.scale);
    sbuf[lay.idx(0, k)] = w;
    if (!(nrows == 1 && kp == k)) sbuf[lay.idx(ip, kp)] = cconj(w);
  }
  __syncthreads();
  for (uint32_t e = tid; e < nrows * H; e += nthr) {
    const uint32_t i = e >= H ? 1 : 0, k = e - i * H;
    const uint32_t r = rr[i];
    double2 w1 = sbuf[lay.idx(i, k)], w2 = sbuf[lay.idx(i, k + H)];
    double2 ev = cadd(w1, w2);
    const uint32_t kk = r + AB * k;  // < L/2
    double2 o = cmulc(csub(w1, w2), a.tw.get(kk));
    sbuf[lay.idx(i, k)] = make_double2(ev.x - o.y, ev.y + o.x);
  }
  __syncthreads();
  fft_smem<true>(sbuf, lay, a.inv, tid, nthr);
  for (uint32_t e = tid; e < nrows * H; e += nthr) {
    const uint32_t i = e >= H ? 1 : 0, m = e - i * H;
    const uint32_t r = rr[i];
    double2 z = sbuf[lay.idx(i, m)];
    const uint32_t x = 2u * r * m;  // omega_{L/2}^{r m} = omega_L^{2 r m}
    if (x) z = cmulc(z, a.tw.get(x));
    a.data[base[i] + m] = z;
  }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512)
k_ilast(ILastArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const uint32_t c = 1u << a.logc;
  const uint32_t col0 = blockIdx.x * c;
  const uint32_t R = a.fft.R;
  LayCols lay{a.logc, c - 1};
  const uint32_t tot = R * c;
  for (uint32_t e = tid; e < tot; e += nthr) {
    const uint32_t row = e >> a.logc, q = e & (c - 1);
    sbuf[lay.idx(q, row)] = a.data[col_off(a.g, 0, row, col0 + q)];
  }
  __syncthreads();
  fft_smem<true>(sbuf, lay, a.fft, tid, nthr);
  for (uint32_t e = tid; e < tot; e += nthr) {
    const uint32_t ma = e >> a.logc, q = e & (c - 1);
    a.coef[int64_t(ma) * a.g.ncols + col0 + q] = sbuf[lay.idx(q, ma)];
  }
}

// ---------------------------------------------------------------------------
// Post-map, rounding and carry propagation over all limbs.
__global__ void __launch_bounds__(kCarryThreads)
k_carry(CarryArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t sw[32];
  __shared__ uint32_t s_blk;
  __shared__ int s_cin;
  __shared__ double s_psi;
  __shared__ uint32_t s_flags, s_top, s_low;
  const int tid = threadIdx.x;
  const MapConsts& mc = a.mc;
  const int b = mc.b;
  const int64_t N = mc.N;
  if (tid == 0) {
    s_blk = uint32_t(atomicAdd(a.scan.ctr, 1ull));
    s_flags = 0;
    s_top = 0;
    s_low = 0;
  }
  __syncthreads();
  const uint32_t blk = s_blk;
  constexpr int LB = kCarryThreads * kCarryPerThread;
  const int64_t ms = int64_t(blk) * LB;
  const int64_t me = min(a.ML, ms + LB);
  const int64_t K = a.K;
  const double* gw = a.w;
  auto W = [&](int64_t j) { return __ldg(gw + j); };

  // coefficient window of this block: lanes ms-1 .. me (inclusive)
  int64_t klo = (64 * (ms - 1) + b - 1) / b;
  if (ms == 0) klo = 0;
  int64_t khi = (64 * (me + 1) + 64 + b - 1) / b;
  if (khi > K) khi = K;
  long long* se = reinterpret_cast<long long*>(smem_raw);
  uint64_t* sv = reinterpret_cast<uint64_t*>(se + (khi - klo) + 1);

  if (mc.mode == kModeHigh && tid == 0) s_psi = high_psi(mc, W, a.aux[0]);
  __syncthreads();
  const double psi = s_psi;
  RoundAcc ra;
  uint32_t flags = 0;
  long long c0v = 0;
  if (mc.mode == kModeLow && ms == 0) {
    // c_0 feeds e_0 (low product shift by b, products_f64.cpp:137-142)
    RoundAcc r0;
    c0v = r0.round(postmap_low(mc, W, 0));
    ra.max_err = r0.max_err;
    ra.max_abs = r0.max_abs;
    ra.flags = r0.flags;
    if (c0v & ((1ll << b) - 1)) flags |= kFlagLowNotDivisible;
  }
  for (int64_t k = klo + tid; k < khi; k += kCarryThreads) {
    double x;
    if (mc.mode == kModeFull) x = W(k);
    else if (mc.mode == kModeLow) x = postmap_low(mc, W, k + 1);
    else x = postmap_high(mc, W, k, psi);
    long long e = ra.round(x);
    if (mc.mode == kModeLow && k == 0) e += (c0v >> b);
    se[k - klo] = e;
  }
  __syncthreads();
  flags |= ra.flags;
  {
    double e = ra.max_err, m = ra.max_abs;
    for (int off = 16; off > 0; off >>= 1) {
      e = fmax(e, __shfl_xor_sync(0xffffffffu, e, off));
      m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    }
    if ((tid & 31) == 0) status_merge(a.status, e, m, 0);
  }
  auto E = [&](int64_t k) -> long long { return se[k - klo]; };

  const int64_t m0 = ms + int64_t(tid) * kCarryPerThread;
  const int64_t m1 = min(me, m0 + kCarryPerThread);
  auto lane = [&](int64_t m) -> __int128 {
    return (m < 0) ? (__int128)0 : lane_value(E, m, b, khi);
  };
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
  if (tid == 0) s_cin = lookback_carry(a.scan.state, blk, agg, a.scan.epoch, 0);
  __syncthreads();
  int c = tf_apply(ex, s_cin);
  prev = lane(m0 - 1);
  for (int64_t m = m0; m < m1; ++m) {
    __int128 cur = lane(m);
    __int128 s = (__int128)(unsigned long long)cur + (prev >> 64);
    uint32_t tfm = limb_tf(s, flags);
    sv[m - ms] = (unsigned long long)(s + c);
    c = tf_apply(tfm, c);
    prev = cur;
  }
  if (m1 == me && m0 < m1 && me == a.ML && c < 0) {
    // sign of the recombined value (carry out of the top limb)
    if (mc.mode == kModeFull) flags |= kFlagNegative;
    if (mc.mode == kModeHigh) flags |= kFlagHighRange;
  }
  __syncthreads();

  // outputs
  const int64_t OL = a.out_limbs;
  if (mc.mode == kModeFull) {
    const int64_t nb2 = 2 * a.n;
    for (int64_t m = ms + tid; m < me; m += kCarryThreads) {
      uint64_t x = sv[m - ms];
      if (m < OL) {
        if (m == OL - 1 && (nb2 & 63) && (x >> (nb2 & 63))) flags |= kFlagFullOverflow;
        a.out[m] = x;
      } else if (x) {
        flags |= kFlagFullOverflow;
      }
    }
  } else if (mc.mode == kModeLow) {
    for (int64_t m = ms + tid; m < me; m += kCarryThreads) {
      uint64_t x = sv[m - ms];
      if (m < OL) {
        if (m == OL - 1 && (a.n & 63)) x &= (1ull << (a.n & 63)) - 1;
        a.out[m] = x;
      }
    }
  } else {
    // high: keep all limbs of t; OR the bits strictly below s-1 (sticky)
    const int64_t sb = a.shift_s - 1;  // bit s-1
    uint32_t sticky = 0;
    for (int64_t m = ms + tid; m < me; m += kCarryThreads) {
      uint64_t x = sv[m - ms];
      a.tbuf[m] = x;
      const int64_t bit0 = 64 * m;
      if (bit0 + 64 <= sb) {
        if (x) sticky = 1;
      } else if (bit0 < sb) {
        if (x & ((1ull << (sb - bit0)) - 1)) sticky = 1;
      }
    }
    if (sticky) atomicOr(&s_low, 1u);
  }
  if (flags) atomicOr(&s_flags, flags);
  __syncthreads();
  if (tid == 0) {
    if (s_flags) atomicOr(&a.status->flags, s_flags);
    if (s_low) atomicOr(&a.status->high_sticky, 1u);
    __threadfence();
    if (atomicAdd(a.scan.ctr + 1, 1ull) == gridDim.x - 1) {
      a.scan.ctr[0] = 0;
      a.scan.ctr[1] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// High product rounding (products_f64.cpp:162-166): w = round_even(t / 2^s)
// = (t >> s) + inc, inc = bit_{s-1}(t) & (sticky_{<s-1} | bit_s(t)).  The
// increment ripples through all-ones limbs of t >> s: a second carry scan
// with the increment as the carry into limb 0.  Then the range test
// 0 <= w <= 2^n.
__global__ void __launch_bounds__(kCarryThreads)
k_high_round(HighRoundArgs a) {
  __shared__ uint32_t sw[32];
  __shared__ uint32_t s_blk;
  __shared__ int s_cin;
  __shared__ uint32_t s_flags, s_top, s_low;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_blk = uint32_t(atomicAdd(a.scan.ctr, 1ull));
    s_flags = 0;
    s_top = 0;
    s_low = 0;
  }
  __syncthreads();
  const uint32_t blk = s_blk;
  const int64_t s = a.shift_s;
  const int64_t q = s >> 6;
  const int r = int(s & 63);
  const uint64_t* t = a.tbuf;
  auto tl = [&](int64_t m) -> uint64_t { return m < a.ML ? t[m] : 0ull; };
  const int inc = int((tl((s - 1) >> 6) >> ((s - 1) & 63)) & 1) &
                  int(a.status->high_sticky != 0 || ((tl(s >> 6) >> (s & 63)) & 1));
  constexpr int LB = kCarryThreads * kCarryPerThread;
  const int64_t ms = int64_t(blk) * LB;
  const int64_t me = min(a.WL, ms + LB);
  const int64_t m0 = ms + int64_t(tid) * kCarryPerThread;
  const int64_t m1 = min(me, m0 + kCarryPerThread);
  uint64_t w0[kCarryPerThread];
  uint32_t f = kTfIdentity;
#pragma unroll
  for (int i = 0; i < kCarryPerThread; ++i) {
    const int64_t m = m0 + i;
    if (m < m1) {
      uint64_t lo = tl(m + q), hi = tl(m + q + 1);
      w0[i] = r ? ((lo >> r) | (hi << (64 - r))) : lo;
      f = tf_compose(f, w0[i] == ~0ull ? kTfIdentity : tf_const(0));
    }
  }
  uint32_t agg;
  uint32_t ex = block_scan_tf(f, sw, &agg);
  if (tid == 0) s_cin = lookback_carry(a.scan.state, blk, agg, a.scan.epoch, inc);
  __syncthreads();
  int c = tf_apply(ex, s_cin);
  uint32_t flags = 0, topbit = 0, lownz = 0;
  const int64_t OL = a.out_limbs;
#pragma unroll
  for (int i = 0; i < kCarryPerThread; ++i) {
    const int64_t m = m0 + i;
    if (m < m1) {
      const uint64_t x = w0[i] + uint64_t(c);
      c = (c && w0[i] == ~0ull) ? 1 : 0;
      high_classify(x, m, a.n, topbit, lownz, flags);
      if (m < OL) a.out[m] = x & high_mask(m, OL, a.n);
    }
  }
  if (flags) atomicOr(&s_flags, flags);
  if (topbit) atomicOr(&s_top, 1u);
  if (lownz) atomicOr(&s_low, 1u);
  __syncthreads();
  if (tid == 0) {
    if (s_flags) atomicOr(&a.status->flags, s_flags);
    if (s_top) atomicOr(&a.status->high_topbit, 1u);
    if (s_low) atomicOr(&a.status->high_lownz, 1u);
    __threadfence();
    if (atomicAdd(a.scan.ctr + 1, 1ull) == gridDim.x - 1) {
      a.scan.ctr[0] = 0;
      a.scan.ctr[1] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
__global__ void k_basecase(BaseArgs a) {
  // column sums as 192-bit accumulators, then one sequential carry pass
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(smem_raw);
  const int64_t nl = a.nlimbs;
  const int64_t nc = 2 * nl;
  for (int64_t k = threadIdx.x; k < nc; k += blockDim.x) {
    unsigned long long lo = 0, mid = 0, hi = 0;
    int64_t i0 = k - (nl - 1);
    if (i0 < 0) i0 = 0;
    for (int64_t i = i0; i <= k && i < nl; ++i) {
      unsigned long long x = a.u[i], y = a.v[k - i];
      unsigned long long pl = x * y, ph = __umul64hi(x, y);
      unsigned long long t = lo + pl;
      unsigned long long c1 = t < lo;
      lo = t;
      t = mid + ph;
      unsigned long long c2 = t < mid;
      mid = t + c1;
      c2 += (mid < t);
      hi += c2;
    }
    acc[3 * k] = lo;
    acc[3 * k + 1] = mid;
    acc[3 * k + 2] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long c0 = 0, c1 = 0;  // running carry (128-bit)
    for (int64_t k = 0; k < nc; ++k) {
      unsigned long long lo = acc[3 * k], mid = acc[3 * k + 1], hi = acc[3 * k + 2];
      unsigned long long t = lo + c0;
      unsigned long long cy = t < lo;
      a.prod[k] = t;
      // new carry = mid + hi*2^64 + c1*2^64 + cy
      unsigned long long n0 = mid + c1;
      unsigned long long k1 = n0 < mid;
      unsigned long long n0b = n0 + cy;
      k1 += n0b < n0;
      c0 = n0b;
      c1 = hi + k1;
    }
  }
}

}  // namespace tmg
