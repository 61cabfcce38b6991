// First column pass that applies the pre-map itself (k_f1d_ct).
//
// k_zgen stores the balanced digits of both operands in z's tile order as
// short2 (b <= 14) or int2, four or eight bytes per chunk in place of the
// sixteen of a pre-mapped double2 coefficient, and leaves the pre-map out.
// This pass reads a tile's digit rows with coalesced 16-byte loads (c
// consecutive chunks of a row are contiguous in the tile), forms the
// pre-mapped coefficients z_j = (alpha* U)_j + i (alpha* V)_j (gamma+ with
// the top-chunk fold for the high product) for its c columns, one row per
// thread with the series coefficients of an output shared by both operands
// and every digit converted once, and runs the compile-time column DFT over
// A on them.  The full product has no pre-map: its digits feed the first
// stage straight from global memory.
//
// The pre-map arithmetic is k_zgen's (same factors, same operation order),
// so the coefficients are bit-identical to the two-kernel form.
//
// Reference: maps_f64.cpp:48-136 and 317-348 (alpha*, gamma+), split.cpp:66-102.
#include "colct.cuh"

namespace tmg {

namespace {

// Exact int32 -> double on the FP64 pipe (2^52 + 2^31 magic).
__device__ __forceinline__ double dig2d(int32_t x) {
  return __hiloint2double(0x43300000, int(uint32_t(x) ^ 0x80000000u)) - 4503601774854144.0;
}

// c digit pairs of one tile row from 16-byte shared-memory loads.
template <class DigT, int C>
struct DigRow {
  int32_t u[C], v[C];
  __device__ __forceinline__ void load(const DigT* p) {
    static_assert((sizeof(DigT) * C) % 16 == 0, "digit rows are whole 16-byte vectors");
    const uint4* q = reinterpret_cast<const uint4*>(p);
#pragma unroll
    for (int i = 0; i < int(sizeof(DigT) * C / 16); ++i) {
      const uint4 w = q[i];
      const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
      if constexpr (sizeof(DigT) == 4) {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          u[4 * i + t] = int32_t(int16_t(ws[t] & 0xffffu));
          v[4 * i + t] = int32_t(ws[t]) >> 16;
        }
      } else {
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          u[2 * i + t] = int32_t(ws[2 * t]);
          v[2 * i + t] = int32_t(ws[2 * t + 1]);
        }
      }
    }
  }
};

// Full product: the digits themselves, read by the first stage from the
// staged slab; rows at and above N / ncols are the zero padding of the full
// product's transform.
template <class DigT>
struct DigSrc {
  const DigT* slab;  // row e, item i at e c + i
  int64_t N;
  uint32_t ncols, col0, logc;
  __device__ __forceinline__ double2 operator()(uint32_t item, uint32_t e) const {
    const int64_t j = int64_t(e) * ncols + col0 + item;
    if (j >= N) return make_double2(0.0, 0.0);
    const DigT d = slab[(e << logc) + item];
    return make_double2(dig2d(int32_t(d.x)), dig2d(int32_t(d.y)));
  }
};

// Pre-mapped coefficients of the tile's rows into shared memory.  Row e
// holds chunks j = e ncols + col0 + i (i < c); output j sums rows
// r = LAM-1 .. 0 of digit j - r (cyclic mod N = R ncols), whose halo of
// LAM - 1 digits is the previous tile's row (the last tile of row e - 1 for
// the first tile).  Coefficient of row r: ((j - r) g_1 ... g_{r-1}) c_r,
// g_i = j -/+ i N (coef_r, digits.cuh), with j + N in place of j for the
// wrapped terms of the first LAM - 1 outputs.
template <int LAM, int LOGC, int NTHR, class DigT>
__device__ __forceinline__ void f1d_premap(const F1Args& a, double2* __restrict__ sbuf,
                                           const LayCols& lay, uint32_t R, uint32_t col0,
                                           const DigT* own_slab, const DigT* prev_slab, double topu,
                                           double topv, int tid) {
  constexpr int c = 1 << LOGC;
  constexpr int E = LAM - 1;
  static_assert(E <= c, "the halo lies in the previous tile");
  const MapConsts& mc = a.mc;
  const int64_t N = mc.N;
  const double Nd = double(N);
  const bool low = mc.mode == kModeLow;
  const bool high = mc.mode == kModeHigh;
  const double st = low ? -Nd : Nd;
  double cr[LAM];
#pragma unroll
  for (int r = 0; r < LAM; ++r) cr[r] = mc.cpre[r];
  double gst[LAM > 2 ? LAM - 1 : 1];  // i st, exact
#pragma unroll
  for (int i = 1; i < LAM - 1; ++i) gst[i] = double(i) * st;
  const int64_t fold_end = high ? int64_t(mc.nfold) + LAM : 0;
  for (uint32_t e = uint32_t(tid); e < R; e += NTHR) {
    DigRow<DigT, c> own, prv;
    own.load(own_slab + e * c);
    prv.load(prev_slab + e * c);
    double du[c + E], dv[c + E];
#pragma unroll
    for (int i = 0; i < E; ++i) {
      du[i] = dig2d(prv.u[c - E + i]);
      dv[i] = dig2d(prv.v[c - E + i]);
    }
#pragma unroll
    for (int i = 0; i < c; ++i) {
      du[E + i] = dig2d(own.u[i]);
      dv[E + i] = dig2d(own.v[i]);
    }
    const uint32_t j0 = e * a.ncols + col0;  // < N < 2^31
    const bool wrap = j0 < uint32_t(E);      // some outputs read chunks -1 .. -E (mod N)
#pragma unroll
    for (int i = 0; i < c; ++i) {
      const uint32_t j = j0 + uint32_t(i);
      const double jd = __hiloint2double(0x43300000, int(j)) - 4503599627370496.0;
      double g[LAM > 2 ? LAM - 1 : 1];
#pragma unroll
      for (int t = 1; t < LAM - 1; ++t) g[t] = jd + gst[t];
      double au = 0.0, av = 0.0;
#pragma unroll
      for (int r = LAM - 1; r >= 0; --r) {
        double cf = 1.0;
        if (r > 0) {
          double pp;
          if (wrap && j < uint32_t(r)) {
            // k = j - r + N
            const double base = jd + Nd;
            pp = base - double(r);
#pragma unroll
            for (int t = 1; t < r; ++t) pp *= base + gst[t];
          } else {
            pp = jd - double(r);
#pragma unroll
            for (int t = 1; t < r; ++t) pp *= g[t];
          }
          cf = pp * cr[r];
        }
        au += du[E + i - r] * cf;
        av += dv[E + i - r] * cf;
      }
      double2 v = make_double2(au, av);
      if (high && int64_t(j) < fold_end) high_top_fold(mc, int64_t(j), N, topu, topv, v);
      sbuf[lay.idx(uint32_t(i), e)] = v;
    }
  }
}

// Digit slabs of a tile (rows x c digit pairs, contiguous in z's tile
// order): the tile's own and, with a pre-map, the previous tile's (whose
// last lambda - 1 columns are the halo).  The previous tile of tile 0 is the
// last tile shifted down one row (row e - 1; row R - 1 for e = 0, chunk
// N - 1 preceding chunk 0).  Copied by the TMA engine (cp.async.bulk) into
// one of two shared-memory buffers, one tile ahead of the computation.
template <class DigT, int LAM>
__device__ __forceinline__ void f1d_issue(const DigT* dig, uint32_t tile, uint32_t ntiles, uint32_t zrows,
                                          uint32_t c, DigT* dst, uint64_t* bar) {
  const uint32_t tb = zrows * c * uint32_t(sizeof(DigT));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(bar, LAM > 0 ? 2 * tb : tb);
  bulk_g2s(dst, dig + size_t(tile) * zrows * c, tb, bar);
  if constexpr (LAM > 0) {
    DigT* p = dst + zrows * c;
    if (tile) {
      bulk_g2s(p, dig + size_t(tile - 1) * zrows * c, tb, bar);
    } else {
      const DigT* last = dig + size_t(ntiles - 1) * zrows * c;
      const uint32_t rb = c * uint32_t(sizeof(DigT));
      bulk_g2s(p, last + (zrows - 1) * c, rb, bar);
      bulk_g2s(p + c, last, tb - rb, bar);
    }
  }
}

// k_f1_ct with the pre-map (LAM > 0) or the digit conversion (LAM = 0)
// folded into its first stage; DIG: 1 short2 digits, 2 int2.
template <class SC, int LOGC, int NTHR, int P, int LAM, int DIG>
__global__ void __launch_bounds__(NTHR, (NTHR <= 288 ? 2 : 1)) k_f1d_ct(F1Args a) {
  using DigT = typename std::conditional<DIG == 1, short2, int2>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  constexpr uint32_t c = 1u << LOGC, R = SC::R;
  constexpr uint32_t RL = ct_last_rad<SC>(), NSL = ct_last_ns<SC>();
  constexpr uint32_t nslab = LAM > 0 ? 2 : 1;
  const int tid = threadIdx.x;
  const MapConsts& mc = a.mc;
  const int64_t N = mc.N;
  double2* stab = sbuf + padded_len(R * c);
  double2* qt2 = stab + a.fft.stablen;
  DigT* slabs = reinterpret_cast<DigT*>(qt2 + 2 * c * RL);  // 2 buffers x nslab slabs x zrows x c
  const uint32_t zrows = a.zt.zrows;
  uint64_t* bars = reinterpret_cast<uint64_t*>(slabs + 2 * nslab * zrows * c);
  const TwGlobal tw = a.tw;
  const uint32_t ntiles = a.ncols >> LOGC;
  const DigT* dig = static_cast<const DigT*>(a.dig);
  pdl_trigger();
  if (tid == 0) {
    mbar_init(bars, 1);
    mbar_init(bars + 1, 1);
  }
  for (uint32_t i = tid; i < a.fft.stablen; i += NTHR) stab[i] = __ldg(a.fft.stab + i);
  pdl_wait();
  if (tid == 0 && blockIdx.x < ntiles)
    f1d_issue<DigT, LAM>(dig, blockIdx.x, ntiles, zrows, c, slabs, bars);
  if (mc.mode == kModeHigh && blockIdx.x == 0 && tid == 0) {
    auto Du = [&](int64_t i) { return digit_at(a.u, a.nlimbs, a.b, a.lead, a.count, a.cbits_u, i, mc.balanced != 0); };
    auto Dv = [&](int64_t i) { return digit_at(a.v, a.nlimbs, a.b, a.lead, a.count, a.cbits_v, i, mc.balanced != 0); };
    double tu = 0.0, tv = 0.0;
    if (0 < uint32_t(mc.nfold + mc.lambda)) {
      tu = Du(N);
      tv = Dv(N);
    }
    a.aux[0] = root_channel(mc, Du, tu) * root_channel(mc, Dv, tv);
  }
  __syncthreads();
  const LayCols lay{uint32_t(LOGC), c - 1};
  uint32_t it = 0;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const uint32_t col0 = tile * c;
    const uint32_t nx = tile + gridDim.x;
    const uint32_t buf = it & 1u;
    // the other buffer was last read before the previous tile's barriers
    if (tid == 0 && nx < ntiles)
      f1d_issue<DigT, LAM>(dig, nx, ntiles, zrows, c, slabs + (buf ^ 1u) * nslab * zrows * c, bars + (buf ^ 1u));
    double2* qt = qt2 + buf * (c * RL);
    for (uint32_t i = tid; i < c * RL; i += NTHR) {
      const uint32_t itm = i / RL, q = i - itm * RL;
      const uint32_t x = (col0 + itm) * NSL * q;
      qt[i] = x ? tw.get(x) : make_double2(1.0, 0.0);
    }
    const DigT* own = slabs + buf * nslab * zrows * c;
    double2 x[P];
    if constexpr (LAM == 0) {
      mbar_wait(bars + buf, (it >> 1) & 1u);
      cc_stages<false, SC, 0, LOGC, NTHR, P>(x, sbuf, lay, stab, a.fft,
                                             DigSrc<DigT>{own, N, a.ncols, col0, uint32_t(LOGC)},
                                             F1SinkQ<RL>{a.out, a.ncols, col0, tw, qt}, tid);
    } else {
      double topu = 0.0, topv = 0.0;
      if (mc.mode == kModeHigh && col0 < uint32_t(mc.nfold + mc.lambda)) {
        topu = digit_at(a.u, a.nlimbs, a.b, a.lead, a.count, a.cbits_u, N, mc.balanced != 0);
        topv = digit_at(a.v, a.nlimbs, a.b, a.lead, a.count, a.cbits_v, N, mc.balanced != 0);
      }
      mbar_wait(bars + buf, (it >> 1) & 1u);
      f1d_premap<LAM, LOGC, NTHR, DigT>(a, sbuf, lay, R, col0, own, own + zrows * c, topu, topv, tid);
      __syncthreads();
      cc_stages<false, SC, 0, LOGC, NTHR, P>(x, sbuf, lay, stab, a.fft, SmemSrc<LayCols>{sbuf, lay},
                                             F1SinkQ<RL>{a.out, a.ncols, col0, tw, qt}, tid);
    }
  }
}

template <class SC, int LOGC, int NTHR, int P, int LAM, int DIG>
constexpr F1Fn f1d_fn() {
  if constexpr (LAM > 0 && LAM - 1 > (1 << LOGC)) {
    return nullptr;
  } else {
    return k_f1d_ct<SC, LOGC, NTHR, P, LAM, DIG>;
  }
}

}  // namespace

// Shapes: the radix schedules of the compiled column passes
// (kColCtShapes, k_multipass.cu) with at least four columns per CTA.
// Variants: 0 full short2, 1 full int2, 2 lambda 4 short2, 3 lambda 4
// int2, 4 lambda 5 short2 (lambda = max(4, ceil(52 / b)), so b <= 14 for
// lambda 5 and the int2 form only occurs with lambda 4).
#define TMG_F1D(R_, LOGC_, NTHR_, P_, ...)                                                    \
  {R_, LOGC_, NTHR_, {__VA_ARGS__}, ct_last_rad<Sched<__VA_ARGS__>>(),                       \
   {f1d_fn<Sched<__VA_ARGS__>, LOGC_, NTHR_, P_, 0, 1>(), f1d_fn<Sched<__VA_ARGS__>, LOGC_, NTHR_, P_, 0, 2>(), \
    f1d_fn<Sched<__VA_ARGS__>, LOGC_, NTHR_, P_, 4, 1>(), f1d_fn<Sched<__VA_ARGS__>, LOGC_, NTHR_, P_, 4, 2>(), \
    f1d_fn<Sched<__VA_ARGS__>, LOGC_, NTHR_, P_, 5, 1>()}}
static const F1DShape kF1DShapes[] = {
    TMG_F1D(1728, 2, 576, 12, 12, 12, 12),
    TMG_F1D(1440, 2, 576, 12, 12, 12, 10),
    // 2^24 (BASELINE config 2): 448 x 4096 full, 320 x 4096 low/high
    TMG_F1D(448, 4, 512, 16, 16, 4, 7),
    TMG_F1D(320, 4, 512, 16, 16, 5, 4),
};
#undef TMG_F1D

size_t f1d_smem_bytes(uint32_t R, uint32_t c, uint32_t stablen, uint32_t radl, uint32_t zrows, int lam,
                      int dig) {
  const size_t slab = size_t(zrows) * c * (dig == 1 ? 4 : 8);
  return size_t(padded_len(R * c)) * 16 + size_t(stablen) * 16 + 2 * size_t(c) * radl * 16 +
         2 * (lam > 0 ? 2 : 1) * slab + 16;
}

const F1DShape* f1d_for(uint32_t R) {
  for (const F1DShape& sh : kF1DShapes)
    if (sh.R == R) return &sh;
  return nullptr;
}

int f1d_variant(int lam, int dig) {
  if (lam == 0) return dig == 1 ? 0 : 1;
  if (lam == 4) return dig == 1 ? 2 : 3;
  if (lam == 5 && dig == 1) return 4;
  return -1;
}

}  // namespace tmg
