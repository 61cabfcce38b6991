// Multi-pass product pipeline for transform lengths beyond one CTA.
//
//   k_zstat/k_zgen (k_zgen.cu) balanced split (+ pre-map where k_f1d_ct
//                 does not apply it); carries composed from per-block
//                 aggregates
//   k_f1d_ct      (k_f1d.cu) first column pass on the split's stored digits,
//                 pre-map in its first stage; k_f1_ct reads pre-mapped
//                 coefficients, with a compile-time schedule for the hot
//                 column lengths; k_f1 / k_f1_pp otherwise
//   k_col_ct      middle column passes of three-pass plans (over B, in
//                 place); k_col / the ping-pong variants otherwise
//   k_mid_4096    row DFTs over C = 4096 for a conjugate row pair, spectral
//                 product and repack in registers (shuffles between the
//                 pair's lanes), half-length inverse, output twiddle
//                 (persistent, next pair's row 0 staged by TMA); k_mid for
//                 other row lengths
//   k_ilast_ct    inverse column DFTs over A -> convolution coefficients;
//                 k_ilast / k_ilast_pp otherwise
//   k_carry       single-pass look-back carry beyond 2^32 carry bits (the
//                 default is k_carry_lb, or k_carry_lanes + k_carry_patch,
//                 in k_carry2.cu)
//   k_high_agg / k_high_round  round(t / 2^s) of the high product
//
// Reference path: products_f64.cpp:106-171 with the FFTW convolution of
// convolution.cpp:175-195.
#include <vector>

#include "kernels.cuh"
#include "fft_ct.cuh"
#include "colct.cuh"

namespace tmg {

struct SmemLimbs {
  const uint64_t* s;  // s[i - i0] for i in [i0, i0 + n)
  int64_t i0, n;
  __device__ __forceinline__ uint64_t operator()(int64_t i) const {
    const int64_t o = i - i0;
    return (o >= 0 && o < n) ? s[o] : 0ull;
  }
};

__device__ __forceinline__ uint32_t take_ticket(unsigned long long* ctr) {
  return uint32_t(atomicAdd(ctr, 1ull));
}

__device__ __forceinline__ void release_ticket(unsigned long long* ctr,
                                               unsigned grid) {
  __threadfence();
  if (atomicAdd(ctr + 1, 1ull) == grid - 1) {
    ctr[0] = 0;
    ctr[1] = 0;
  }
}

// ---------------------------------------------------------------------------
// Column-pass sources and sinks.
__device__ __forceinline__ int64_t col_off(const ColGeom& g, int64_t outer,
                                           uint32_t row, uint32_t col) {
  return outer * g.os + int64_t(row) * g.rs + int64_t(col / g.cw) * g.cs +
         (col % g.cw);
}

struct ColSrc {
  const double2* data;
  ColGeom g;
  int64_t outer;
  uint32_t col0;
  __device__ __forceinline__ double2 operator()(uint32_t item, uint32_t e) const {
    return data[col_off(g, outer, e, col0 + item)];
  }
};

struct ColSink {
  double2* data;
  ColGeom g;
  int64_t outer;
  uint32_t col0;
  TwGlobal tw;
  uint32_t to, tc, tmul;
  bool inv, twiddle;
  __device__ __forceinline__ void operator()(uint32_t item, uint32_t k, double2 v) const {
    const uint32_t col = col0 + item;
    if (twiddle) {
      const uint32_t x = (uint32_t(outer) * to + col * tc) * k * tmul;
      if (x) {
        const double2 w = tw.get(x);
        v = inv ? cmulc(v, w) : cmul(v, w);
      }
    }
    data[col_off(g, outer, k, col)] = v;
  }
  __device__ __forceinline__ double2 pre(uint32_t item, uint32_t k) const {
    return tw.get((uint32_t(outer) * to + (col0 + item) * tc) * k * tmul);
  }
  __device__ __forceinline__ void put(uint32_t item, uint32_t k, double2 v, double2 w) const {
    data[col_off(g, outer, k, col0 + item)] = inv ? cmulc(v, w) : cmul(v, w);
  }
};

// ---------------------------------------------------------------------------
// F1: forward column DFTs over A of the pre-mapped coefficients z_j
// (j = j_a * ncols + col; zero for j >= N, the full product's padding), the
// high product's top-chunk fold added on the fly, twiddle omega_L^{col k_a},
// store T[k_a][col].
struct ZSrc {
  const double2* z;
  ZTile zt;
  int64_t N;
  uint32_t ncols, col0;
  const MapConsts* mc;
  double topu, topv;
  __device__ __forceinline__ double2 operator()(uint32_t item, uint32_t e) const {
    const int64_t j = int64_t(e) * ncols + col0 + item;
    if (j >= N) return make_double2(0.0, 0.0);
    // tile of this CTA: rows consecutive, 2^logc columns per row
    double2 v = zt.natural ? z[j] : z[((col0 >> zt.logc) * zt.zrows + e) * (1u << zt.logc) + item];
    if (mc->mode == kModeHigh && j < mc->nfold + mc->lambda) high_top_fold(*mc, j, N, topu, topv, v);
    return v;
  }
};

struct F1Sink {
  double2* out;
  uint32_t ncols, col0;
  TwGlobal tw;
  __device__ __forceinline__ void operator()(uint32_t item, uint32_t k, double2 v) const {
    const uint32_t col = col0 + item;
    const uint32_t x = col * k;
    if (x) v = cmul(v, tw.get(x));
    out[int64_t(k) * ncols + col] = v;
  }
  // omega^0 = (1, 0) exactly, so x = 0 multiplies exactly
  __device__ __forceinline__ double2 pre(uint32_t item, uint32_t k) const {
    return tw.get((col0 + item) * k);
  }
  __device__ __forceinline__ void put(uint32_t item, uint32_t k, double2 v, double2 w) const {
    out[int64_t(k) * ncols + col0 + item] = cmul(v, w);
  }
};

// transfers in flight per thread in the single-buffer column passes
#ifndef TMG_COL_U
#define TMG_COL_U 4
#endif
constexpr int kColU = TMG_COL_U;

// Tile <-> shared memory copies of a column pass: element (item, e) of the
// R x c tile, consecutive threads on consecutive items (columns) so each
// warp touches c-element row segments; 8 transfers per thread in flight.
template <int U = 8, class Lay, class Src>
__device__ __forceinline__ void tile_load(double2* __restrict__ buf, const Lay& lay, uint32_t R,
                                          uint32_t c, const Src& src, int tid, int nthr) {
  const uint32_t n = R * c, lc = 31 - __clz(c);
  uint32_t i = tid;
  for (; i + (U - 1) * nthr < n; i += U * nthr) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t t = i + u * nthr;
      v[u] = src(t & (c - 1), t >> lc);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t t = i + u * nthr;
      buf[lay.idx(t & (c - 1), t >> lc)] = v[u];
    }
  }
  for (; i < n; i += nthr) buf[lay.idx(i & (c - 1), i >> lc)] = src(i & (c - 1), i >> lc);
}
// Sinks with a twiddle expose pre(item, e) (the twiddle, fetched early) and
// put(item, e, v, w); the store loop keeps 8 elements' fetches in flight.
template <class Sink>
struct TileSinkPre {
  static constexpr bool value = false;
};
// U: transfers in flight per thread (8; 4 in the 1024-thread ping-pong
// kernels, whose 64-register budget holds 4 values and 4 twiddles).
template <int U = 8, class Lay, class Sink>
__device__ __forceinline__ void tile_store(const double2* __restrict__ buf, const Lay& lay,
                                           uint32_t R, uint32_t c, const Sink& sink, int tid,
                                           int nthr) {
  const uint32_t n = R * c, lc = 31 - __clz(c);
  uint32_t i = tid;
  for (; i + (U - 1) * nthr < n; i += U * nthr) {
    double2 v[U], w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t t = i + u * nthr;
      v[u] = buf[lay.idx(t & (c - 1), t >> lc)];
      if constexpr (TileSinkPre<Sink>::value) w[u] = sink.pre(t & (c - 1), t >> lc);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t t = i + u * nthr;
      if constexpr (TileSinkPre<Sink>::value) sink.put(t & (c - 1), t >> lc, v[u], w[u]);
      else sink(t & (c - 1), t >> lc, v[u]);
    }
  }
  for (; i < n; i += nthr) {
    const uint32_t item = i & (c - 1), e = i >> lc;
    sink(item, e, buf[lay.idx(item, e)]);
  }
}

template <>
struct TileSinkPre<F1Sink> {
  static constexpr bool value = true;
};
template <>
struct TileSinkPre<ColSink> {
  static constexpr bool value = true;
};

// Inter-pass twiddles of the first column pass without global loads at
// store time.  With nthr a multiple of c, thread tid always stores column
// item = tid & (c - 1) at rows k = k0 + D s (k0 = tid >> logc,
// D = nthr >> logc), so omega_L^{col k} = omega_L^{col k0} * omega_L^{col D s}:
// one factor per thread (base) and a c x S table per CTA (step), both taken
// from the exact two-level global table at kernel entry, where their latency
// hides behind the tile load.  The store then reads two shared-memory values
// per element instead of two global ones.  x = 0 factors are (1, 0) exactly,
// so untwiddled elements stay exact.
__host__ __device__ inline uint32_t f1_tw_S(uint32_t A, uint32_t c, uint32_t nthr) {
  return (A * c + nthr - 1) / nthr;
}
size_t f1_tw_bytes(uint32_t A, uint32_t c, uint32_t nthr) {
  return (nthr % c) ? 0 : (size_t(nthr) + size_t(c) * f1_tw_S(A, c, nthr)) * 16;
}

struct F1Tw {
  double2* base;  // nthr entries
  double2* step;  // S x c entries, step[(s << logc) + item]
  uint32_t S;
};

__device__ __forceinline__ F1Tw f1_tw_stage(double2* dst, const F1Sink& sink, uint32_t A,
                                           uint32_t logc, int tid, int nthr) {
  const uint32_t c = 1u << logc;
  F1Tw t{dst, dst + nthr, f1_tw_S(A, c, uint32_t(nthr))};
  const uint32_t item = uint32_t(tid) & (c - 1), k0 = uint32_t(tid) >> logc;
  const uint32_t D = uint32_t(nthr) >> logc;
  const uint32_t xb = (sink.col0 + item) * k0;
  t.base[tid] = (k0 < A && xb) ? sink.tw.get(xb) : make_double2(1.0, 0.0);
  for (uint32_t i = tid; i < (t.S << logc); i += nthr) {
    const uint32_t x = (sink.col0 + (i & (c - 1))) * D * (i >> logc);
    t.step[i] = x ? sink.tw.get(x) : make_double2(1.0, 0.0);
  }
  return t;
}

template <int U, class Lay>
__device__ __forceinline__ void f1_store(const double2* __restrict__ buf, const Lay& lay,
                                         uint32_t A, uint32_t logc, const F1Sink& sink,
                                         const F1Tw& t, int tid, int nthr) {
  const uint32_t c = 1u << logc;
  const uint32_t item = uint32_t(tid) & (c - 1), k0 = uint32_t(tid) >> logc;
  const uint32_t D = uint32_t(nthr) >> logc;
  const double2 b = t.base[tid];
  double2* out = sink.out + (sink.col0 + item);
  for (uint32_t s0 = 0; s0 < t.S; s0 += U) {
    double2 v[U], w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t s = s0 + u, k = k0 + D * s;
      if (s < t.S && k < A) {
        v[u] = buf[lay.idx(item, k)];
        w[u] = t.step[(s << logc) + item];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t s = s0 + u, k = k0 + D * s;
      if (s < t.S && k < A) out[int64_t(k) * sink.ncols] = cmul(v[u], cmul(b, w[u]));
    }
  }
}

size_t f1_smem_bytes(uint32_t A, uint32_t c) {
  return size_t(padded_len(A * c)) * 16 + size_t(A) * 16;  // data + stage table (< A)
}

__global__ void __launch_bounds__(512)
k_f1(F1Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const uint32_t c = 1u << a.logc;
  const uint32_t col0 = blockIdx.x * c;
  const uint32_t A = a.fft.R;
  const MapConsts& mc = a.mc;
  const int64_t N = mc.N;
  LayCols lay{a.logc, c - 1};
  pdl_trigger();
  const TwStage tw = load_tw_stage(sbuf + padded_len(A * c), a.fft, tid, nthr);
  pdl_wait();
  double topu = 0.0, topv = 0.0;
  if (mc.mode == kModeHigh && col0 < uint32_t(mc.nfold + mc.lambda)) {
    topu = digit_at(a.u, a.nlimbs, a.b, a.lead, a.count, a.cbits_u, N, mc.balanced != 0);
    topv = digit_at(a.v, a.nlimbs, a.b, a.lead, a.count, a.cbits_v, N, mc.balanced != 0);
  }
  if (mc.mode == kModeHigh && blockIdx.x == 0 && tid == 0) {
    auto Du = [&](int64_t i) { return digit_at(a.u, a.nlimbs, a.b, a.lead, a.count, a.cbits_u, i, mc.balanced != 0); };
    auto Dv = [&](int64_t i) { return digit_at(a.v, a.nlimbs, a.b, a.lead, a.count, a.cbits_v, i, mc.balanced != 0); };
    a.aux[0] = root_channel(mc, Du, topu) * root_channel(mc, Dv, topv);
  }
  // tile -> shared memory: all loads of a thread in flight together
  const F1Sink sink{a.out, a.ncols, col0, a.tw};
  const bool stw = a.stw != 0;
  F1Tw ftw{};
  if (stw) ftw = f1_tw_stage(sbuf + padded_len(A * c) + A, sink, A, a.logc, tid, nthr);
  const ZSrc src{a.z, a.zt, N, a.ncols, col0, &a.mc, topu, topv};
  tile_load<kColU>(sbuf, lay, A, c, src, tid, nthr);
  __syncthreads();
  fft_smem_compact<false>(sbuf, lay, a.fft, tw, tid, nthr);
  if (stw) f1_store<kColU>(sbuf, lay, A, a.logc, sink, ftw, tid, nthr);
  else tile_store<kColU>(sbuf, lay, A, c, sink, tid, nthr);
}

// ---------------------------------------------------------------------------
size_t col_smem_bytes(uint32_t R, uint32_t c) {
  return size_t(padded_len(R * c)) * 16 + size_t(R) * 16;
}

__global__ void __launch_bounds__(512)
k_col(ColArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const uint32_t c = 1u << a.logc;
  const uint32_t col0 = blockIdx.x * c;
  const int64_t outer = blockIdx.y;
  LayCols lay{a.logc, c - 1};
  pdl_trigger();
  const TwStage tw = load_tw_stage(sbuf + padded_len(a.fft.R * c), a.fft, tid, nthr);
  pdl_wait();
  __syncthreads();
  ColSrc src{a.data, a.g, outer, col0};
  ColSink sink{a.data, a.g, outer, col0, a.tw, a.to, a.tc, a.tmul, a.inv != 0, true};
  tile_load<kColU>(sbuf, lay, a.fft.R, c, src, tid, nthr);
  __syncthreads();
  if (a.inv) fft_smem_compact<true>(sbuf, lay, a.fft, tw, tid, nthr);
  else fft_smem_compact<false>(sbuf, lay, a.fft, tw, tid, nthr);
  tile_store<kColU>(sbuf, lay, a.fft.R, c, sink, tid, nthr);
}

// ---------------------------------------------------------------------------
// Ping-pong column passes (fft_pp): two tiles in shared memory, one barrier
// per stage, 1024 threads at 64 registers, radix <= 8 schedules, stage
// twiddles through L1.  Same tiles, sources and sinks as above.
size_t colpp_smem_bytes(uint32_t R, uint32_t c) { return 2 * size_t(padded_len(R * c)) * 16; }

__global__ void __launch_bounds__(kColPPThreads, 1)
k_f1_pp(F1Args a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* b0 = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const uint32_t c = 1u << a.logc;
  const uint32_t col0 = blockIdx.x * c;
  const uint32_t A = a.fft.R;
  double2* b1 = b0 + padded_len(A * c);
  const MapConsts& mc = a.mc;
  const int64_t N = mc.N;
  LayCols lay{a.logc, c - 1};
  double topu = 0.0, topv = 0.0;
  if (mc.mode == kModeHigh && col0 < uint32_t(mc.nfold + mc.lambda)) {
    topu = digit_at(a.u, a.nlimbs, a.b, a.lead, a.count, a.cbits_u, N, mc.balanced != 0);
    topv = digit_at(a.v, a.nlimbs, a.b, a.lead, a.count, a.cbits_v, N, mc.balanced != 0);
  }
  if (mc.mode == kModeHigh && blockIdx.x == 0 && tid == 0) {
    auto Du = [&](int64_t i) { return digit_at(a.u, a.nlimbs, a.b, a.lead, a.count, a.cbits_u, i, mc.balanced != 0); };
    auto Dv = [&](int64_t i) { return digit_at(a.v, a.nlimbs, a.b, a.lead, a.count, a.cbits_v, i, mc.balanced != 0); };
    a.aux[0] = root_channel(mc, Du, topu) * root_channel(mc, Dv, topv);
  }
  const F1Sink sink{a.out, a.ncols, col0, a.tw};
  const bool stw = a.stw != 0;
  F1Tw ftw{};
  if (stw) ftw = f1_tw_stage(b1 + padded_len(A * c), sink, A, a.logc, tid, nthr);
  const ZSrc src{a.z, a.zt, N, a.ncols, col0, &a.mc, topu, topv};
  tile_load<4>(b0, lay, A, c, src, tid, nthr);
  __syncthreads();
  const double2* res = fft_pp<false>(b0, b1, lay, a.fft, tid, nthr);
  if (stw) f1_store<4>(res, lay, A, a.logc, sink, ftw, tid, nthr);
  else tile_store<4>(res, lay, A, c, sink, tid, nthr);
}

// INV at compile time: one transform direction per instantiation keeps the
// kernel within its 64 registers.
template <bool INV>
__global__ void __launch_bounds__(kColPPThreads, 1)
k_col_pp_t(ColArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* b0 = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const uint32_t c = 1u << a.logc;
  const uint32_t col0 = blockIdx.x * c;
  const int64_t outer = blockIdx.y;
  double2* b1 = b0 + padded_len(a.fft.R * c);
  LayCols lay{a.logc, c - 1};
  ColSrc src{a.data, a.g, outer, col0};
  ColSink sink{a.data, a.g, outer, col0, a.tw, a.to, a.tc, a.tmul, a.inv != 0, true};
  tile_load<4>(b0, lay, a.fft.R, c, src, tid, nthr);
  __syncthreads();
  const double2* res = fft_pp<INV>(b0, b1, lay, a.fft, tid, nthr);
  tile_store<4>(res, lay, a.fft.R, c, sink, tid, nthr);
}

ColFn col_pp_kernel(bool inv) { return inv ? k_col_pp_t<true> : k_col_pp_t<false>; }

// ---------------------------------------------------------------------------
// Row pass: conjugate row pair (r, AB - r), r = k_a + A k_b.
struct RowSrc {
  const double2* data;
  int64_t base0, base1;
  __device__ __forceinline__ double2 operator()(uint32_t item, uint32_t e) const {
    return data[(item ? base1 : base0) + e];
  }
};

struct RowSink {
  double2* data;
  int64_t base0, base1;
  uint32_t r0, r1;
  TwGlobal tw;
  __device__ __forceinline__ void operator()(uint32_t item, uint32_t m, double2 v) const {
    const uint32_t x = 2u * (item ? r1 : r0) * m;  // omega_{L/2}^{r m} = omega_L^{2 r m}
    if (x) v = cmulc(v, tw.get(x));
    data[(item ? base1 : base0) + m] = v;
  }
};

// Output twiddles of the C = 4096 row pass: the last inverse stage's thread
// stores m = ob + q NS (q < RAD) of its row, and
// omega_L^{2 r m} = omega_L^{2 r ob} * omega_L^{2 r NS q}: the first factor
// is fetched (two-level global table) before the stage's DFT, the second
// comes from a per-pair table qt[item * RAD + q] staged in shared memory,
// so the store does no global twiddle loads.  Both factors are (1, 0)
// exactly at x = 0.
template <uint32_t RAD>
struct RowSinkQ {
  double2* data;
  int64_t base0, base1;
  uint32_t r0, r1;
  TwGlobal tw;
  const double2* qt;
  __device__ __forceinline__ double2 prep(uint32_t item, uint32_t ob) const {
    const uint32_t x = 2u * (item ? r1 : r0) * ob;
    return x ? tw.get(x) : make_double2(1.0, 0.0);
  }
  __device__ __forceinline__ void put(uint32_t item, uint32_t m, uint32_t q, double2 v,
                                      double2 b) const {
    v = cmulc(v, cmul(b, qt[item * RAD + q]));
    data[(item ? base1 : base0) + m] = v;
  }
};
template <uint32_t RAD>
struct SinkPrep<RowSinkQ<RAD>> {
  static constexpr bool value = true;
};
constexpr uint32_t kMidQEntries = 32;  // 2 rows x last-stage radix (<= 16)

size_t mid_smem_bytes(uint32_t C, uint32_t inv_stablen) {
  return size_t(2) * (padded_len(C) + 4) * 16 + size_t(C) * 16 + size_t(inv_stablen) * 16 +
         size_t(kMidQEntries) * 16;
}

__global__ void __launch_bounds__(512)
k_mid(MidArgs a) {
  pdl_trigger();
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.gen += 1u;  // next look-backs' generation
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
  const int64_t base0 = (int64_t(r0 % a.A) * a.B + (r0 / a.A)) * int64_t(C);
  const int64_t base1 = (int64_t(r1 % a.A) * a.B + (r1 / a.A)) * int64_t(C);
  double2* stw = sbuf + 2 * rowstride;
  const TwStage tw = load_tw_stage(stw, a.fwd, tid, nthr);
  const TwStage twi = (a.inv.stab == a.fwd.stab)
                          ? tw
                          : load_tw_stage(stw + a.fwd.stablen, a.inv, tid, nthr);

  fft_pass<false>(sbuf, lay, a.fwd, tw, RowSrc{a.data, base0, base1},
                  SmemSink<LayRows>{sbuf, lay}, tid, nthr);
  __syncthreads();

  // spectral product over the pair:
  // W_k = (Z_k + conj Z_-k)(Z_k - conj Z_-k) / (4 i L), W_-k = conj W_k
  const uint32_t brw = (r0 != 0) ? 1u : 0u;  // borrow of -k when r != 0
  for (uint32_t k = tid; k < C; k += nthr) {
    const uint32_t kp = (C - k - brw) % C;
    const uint32_t ip = (nrows == 2) ? 1u : 0u;
    if (nrows == 1 && kp < k) continue;
    const double2 z1 = sbuf[lay.idx(0, k)], z2 = sbuf[lay.idx(ip, kp)];
    const double2 p = make_double2(z1.x + z2.x, z1.y - z2.y);
    const double2 q = make_double2(z1.x - z2.x, z1.y + z2.y);
    const double2 pq = cmul(p, q);
    const double2 w = make_double2(pq.y, -pq.x);  // unscaled (see CoefSink)
    sbuf[lay.idx(0, k)] = w;
    if (!(nrows == 1 && kp == k)) sbuf[lay.idx(ip, kp)] = cconj(w);
  }
  __syncthreads();
  // Y_k = (W_k + W_{k+L/2}) + i e^{2 pi i k / L} (W_k - W_{k+L/2})
  for (uint32_t e = tid; e < nrows * H; e += nthr) {
    const uint32_t i = e >= H ? 1 : 0, k = e - i * H;
    const uint32_t r = i ? r1 : r0;
    const double2 w1 = sbuf[lay.idx(i, k)], w2 = sbuf[lay.idx(i, k + H)];
    const double2 ev = cadd(w1, w2);
    const double2 o = cmulc(csub(w1, w2), a.tw.get(r + AB * k));
    sbuf[lay.idx(i, k)] = make_double2(ev.x - o.y, ev.y + o.x);
  }
  __syncthreads();
  fft_pass<true>(sbuf, lay, a.inv, twi, SmemSrc<LayRows>{sbuf, lay},
                 RowSink{a.data, base0, base1, r0, r1, a.tw}, tid, nthr);
}

// ---------------------------------------------------------------------------
// Row pass specialised for C = 4096 (forward 16 x 16 x 16, inverse
// 2048 = 8 x 16 x 16 reading the forward stage table): persistent CTAs (one
// per SM, the row pair fills shared memory), the stage table staged once per
// CTA, the next pair's row 1 prefetched into L2 while the current pair
// computes.  Row 0 of the next pair is copied (cp.async.bulk, two 32 KB halves) into
// the upper halves of the two row buffers, which nothing reads after the
// last forward stage, while the current pair's inverse runs in the lower
// halves; the next pair's first stage reads row 0 from there.
constexpr uint32_t kMidStage = 2176;  // padidx(2048): first slot of a row's upper half
struct RowSrcStaged {
  const double2* data;
  const double2* stg;  // staged row 0: e < 2048 at stg[e], else stg[rowstride + e - 2048]
  int64_t base0, base1;
  uint32_t rowstride;
  bool staged;
  __device__ __forceinline__ double2 operator()(uint32_t item, uint32_t e) const {
    if (item == 0 && staged) return stg[e < 2048u ? e : rowstride + e - 2048u];
    return data[(item ? base1 : base0) + e];
  }
};

template <int NTHR>
__device__ __forceinline__ void mid_pair_4096_reg(const MidArgs& a, double2* __restrict__ sbuf,
                                                  const double2* __restrict__ stab,
                                                  double2* __restrict__ qt, uint32_t r0, int tid,
                                                  double2 wct, bool staged, uint32_t phase,
                                                  const double2* next_row0, uint64_t* bar) {
  using Fwd = Sched<16, 16, 16>;
  using Inv = Sched<8, 16, 16>;
  constexpr uint32_t C = 4096;
  const uint32_t AB = a.A * a.B;
  const uint32_t r1 = (AB - r0) % AB;
  // self-paired rows (0 and AB/2): one row, both lane halves on it
  const uint32_t nrows = (r1 == r0) ? 1u : 2u;
  const RowPair lay{padded_len(C) + 4, nrows};
  const int64_t base0 = (int64_t(r0 % a.A) * a.B + (r0 / a.A)) * int64_t(C);
  const int64_t base1 = (int64_t(r1 % a.A) * a.B + (r1 / a.A)) * int64_t(C);
  double2 x[16];
  // forward stages 0 and 1 (half of the CTA per row)
  if (staged && tid < NTHR / 2) mbar_wait(bar, phase);
  ct_load<16, C, NTHR>(x, lay,
                       RowSrcStaged{a.data, sbuf + kMidStage, base0, base1, lay.rowstride, staged}, tid);
  __syncthreads();  // row 1's stores overwrite the staged row's second half
  ct_store<16, false, C, 1, NTHR>(x, lay, stab + a.fwd.toff[0], a.fwd.qmul[0], SmemSink<RowPair>{sbuf, lay}, tid);
  ct_sync<NTHR>(tid);
  ct_load<16, C, NTHR>(x, lay, SmemSrc<RowPair>{sbuf, lay}, tid);
  ct_sync<NTHR>(tid);
  ct_store<16, false, C, 16, NTHR>(x, lay, stab + a.fwd.toff[1], a.fwd.qmul[1], SmemSink<RowPair>{sbuf, lay},
                                   tid);
  __syncthreads();
  // per-pair table of the output twiddles' second factor (RowSinkQ)
  constexpr uint32_t RL = uint32_t(Inv::rad(Inv::nst - 1));
  constexpr uint32_t NSL = Inv::ns(Inv::nst - 1);
  static_assert(2 * RL <= kMidQEntries, "output twiddle table");
  if (uint32_t(tid) < 2 * RL) {
    const uint32_t it = uint32_t(tid) / RL, q = uint32_t(tid) - it * RL;
    const uint32_t xq = 2u * (it ? r1 : r0) * NSL * q;
    qt[tid] = xq ? a.tw.get(xq) : make_double2(1.0, 0.0);
  }
  // forward stage 2 on the lane assignment above
  const int lane = tid & 31, w = tid >> 5;
  const uint32_t row = lane >> 4;
  const uint32_t phys = nrows == 2 ? row : 0u;
  const uint32_t t = row ? 255u - uint32_t(16 * w + (lane & 15)) : uint32_t(16 * w + lane);
#pragma unroll
  for (int q = 0; q < 16; ++q) x[q] = sbuf[lay.idx(phys, t + 256u * uint32_t(q))];
  if (t != 0) {
    const double2* st2 = stab + a.fwd.toff[2];
#pragma unroll
    for (int q = 1; q < 16; ++q) x[q] = cmul(x[q], st2[(uint32_t(q) * a.fwd.qmul[2] - 1) * 256u + t]);
  }
  dft<16, false>(x);
  // spectral product and repack: Y_r[k] for k = t + 256 q, q < 8, into x[q]
  auto spec = [](double2 z1, double2 z2) {
    const double2 p = make_double2(z1.x + z2.x, z1.y - z2.y);
    const double2 q = make_double2(z1.x - z2.x, z1.y + z2.y);
    const double2 pq = cmul(p, q);
    return make_double2(pq.y, -pq.x);  // -i pq, unscaled (see CoefSink)
  };
  auto repack_w = [](double2 w1, double2 w2, double2 tk) {
    const double2 ev = cadd(w1, w2);
    const double2 o = cmulc(csub(w1, w2), tk);
    return make_double2(ev.x - o.y, ev.y + o.x);
  };
  auto shfl2 = [](double2 v) {
    return make_double2(__shfl_xor_sync(0xffffffffu, v.x, 16), __shfl_xor_sync(0xffffffffu, v.y, 16));
  };
  // repack twiddle omega_L^{r + AB k} = omega_L^r omega_C^t omega_16^q
  const double2 tb = cmul(a.tw.get(row ? r1 : r0), wct);
  if (r0 != 0) {
    // partner (same row when self-paired, AB/2): Z_-k-1 = lane ^ 16
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int qb = 7 - q;
      // partner's Z at q' = 15 - q, 7 - q (for Y[q]) and 8 + q, q (for Y[7 - q])
      const double2 p15 = shfl2(x[15 - q]), p7 = shfl2(x[7 - q]);
      const double2 p8 = shfl2(x[8 + q]), p0 = shfl2(x[q]);
      const double2 ya = repack_w(spec(x[q], p15), spec(x[q + 8], p7), w16<false>(tb, q));
      const double2 yb = repack_w(spec(x[qb], p8), spec(x[qb + 8], p0), w16<false>(tb, qb));
      x[q] = ya;
      x[qb] = yb;
    }
  } else {
    // row 0 pairs index k with -k (no borrow): through shared memory
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 16; ++q) sbuf[lay.idx(0, t + 256u * uint32_t(q))] = x[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t k = t + 256u * uint32_t(q);
      const double2 zm = sbuf[lay.idx(0, (C - k) & (C - 1))], zh = sbuf[lay.idx(0, C / 2 - k)];
      x[q] = repack_w(spec(x[q], zm), spec(x[q + 8], zh), w16<false>(tb, q));
    }
  }
  // inverse stage 0 (radix 8, butterfly t, no twiddles): outputs 8 t + q
  dft<8, true>(x);
  __syncthreads();  // every thread has read its forward stage-2 inputs
  if (tid == 0 && next_row0) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar, 2048u * 16u * 2u);
    bulk_g2s(sbuf + kMidStage, next_row0, 2048u * 16u, bar);
    bulk_g2s(sbuf + lay.rowstride + kMidStage, next_row0 + 2048, 2048u * 16u, bar);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) sbuf[lay.idx(phys, 8u * t + uint32_t(q))] = x[q];
  __syncthreads();
  ct_stages<true, Inv, 1, NTHR, SmemSrc<RowPair>, RowSinkQ<RL>, 2>(
      x, sbuf, lay, stab, a.fwd, SmemSrc<RowPair>{sbuf, lay},
      RowSinkQ<RL>{a.data, base0, base1, r0, r1, a.tw, qt}, tid);
}

template <int NTHR>
__device__ __forceinline__ void mid_4096_body(const MidArgs& a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x;
  constexpr uint32_t C = 4096;
  const uint32_t AB = a.A * a.B;
  const uint32_t npairs = AB / 2 + 1;
  double2* stw = sbuf + 2 * (padded_len(C) + 4);
  pdl_trigger();
  for (uint32_t i = tid; i < a.fwd.stablen; i += NTHR) stw[i] = __ldg(a.fwd.stab + i);
  pdl_wait();
  // a new generation for the look-backs after this kernel (this product's
  // carry, the next product's split): they follow it in stream order, the
  // split and the carry of this product that precede it have completed
  if (blockIdx.x == 0 && tid == 0) *a.gen += 1u;
  auto row_base = [&](uint32_t r) {
    return a.data + (int64_t(r % a.A) * a.B + (r / a.A)) * int64_t(C);
  };
  // omega_C^t of this thread's last-forward-stage butterfly (repack twiddles)
  const uint32_t lane = uint32_t(tid) & 31u, wp = uint32_t(tid) >> 5;
  const uint32_t treg = (lane >> 4) ? 255u - (16u * wp + (lane & 15u)) : 16u * wp + lane;
  const double2 wct = treg ? a.tw.get(AB * treg) : make_double2(1.0, 0.0);
  __shared__ __align__(8) uint64_t s_bar;
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    if (blockIdx.x < npairs) {
      prefetch_l2(row_base(blockIdx.x), C * 16);
      prefetch_l2(row_base((AB - blockIdx.x) % AB), C * 16);
    }
  }
  __syncthreads();
  uint32_t it = 0;
  for (uint32_t r0 = blockIdx.x; r0 < npairs; r0 += gridDim.x, ++it) {
    const uint32_t nx = r0 + gridDim.x;
    if (tid == 0 && nx < npairs) prefetch_l2(row_base((AB - nx) % AB), C * 16);
    // row 0 of this pair was staged by the previous one (phase it - 1)
    mid_pair_4096_reg<NTHR>(a, sbuf, stw, stw + C, r0, tid, wct, it > 0, (it - 1) & 1u,
                            nx < npairs ? row_base(nx) : nullptr, &s_bar);
  }
}

__global__ void __launch_bounds__(kMidCtThreads)
k_mid_4096(MidArgs a) {
  mid_4096_body<kMidCtThreads>(a);
}

// ---------------------------------------------------------------------------
// Row pass for the shorter rows of mid-size products (C = 2048, 1024: more
// row pairs, each a fraction of a 4096-point pair's latency).  Forward
// (8|4) x 16 x 16 and inverse (4|2) x 16 x 16 with one butterfly per thread
// and stage (512 threads, half a CTA per row), the inverse reading the
// forward stage table at every second entry; the spectral product and
// repack in shared memory between them, one thread per four slots.
// Persistent over the row pairs.
template <uint32_t M>
__device__ __forceinline__ double2 rot_m(double2 t, int si) {
  // t omega_M^si (forward sign), M in {2, 4, 8}, si < M / ... via omega_8
  const int e = si * int(8 / M);
  return e == 0 ? t : e == 1 ? w8_1<false>(t) : e == 2 ? mul_mi<false>(t) : w8_3<false>(t);
}
template <uint32_t M>
__device__ __forceinline__ double2 rot_m_inv(double2 t, int si) {
  const int e = si * int(8 / M);
  return e == 0 ? t : e == 1 ? w8_1<true>(t) : e == 2 ? mul_mi<true>(t) : w8_3<true>(t);
}

template <uint32_t C, int NTHR, class Fwd, class Inv>
__device__ __forceinline__ void mid_pair_ct(const MidArgs& a, double2* __restrict__ sbuf,
                                            const double2* __restrict__ stab, double2* __restrict__ qt,
                                            uint32_t r0, int tid, double2 wc0, double2 wc1) {
  constexpr uint32_t H = C / 2;
  const uint32_t AB = a.A * a.B;
  const uint32_t r1 = (AB - r0) % AB;
  const uint32_t nrows = (r1 == r0) ? 1 : 2;
  const RowPair lay{padded_len(C) + 4, nrows};
  const int64_t base0 = (int64_t(r0 % a.A) * a.B + (r0 / a.A)) * int64_t(C);
  const int64_t base1 = (int64_t(r1 % a.A) * a.B + (r1 / a.A)) * int64_t(C);
  double2 x[16];
  ct_stages<false, Fwd, 0, NTHR>(x, sbuf, lay, stab, a.fwd, RowSrc{a.data, base0, base1},
                                 SmemSink<RowPair>{sbuf, lay}, tid);
  __syncthreads();
  constexpr uint32_t RL = uint32_t(Inv::rad(Inv::nst - 1));
  constexpr uint32_t NSL = Inv::ns(Inv::nst - 1);
  static_assert(2 * RL <= kMidQEntries, "output twiddle table");
  if (uint32_t(tid) < 2 * RL) {
    const uint32_t it = uint32_t(tid) / RL, q = uint32_t(tid) - it * RL;
    const uint32_t xq = 2u * (it ? r1 : r0) * NSL * q;
    qt[tid] = xq ? a.tw.get(xq) : make_double2(1.0, 0.0);
  }
  auto spec = [&](double2 z1, double2 z2) {
    const double2 p = make_double2(z1.x + z2.x, z1.y - z2.y);
    const double2 q = make_double2(z1.x - z2.x, z1.y + z2.y);
    const double2 pq = cmul(p, q);
    return make_double2(pq.y, -pq.x);  // -i pq, unscaled (see CoefSink)
  };
  auto repack_w = [&](double2 w1, double2 w2, double2 t) {
    const double2 ev = cadd(w1, w2);
    const double2 o = cmulc(csub(w1, w2), t);
    return make_double2(ev.x - o.y, ev.y + o.x);
  };
  if (nrows == 2) {
    // (the pairing and twiddle factorisation of mid_pair_4096_reg's
    // smem form: thread k reads Z0_k, Z0_{k+H}, Z1_{C-1-k}, Z1_{H-1-k} and
    // writes Y0_k, Y1_{H-1-k}; omega_C^{NTHR si} = omega_{C/NTHR}^si)
    static_assert(H % NTHR == 0, "repack twiddle layout");
    const double2 t0 = cmul(a.tw.get(r0), wc0), t1 = cmul(a.tw.get(r1), wc1);
#pragma unroll
    for (int si = 0; si < int(H / NTHR); ++si) {
      const uint32_t k = uint32_t(tid) + NTHR * uint32_t(si);
      const uint32_t kq = H - 1 - k;
      const double2 a0 = sbuf[lay.idx(0, k)], a1 = sbuf[lay.idx(0, k + H)];
      const double2 b0 = sbuf[lay.idx(1, C - 1 - k)], b1 = sbuf[lay.idx(1, kq)];
      const double2 wk = spec(a0, b0), wkh = spec(a1, b1);
      sbuf[lay.idx(0, k)] = repack_w(wk, wkh, rot_m<C / NTHR>(t0, si));
      sbuf[lay.idx(1, kq)] = repack_w(cconj(wkh), cconj(wk), rot_m_inv<C / NTHR>(t1, si));
    }
  } else {
    const uint32_t brw = (r0 != 0) ? 1u : 0u;
    for (uint32_t k = tid; k < C; k += NTHR) {
      const uint32_t kp = (C - k - brw) & (C - 1);
      if (kp < k) continue;
      const double2 w = spec(sbuf[lay.idx(0, k)], sbuf[lay.idx(0, kp)]);
      sbuf[lay.idx(0, k)] = w;
      if (kp != k) sbuf[lay.idx(0, kp)] = cconj(w);
    }
    __syncthreads();
    for (uint32_t k = tid; k < H; k += NTHR)
      sbuf[lay.idx(0, k)] = repack_w(sbuf[lay.idx(0, k)], sbuf[lay.idx(0, k + H)], a.tw.get(r0 + AB * k));
  }
  __syncthreads();
  ct_stages<true, Inv, 0, NTHR, SmemSrc<RowPair>, RowSinkQ<RL>, 2>(
      x, sbuf, lay, stab, a.fwd, SmemSrc<RowPair>{sbuf, lay},
      RowSinkQ<RL>{a.data, base0, base1, r0, r1, a.tw, qt}, tid);
}

template <uint32_t C, class Fwd, class Inv>
__device__ __forceinline__ void mid_ct_body(const MidArgs& a) {
  constexpr int NTHR = kMidCtThreads;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x;
  const uint32_t AB = a.A * a.B;
  const uint32_t npairs = AB / 2 + 1;
  double2* stw = sbuf + 2 * (padded_len(C) + 4);
  pdl_trigger();
  for (uint32_t i = tid; i < a.fwd.stablen; i += NTHR) stw[i] = __ldg(a.fwd.stab + i);
  pdl_wait();
  if (blockIdx.x == 0 && tid == 0) *a.gen += 1u;  // next look-backs' generation
  // omega_C^tid and omega_C^{H-1-tid} (repack twiddles, tid < H)
  const double2 wc0 = tid ? a.tw.get(AB * uint32_t(tid)) : make_double2(1.0, 0.0);
  const double2 wc1 = a.tw.get(AB * (C / 2 - 1 - uint32_t(tid) % (C / 2)));
  __syncthreads();
  for (uint32_t r0 = blockIdx.x; r0 < npairs; r0 += gridDim.x)
    mid_pair_ct<C, NTHR, Fwd, Inv>(a, sbuf, stw, stw + C, r0, tid, wc0, wc1);
}

__global__ void __launch_bounds__(kMidCtThreads)
k_mid_2048(MidArgs a) {
  mid_ct_body<2048, Sched<8, 16, 16>, Sched<4, 16, 16>>(a);
}
__global__ void __launch_bounds__(kMidCtThreads)
k_mid_1024(MidArgs a) {
  mid_ct_body<1024, Sched<4, 16, 16>, Sched<2, 16, 16>>(a);
}

// radices of the compiled row passes' forward schedules (plan.cu builds the
// stage table with them); empty for other lengths
std::vector<int> mid_ct_radices(uint32_t C) {
  if (C == 2048) return {8, 16, 16};
  if (C == 1024) return {4, 16, 16};
  return {};
}

// ---------------------------------------------------------------------------
// The convolution's 1 / (4 L) is applied here, to the inverse transform's
// outputs, and not to the spectrum before it (where FFTW's c2r plan of the
// reference receives it, convolution.cpp:186-192): structured operands (long
// runs of equal limbs, BASELINE config 5) give spectra and partial sums with
// few significant bits, which the unscaled inverse keeps exact; a
// non-dyadic scale on the spectrum makes every one of them round, and the
// roundings add up coherently (2^22 alternating low: 3 -> 1 ulp of the
// largest coefficient).  One rounding against the exact constant (hi + lo).
struct CoefSink {
  double2* coef;
  uint32_t ncols, col0;
  double scale, scale_lo;
  __device__ __forceinline__ void operator()(uint32_t item, uint32_t ma, double2 v) const {
    coef[int64_t(ma) * ncols + col0 + item] =
        make_double2(mul_hl(v.x, scale, scale_lo), mul_hl(v.y, scale, scale_lo));
  }
};

__global__ void __launch_bounds__(512)
k_ilast(ILastArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const uint32_t c = 1u << a.logc;
  const uint32_t col0 = blockIdx.x * c;
  LayCols lay{a.logc, c - 1};
  pdl_trigger();
  const TwStage tw = load_tw_stage(sbuf + padded_len(a.fft.R * c), a.fft, tid, nthr);
  pdl_wait();
  tile_load<kColU>(sbuf, lay, a.fft.R, c, ColSrc{a.data, a.g, 0, col0}, tid, nthr);
  __syncthreads();
  fft_smem_compact<true>(sbuf, lay, a.fft, tw, tid, nthr);
  tile_store<kColU>(sbuf, lay, a.fft.R, c, CoefSink{a.coef, a.g.ncols, col0, a.scale, a.scale_lo}, tid, nthr);
}

__global__ void __launch_bounds__(kColPPThreads, 1)
k_ilast_pp(ILastArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* b0 = reinterpret_cast<double2*>(smem_raw);
  const int tid = threadIdx.x, nthr = blockDim.x;
  const uint32_t c = 1u << a.logc;
  const uint32_t col0 = blockIdx.x * c;
  double2* b1 = b0 + padded_len(a.fft.R * c);
  LayCols lay{a.logc, c - 1};
  tile_load<4>(b0, lay, a.fft.R, c, ColSrc{a.data, a.g, 0, col0}, tid, nthr);
  __syncthreads();
  const double2* res = fft_pp<true>(b0, b1, lay, a.fft, tid, nthr);
  tile_store<4>(res, lay, a.fft.R, c, CoefSink{a.coef, a.g.ncols, col0, a.scale, a.scale_lo}, tid, nthr);
}


size_t colct_smem_bytes(uint32_t R, uint32_t c, uint32_t stablen, uint32_t radl) {
  return size_t(padded_len(R * c)) * 16 + size_t(stablen) * 16 + 2 * size_t(c) * radl * 16;
}

// Both kernels are persistent: a CTA stages the stage table once and walks
// the tiles tile = blockIdx.x + i gridDim.x, prefetching the next tile into
// L2 while the current one computes.  F1's output-twiddle table depends on
// the tile's columns: it is double-buffered by tile parity, so a tile's
// table is written while the previous tile's last stage may still read the
// other one.
template <class SC, int LOGC, int NTHR, int P>
__global__ void __launch_bounds__(NTHR, (NTHR <= 288 ? 2 : 1)) k_f1_ct(F1Args a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  constexpr uint32_t c = 1u << LOGC, R = SC::R;
  constexpr uint32_t RL = ct_last_rad<SC>(), NSL = ct_last_ns<SC>();
  const int tid = threadIdx.x;
  const MapConsts& mc = a.mc;
  const int64_t N = mc.N;
  double2* stab = sbuf + padded_len(R * c);
  double2* qt2 = stab + a.fft.stablen;
  const TwGlobal tw = a.tw;
  const uint32_t ntiles = a.ncols >> LOGC;
  pdl_trigger();
  for (uint32_t i = tid; i < a.fft.stablen; i += NTHR) stab[i] = __ldg(a.fft.stab + i);
  pdl_wait();
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
  const LayCols lay{uint32_t(LOGC), c - 1};
  const uint64_t tile_bytes = uint64_t(a.zt.zrows) * c * 16;
  uint32_t par = 0;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, par ^= 1u) {
    const uint32_t col0 = tile * c;
    const uint32_t nx = tile + gridDim.x;
    if (tid == 0 && nx < ntiles && !a.zt.natural)
      prefetch_l2(a.z + uint64_t(nx) * a.zt.zrows * c, uint32_t(tile_bytes));
    double2* qt = qt2 + par * (c * RL);
    for (uint32_t i = tid; i < c * RL; i += NTHR) {
      const uint32_t it = i / RL, q = i - it * RL;
      const uint32_t x = (col0 + it) * NSL * q;
      qt[i] = x ? tw.get(x) : make_double2(1.0, 0.0);
    }
    double topu = 0.0, topv = 0.0;
    if (mc.mode == kModeHigh && col0 < uint32_t(mc.nfold + mc.lambda)) {
      topu = digit_at(a.u, a.nlimbs, a.b, a.lead, a.count, a.cbits_u, N, mc.balanced != 0);
      topv = digit_at(a.v, a.nlimbs, a.b, a.lead, a.count, a.cbits_v, N, mc.balanced != 0);
    }
    double2 x[P];
    cc_stages<false, SC, 0, LOGC, NTHR, P>(x, sbuf, lay, stab, a.fft,
                                           ZSrc{a.z, a.zt, N, a.ncols, col0, &a.mc, topu, topv},
                                           F1SinkQ<RL>{a.out, a.ncols, col0, tw, qt}, tid);
  }
}

// The tile's raw rows as staged by cp.async: row e, item i at e c + i.
struct RawTileSrc {
  const double2* raw;
  uint32_t logc;
  __device__ __forceinline__ double2 operator()(uint32_t item, uint32_t e) const {
    return raw[(e << logc) + item];
  }
};

// Persistent over the tiles.  A tile's rows (c columns of 16 bytes each)
// arrive by cp.async in the tile's own shared memory, issued once the
// previous tile's last stage has taken its inputs into registers -- the
// buffer is dead from there on -- so the copies fly while that stage
// computes and stores, and the first stage reads shared memory instead of
// waiting on global loads.
template <class SC, int LOGC, int NTHR, int P>
__global__ void __launch_bounds__(NTHR, (NTHR <= 288 ? 2 : 1)) k_ilast_ct(ILastArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  constexpr uint32_t c = 1u << LOGC, R = SC::R;
  const int tid = threadIdx.x;
  double2* stab = sbuf + padded_len(R * c);
  const uint32_t ntiles = a.g.ncols >> LOGC;
  pdl_trigger();
  for (uint32_t i = tid; i < a.fft.stablen; i += NTHR) stab[i] = __ldg(a.fft.stab + i);
  pdl_wait();
  const LayCols lay{uint32_t(LOGC), c - 1};
  auto stage_tile = [&](uint32_t tile) {
    const uint32_t col0 = tile * c;
    for (uint32_t i = tid; i < R * c; i += NTHR)
      cp_async16(sbuf + i, a.data + col_off(a.g, 0, i >> LOGC, col0 + (i & (c - 1))));
    cp_async_commit();
  };
  bool first = true;
  for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint32_t col0 = tile * c;
    const uint32_t nx = tile + gridDim.x;
    auto hook = [&]() {
      if (nx < ntiles) stage_tile(nx);
    };
    const CoefSink sink{a.coef, a.g.ncols, col0, a.scale, a.scale_lo};
    double2 x[P];
    if (first) {
      // the CTA's first tile: straight from global memory (nothing to overlap with)
      first = false;
      cc_stages<true, SC, 0, LOGC, NTHR, P>(x, sbuf, lay, stab, a.fft, ColSrc{a.data, a.g, 0, col0}, sink, tid, hook);
    } else {
      cp_async_wait_all();
      __syncthreads();
      cc_stages<true, SC, 0, LOGC, NTHR, P>(x, sbuf, lay, stab, a.fft, RawTileSrc{sbuf, uint32_t(LOGC)}, sink, tid,
                                            hook);
    }
  }
}

// Middle column passes of three-pass plans (over B, in place) with
// compile-time schedules.  The output twiddle omega_L^{X k}, X = (outer to +
// col tc) tmul, factors like F1's: omega^{X ob} per butterfly (fetched
// before the last DFT) times a per-CTA table omega^{X NS q}.
template <uint32_t RADL>
struct ColSinkQ {
  double2* data;
  ColGeom g;
  int64_t outer;
  uint32_t col0;
  TwGlobal tw;
  uint32_t to, tc, tmul;
  bool inv;
  const double2* qt;
  __device__ __forceinline__ uint32_t X(uint32_t item) const {
    return (uint32_t(outer) * to + (col0 + item) * tc) * tmul;
  }
  __device__ __forceinline__ double2 prep(uint32_t item, uint32_t ob) const {
    const uint32_t x = X(item) * ob;
    return x ? tw.get(x) : make_double2(1.0, 0.0);
  }
  __device__ __forceinline__ void put(uint32_t item, uint32_t k, uint32_t q, double2 v,
                                      double2 b) const {
    const double2 w = cmul(b, qt[item * RADL + q]);
    data[col_off(g, outer, k, col0 + item)] = inv ? cmulc(v, w) : cmul(v, w);
  }
};
template <uint32_t RADL>
struct SinkPrep<ColSinkQ<RADL>> {
  static constexpr bool value = true;
};

template <class SC, int LOGC, int NTHR, int P>
__global__ void __launch_bounds__(NTHR, (NTHR <= 288 ? 2 : 1)) k_col_ct(ColArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sbuf = reinterpret_cast<double2*>(smem_raw);
  constexpr uint32_t c = 1u << LOGC, R = SC::R;
  constexpr uint32_t RL = ct_last_rad<SC>(), NSL = ct_last_ns<SC>();
  const int tid = threadIdx.x;
  const uint32_t col0 = blockIdx.x * c;
  const int64_t outer = blockIdx.y;
  double2* stab = sbuf + padded_len(R * c);
  double2* qt = stab + a.fft.stablen;
  pdl_trigger();
  for (uint32_t i = tid; i < a.fft.stablen; i += NTHR) stab[i] = __ldg(a.fft.stab + i);
  const ColSinkQ<RL> sink{a.data, a.g, outer, col0, a.tw, a.to, a.tc, a.tmul, a.inv != 0, qt};
  for (uint32_t i = tid; i < c * RL; i += NTHR) {
    const uint32_t it = i / RL, q = i - it * RL;
    const uint32_t x = sink.X(it) * NSL * q;
    qt[i] = x ? a.tw.get(x) : make_double2(1.0, 0.0);
  }
  pdl_wait();
  const LayCols lay{uint32_t(LOGC), c - 1};
  double2 x[P];
  if (a.inv)
    cc_stages<true, SC, 0, LOGC, NTHR, P>(x, sbuf, lay, stab, a.fft, ColSrc{a.data, a.g, outer, col0},
                                          sink, tid);
  else
    cc_stages<false, SC, 0, LOGC, NTHR, P>(x, sbuf, lay, stab, a.fft,
                                           ColSrc{a.data, a.g, outer, col0}, sink, tid);
}

// Compiled column shapes: {R, radices (maxrad 16 schedule), LOGC, NTHR}.
#define TMG_COLCT(R_, LOGC_, NTHR_, P_, USES_, ...)                                       \
  {R_, LOGC_, NTHR_, USES_, {__VA_ARGS__}, k_f1_ct<Sched<__VA_ARGS__>, LOGC_, NTHR_, P_>, \
   k_ilast_ct<Sched<__VA_ARGS__>, LOGC_, NTHR_, P_>,                                     \
   k_col_ct<Sched<__VA_ARGS__>, LOGC_, NTHR_, P_>, ct_last_rad<Sched<__VA_ARGS__>>()}
// Shapes serve passes by `uses`: 1 = F1, 2 = ilast, 4 = the middle (B)
// column passes of three-pass plans.
// (A radix-8, 1024-thread instantiation of 1792 = 8 x 8 x 4 x 7 measured
// 86.6 / 47.7 us against 84.5 / 45.5 us for the 16 x 16 x 7 one; a
// 560-thread one of 1400 equal at 96 registers.)  The first shape of a
// length that serves a pass (uses: 1 = F1, 2 = ilast) is the one used; the
// composite radices 10 and 12 (prime-factor DFTs, dft.cuh) give
// three-stage schedules for 1728 = 12^3 and 1440 = 12 x 12 x 10, one
// butterfly per thread and stage.  Measured at 2^26: two columns per CTA
// (two CTAs per SM) suit F1 of 1440 (66 -> 62 us) but not ilast (35 -> 39)
// nor the full product, whose split writes z in F1's tile order (zgen
// 29 -> 33 us with two columns).
static const ColCtShape kColCtShapes[] = {
    TMG_COLCT(1728, 2, 576, 12, 3, 12, 12, 12),
    TMG_COLCT(1440, 1, 288, 12, 1, 12, 12, 10),
    TMG_COLCT(1440, 2, 576, 12, 3, 12, 12, 10),
    TMG_COLCT(1792, 2, 512, 16, 3, 16, 16, 7),
    TMG_COLCT(1400, 2, 512, 16, 3, 8, 5, 5, 7),
    TMG_COLCT(1792, 1, 256, 16, 0, 16, 16, 7),
    TMG_COLCT(1400, 1, 256, 16, 0, 8, 5, 5, 7),
    TMG_COLCT(1728, 1, 288, 12, 0, 12, 12, 12),
    // 2^24 (BASELINE config 2): 448 x 4096 full, 320 x 4096 low/high
    TMG_COLCT(448, 4, 512, 16, 3, 16, 4, 7),
    TMG_COLCT(320, 4, 512, 16, 3, 16, 5, 4),
    TMG_COLCT(112, 5, 256, 16, 7, 16, 7),  // 2^22 full
    // three-pass plans (2^28): A x B columns around the 4096-point rows
    TMG_COLCT(64, 6, 256, 16, 7, 16, 4),
    TMG_COLCT(80, 5, 256, 16, 7, 16, 5),
    TMG_COLCT(128, 5, 256, 16, 7, 16, 8),
    TMG_COLCT(70, 5, 256, 16, 7, 14, 5),
};
#undef TMG_COLCT

const ColCtShape* colct_for(uint32_t R, int role) {
  for (const ColCtShape& sh : kColCtShapes)
    if (sh.R == R && (sh.uses & role) != 0) return &sh;
  return nullptr;
}

int colct_stages(uint32_t R) {
  const ColCtShape* sh = colct_for(R, 1);
  if (!sh) return 0;
  int n = 0;
  while (n < 4 && sh->rad[n]) ++n;
  return n;
}

// ---------------------------------------------------------------------------
// Post-map, rounding and carry propagation over all limbs.
//   phase 1  coefficients e_k of the block's lanes: post-map (once per
//            coefficient; the high product's folded buffer is staged in
//            shared memory so the differencing reads neighbours from there)
//            and the rounding tripwire
//   phase 2  lanes L_m = sum e_k << (kb - 64m), one limb per thread pass
//   phase 3  per-thread runs of 4 limbs: s_m = lo(L_m) + hi(L_{m-1}),
//            carry transfer functions, block scan, warp look-back, limbs
__global__ void __launch_bounds__(kCarryThreads)
k_carry(CarryArgs a) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t sw[32];
  __shared__ uint32_t s_blk;
  __shared__ int s_cin;
  __shared__ double s_psi;
  __shared__ uint32_t s_flags, s_low;
  const int tid = threadIdx.x;
  const MapConsts& mc = a.mc;
  const int b = mc.b;
  if (tid == 0) {
    s_blk = take_ticket(a.scan.ctr);
    s_flags = 0;
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

  // coefficient window of the lanes ms-1 .. me (inclusive)
  const int64_t klo = (ms == 0) ? 0 : (64 * (ms - 1) + b - 1) / b;
  int64_t khi = (64 * (me + 1) + b - 1) / b;
  if (khi > K) khi = K;
  const int64_t nk = khi > klo ? khi - klo : 0;
  long long* se = reinterpret_cast<long long*>(smem_raw);                        // nk + 1
  double* sh = reinterpret_cast<double*>(se + nk + 1);                            // nk + 2
  double* sww = sh + nk + 2;                                                      // nk + 12
  unsigned long long* slo = reinterpret_cast<unsigned long long*>(sww + nk + 12); // LB + 2
  long long* shi = reinterpret_cast<long long*>(slo + LB + 2);                    // LB + 2

  // stage the convolution coefficients under this block (coalesced); the
  // post-maps read their lambda-neighbourhoods from shared memory
  const int64_t nwt = (mc.mode == kModeFull) ? K : mc.N;
  const int64_t wlo = max(int64_t(0), klo - int64_t(mc.lambda) - 2);
  const int64_t whi = min(nwt, khi + 2);
  const int64_t nw = (mc.mode == kModeFull || whi <= wlo) ? 0 : whi - wlo;
  for (int64_t j = wlo + tid; j < wlo + nw; j += kCarryThreads) sww[j - wlo] = W(j);
  auto WS = [&](int64_t j) -> double {
    const int64_t o = j - wlo;
    return (o >= 0 && o < nw) ? sww[o] : __ldg(gw + j);
  };

  if (mc.mode == kModeHigh && tid == 0) s_psi = high_psi(mc, W, a.aux[0]);
  RoundAcc ra;
  uint32_t flags = 0;
  long long c0v = 0;
  __syncthreads();
  if (mc.mode == kModeLow && ms == 0) {
    c0v = ra.round(postmap_low(mc, WS, 0));
    if (c0v & ((1ll << b) - 1)) flags |= kFlagLowNotDivisible;
  }
  if (mc.mode == kModeHigh) {
    // folded delta-dagger buffer for i in [klo - 1, khi)
    for (int64_t i = klo - 1 + tid; i < khi; i += kCarryThreads)
      sh[i - (klo - 1)] = (i >= 0 && i < mc.N) ? high_buf(mc, WS, i) : 0.0;
    __syncthreads();
  }
  const double psi = s_psi;
  for (int64_t k = klo + tid; k < khi; k += kCarryThreads) {
    double x;
    if (mc.mode == kModeFull) {
      x = W(k);
    } else if (mc.mode == kModeLow) {
      x = postmap_low(mc, WS, k + 1);
    } else {
      const int64_t N = mc.N;
      const double hk = (k < N) ? sh[k - (klo - 1)] : 0.0;
      const double hm = (k >= 1) ? sh[k - 1 - (klo - 1)] : 0.0;
      double v;
      if (k == N) v = psi - hm * mc.step;
      else if (k == 0) v = hk;
      else v = hk - hm * mc.step;
      if (k < mc.nfold) v -= psi * mc.fold[k];
      x = v * mc.scale_out;
    }
    long long e = ra.round(x);
    if (mc.mode == kModeLow && k == 0) e += (c0v >> b);
    se[k - klo] = e;
  }
  __syncthreads();
  flags |= ra.all_flags();
  {
    const double e = warp_max_nonneg(ra.max_err), m = warp_max_nonneg(ra.max_abs);
    if ((tid & 31) == 0) status_merge(a.status, e, m, 0);
  }

  // phase 2: lanes of limbs ms-1 .. me
  auto E = [&](int64_t k) -> long long { return se[k - klo]; };
  for (int64_t m = ms - 1 + tid; m <= me; m += kCarryThreads) {
    const __int128 L = (m < 0) ? (__int128)0 : lane_value(E, m, b, khi);
    slo[m - (ms - 1)] = (unsigned long long)L;
    shi[m - (ms - 1)] = (long long)(L >> 64);
  }
  __syncthreads();

  // phase 3: carries
  const int64_t m0 = ms + int64_t(tid) * kCarryPerThread;
  const int64_t m1 = min(me, m0 + kCarryPerThread);
  auto S = [&](int64_t m) -> __int128 {
    const int64_t o = m - (ms - 1);
    return (__int128)slo[o] + (__int128)shi[o - 1];
  };
  uint32_t f = kTfIdentity;
  for (int64_t m = m0; m < m1; ++m) f = tf_compose(f, limb_tf(S(m), flags));
  uint32_t agg;
  const uint32_t ex = block_scan_tf(f, sw, &agg);
  if (tid < 32) {
    const int cin = lookback_warp(a.scan.state, blk, agg, a.scan.epoch, 0);
    if (tid == 0) s_cin = cin;
  }
  __syncthreads();
  int c = tf_apply(ex, s_cin);
  const int64_t OL = a.out_limbs;
  const int64_t sb = a.shift_s - 1;  // high: bit s-1
  uint32_t sticky = 0;
  for (int64_t m = m0; m < m1; ++m) {
    const __int128 s = S(m);
    const uint32_t tfm = limb_tf(s, flags);
    const uint64_t x = (unsigned long long)(s + c);
    c = tf_apply(tfm, c);
    if (mc.mode == kModeFull) {
      const int64_t nb2 = 2 * a.n;
      if (m < OL) {
        if (m == OL - 1 && (nb2 & 63) && (x >> (nb2 & 63))) flags |= kFlagFullOverflow;
        a.out[m] = x;
      } else if (x) {
        flags |= kFlagFullOverflow;
      }
    } else if (mc.mode == kModeLow) {
      if (m < OL) a.out[m] = (m == OL - 1 && (a.n & 63)) ? (x & ((1ull << (a.n & 63)) - 1)) : x;
    } else {
      a.tbuf[m] = x;
      const int64_t bit0 = 64 * m;
      if (bit0 + 64 <= sb) {
        if (x) sticky = 1;
      } else if (bit0 < sb) {
        if (x & ((1ull << (sb - bit0)) - 1)) sticky = 1;
      }
    }
  }
  if (m1 == me && m0 < m1 && me == a.ML && c < 0) {
    // sign of the recombined value (carry out of the top limb)
    if (mc.mode == kModeFull) flags |= kFlagNegative;
    if (mc.mode == kModeHigh) flags |= kFlagHighRange;
  }
  if (sticky) atomicOr(&s_low, 1u);
  if (flags) atomicOr(&s_flags, flags);
  __syncthreads();
  if (tid == 0) {
    if (s_flags) atomicOr(&a.status->flags, s_flags);
    if (s_low) atomicOr(&a.status->high_sticky, 1u);
    release_ticket(a.scan.ctr, gridDim.x);
  }
}

size_t carry_smem(int b) {
  constexpr int LB = kCarryThreads * kCarryPerThread;
  const size_t nk = size_t((64 * (LB + 2) + b - 1) / b + 4);
  return nk * 8 + (nk + 2) * 8 + (nk + 12) * 8 + size_t(2 * (LB + 2)) * 8 + 64;
}

// ---------------------------------------------------------------------------
// High product rounding (products_f64.cpp:162-166): w = round_even(t / 2^s)
// = (t >> s) + inc, inc = bit_{s-1}(t) & (sticky_{<s-1} | bit_s(t)).  The
// increment ripples through all-ones limbs of t >> s: a second carry scan
// with the increment as the carry into limb 0.  Then the range test
// 0 <= w <= 2^n.
// Limb m of t >> s (t in tbuf, ML limbs).
__device__ __forceinline__ uint64_t high_shifted(const HighRoundArgs& a, int64_t m) {
  const int64_t q = int64_t(a.shift_s) >> 6;
  const int r = int(a.shift_s & 63);
  const uint64_t lo = (m + q < a.ML) ? a.tbuf[m + q] : 0ull;
  const uint64_t hi = (m + q + 1 < a.ML) ? a.tbuf[m + q + 1] : 0ull;
  return r ? ((lo >> r) | (hi << (64 - r))) : lo;
}

// The first limb of w0 = t >> s that is not all ones (atomicMin into
// ticket[1]): the limb that stops the rounding increment.  The two-kernel
// carry path computes it in k_carry_lanes / k_carry_patch; this kernel serves the
// single-pass k_carry path.
__global__ void __launch_bounds__(kCarryThreads)
k_high_agg(HighRoundArgs a) {
  pdl_trigger();
  pdl_wait();
  constexpr int LB = kCarryThreads * kHighPerThread;
  const int64_t ms = int64_t(blockIdx.x) * LB;
  const int64_t me = min(a.WL, ms + LB);
  uint32_t first = 0xffffffffu;
  for (int64_t m = ms + threadIdx.x; m < me; m += kCarryThreads)
    if (high_shifted(a, m) != ~0ull) first = min(first, uint32_t(m));
  first = __reduce_min_sync(0xffffffffu, first);
  if ((threadIdx.x & 31) == 0 && first != 0xffffffffu) atomicMin(a.ticket + 1, first);
}

// w = w0 + inc: the increment enters limb 0 and carries through the all-ones
// limbs below the first stopping limb f (k_high_agg / k_carry_lanes + k_carry_patch), so
// limb j adds inc exactly when j <= f.
__global__ void __launch_bounds__(kCarryThreads)
k_high_round(HighRoundArgs a) {
  pdl_trigger();
  pdl_wait();
  __shared__ uint32_t s_flags, s_top, s_low;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_flags = 0;
    s_top = 0;
    s_low = 0;
  }
  __syncthreads();
  const uint32_t blk = blockIdx.x;
  const int64_t s = a.shift_s;
  const int64_t q = s >> 6;
  const int r = int(s & 63);
  const uint64_t* t = a.tbuf;
  auto tl = [&](int64_t m) -> uint64_t { return m < a.ML ? t[m] : 0ull; };
  const int inc = int((tl((s - 1) >> 6) >> ((s - 1) & 63)) & 1) &
                  int(a.status->high_sticky != 0 || ((tl(s >> 6) >> (s & 63)) & 1));
  const uint32_t first = __ldcg(a.ticket + 1);
  constexpr int LB = kCarryThreads * kHighPerThread;
  const int64_t ms = int64_t(blk) * LB;
  const int64_t me = min(a.WL, ms + LB);
  uint32_t flags = 0, topbit = 0, lownz = 0;
  const int64_t OL = a.out_limbs;
  // Blocks whose limbs all lie below bit n, inside t and below the last
  // output limb (block-uniform; all but the top block): no bounds or range
  // tests per limb, 32-bit indices, the upper word from the neighbouring lane.
  if (me == ms + LB && me + q + 1 <= a.ML && 64 * me <= a.n && me <= OL - 1 && a.ML < (int64_t(1) << 31)) {
    const uint64_t* tq = t + q + ms;
    uint64_t* op = a.out + ms;
    uint64_t lo[kHighPerThread];
#pragma unroll
    for (int i = 0; i < kHighPerThread; ++i) lo[i] = tq[tid + i * kCarryThreads];
    const uint32_t f0 = first >= uint32_t(ms) ? first - uint32_t(ms) : 0u;  // limbs ms + j <= first: j <= f0
    const bool anyinc = inc && uint64_t(first) >= uint64_t(ms);
    uint64_t nz = 0;
#pragma unroll
    for (int i = 0; i < kHighPerThread; ++i) {
      const uint32_t j = uint32_t(tid) + uint32_t(i) * kCarryThreads;
      uint64_t hi = __shfl_down_sync(0xffffffffu, lo[i], 1);
      if ((tid & 31) == 31) hi = tq[j + 1];
      const uint64_t w0 = r ? ((lo[i] >> r) | (hi << (64 - r))) : lo[i];
      const uint64_t x = w0 + uint64_t((anyinc && j <= f0) ? 1 : 0);
      nz |= x;
      op[j] = x;
    }
    if (nz) atomicOr(&s_low, 1u);
  } else {
  uint64_t tlo[kHighPerThread], thi[kHighPerThread];
#pragma unroll
  for (int i = 0; i < kHighPerThread; ++i) {
    const int64_t m = ms + tid + int64_t(i) * kCarryThreads;
    tlo[i] = (m < me) ? tl(m + q) : 0ull;
    thi[i] = (m < me) ? tl(m + q + 1) : 0ull;
  }
#pragma unroll
  for (int i = 0; i < kHighPerThread; ++i) {
    const int64_t m = ms + tid + int64_t(i) * kCarryThreads;
    if (m < me) {
      const uint64_t lo = tlo[i], hi = thi[i];
      const uint64_t w0 = r ? ((lo >> r) | (hi << (64 - r))) : lo;
      const uint64_t x = w0 + uint64_t((inc && uint64_t(m) <= uint64_t(first)) ? 1 : 0);
      // the increment carried out of the top examined limb: w > 2^n
      if (inc && m == a.WL - 1 && uint64_t(first) >= uint64_t(a.WL)) flags |= kFlagHighRange;
      high_classify(x, m, a.n, topbit, lownz, flags);
      if (m < OL) a.out[m] = x & high_mask(m, OL, a.n);
    }
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
    // the last block settles this product's range test (w in [0, 2^n]) and
    // clears the high-product words for the next product on the stream
    __threadfence();
    if (atomicAdd(a.ticket, 1u) == gridDim.x - 1) {
      __threadfence();
      volatile DevStatus* st = a.status;
      if (st->high_topbit && st->high_lownz) atomicOr(&a.status->flags, uint32_t(kFlagHighRange));
      st->high_topbit = 0;
      st->high_lownz = 0;
      st->high_sticky = 0;
      a.ticket[1] = 0xffffffffu;  // first stopping limb, for the next product
      *a.ticket = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// One batched product's status (its own word): the device flag word goes to
// flag_out (the batched API's per-product flags) and the status merges into
// the context's (residuals by max, flags by or).
__global__ void k_status_publish(const DevStatus* src, uint32_t* flag_out, DevStatus* merge) {
  pdl_trigger();
  pdl_wait();
  uint32_t f = src->flags;
  if (src->high_topbit && src->high_lownz) f |= kFlagHighRange;
  if (flag_out) *flag_out = f;
  if (merge) {
    atomicMax(&merge->max_err_bits, src->max_err_bits);
    atomicMax(&merge->max_abs_bits, src->max_abs_bits);
    if (f) atomicOr(&merge->flags, f);
  }
}

}  // namespace tmg
