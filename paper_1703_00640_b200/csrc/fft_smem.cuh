// Batched mixed-radix Stockham FFT on shared memory (FP64).
//
// Each stage of radix r reads r strided values per butterfly into registers,
// applies the inter-stage twiddles omega_{Ns r}^{j q} (read from an exact
// twiddle table, no recurrences: the float budget of the reference leaves
// no room for twiddle drift), runs the r-point DFT in registers and writes
// the outputs in autosorted (natural) order.  All loads of a stage complete
// before any store (two barriers), so a single buffer suffices.
//
// This is the device replacement for the FFTW r2c/c2r plans of
// convolution.cpp:92-129.
#pragma once

#include "common.cuh"
#include "dft.cuh"

namespace tmg {

constexpr int kMaxStages = 8;

// Per sub-length plan, built on the host (plan.cu) and passed by value.
struct SubFft {
  uint32_t R;          // transform length
  int32_t nst;         // number of radix stages
  int32_t rad[kMaxStages];
  uint32_t Ns[kMaxStages];      // product of previous radices
  uint32_t twstep[kMaxStages];  // R / (Ns * rad)
  FastDiv fdNs[kMaxStages];
  const double2* tw;  // omega_R^x, x in [0, R), forward sign
};

__device__ __forceinline__ uint32_t padidx(uint32_t i) { return i + (i >> 4); }
__host__ __device__ inline uint32_t padded_len(uint32_t n) {
  return n + (n >> 4) + 1;
}

// Column layout: element (item=column, e=row) at pad(e * ncols + col).
struct LayCols {
  uint32_t lognitems, itemmask;
  __device__ __forceinline__ uint32_t idx(uint32_t item, uint32_t e) const {
    return padidx((e << lognitems) + item);
  }
  __device__ __forceinline__ void split(uint32_t bf, uint32_t /*nbf_item*/,
                                        uint32_t& item, uint32_t& t) const {
    item = bf & itemmask;
    t = bf >> lognitems;
  }
  __device__ __forceinline__ uint32_t nitems() const { return 1u << lognitems; }
};

// Row layout: element (item, e) at item * rowstride + pad(e); at most a few
// items, butterflies of one item are contiguous in bf.
struct LayRows {
  uint32_t nit, rowstride;
  __device__ __forceinline__ uint32_t idx(uint32_t item, uint32_t e) const {
    return item * rowstride + padidx(e);
  }
  __device__ __forceinline__ void split(uint32_t bf, uint32_t nbf_item,
                                        uint32_t& item, uint32_t& t) const {
    item = 0;
    t = bf;
    while (t >= nbf_item) {
      t -= nbf_item;
      ++item;
    }
  }
  __device__ __forceinline__ uint32_t nitems() const { return nit; }
};

constexpr int kXMax = 21;  // max values a thread holds across a barrier

template <int RAD, class Lay>
__device__ __forceinline__ void stage_load(double2 (&x)[kXMax],
                                           const double2* __restrict__ buf,
                                           const Lay& lay, uint32_t R, int tid,
                                           int nthr) {
  constexpr int NB = (16 + RAD - 1) / RAD;
  const uint32_t nbf_item = R / RAD;
  const uint32_t nbf = nbf_item * lay.nitems();
#pragma unroll
  for (int it = 0; it < NB; ++it) {
    uint32_t bf = tid + it * nthr;
    if (bf < nbf) {
      uint32_t item, t;
      lay.split(bf, nbf_item, item, t);
#pragma unroll
      for (int q = 0; q < RAD; ++q) x[it * RAD + q] = buf[lay.idx(item, t + q * nbf_item)];
    }
  }
}

template <int RAD, bool INV, class Lay>
__device__ __forceinline__ void stage_store(double2 (&x)[kXMax],
                                            double2* __restrict__ buf,
                                            const Lay& lay, uint32_t R,
                                            uint32_t Ns, const FastDiv& fdNs,
                                            uint32_t twstep,
                                            const double2* __restrict__ tw,
                                            int tid, int nthr) {
  constexpr int NB = (16 + RAD - 1) / RAD;
  const uint32_t nbf_item = R / RAD;
  const uint32_t nbf = nbf_item * lay.nitems();
#pragma unroll
  for (int it = 0; it < NB; ++it) {
    uint32_t bf = tid + it * nthr;
    if (bf < nbf) {
      uint32_t item, t;
      lay.split(bf, nbf_item, item, t);
      uint32_t tq = fdiv(t, fdNs);
      uint32_t j = t - tq * Ns;
      double2* xv = x + it * RAD;
      if (j != 0) {
        uint32_t step = j * twstep;
#pragma unroll
        for (int q = 1; q < RAD; ++q) {
          double2 w = __ldg(tw + step * q);
          xv[q] = INV ? cmulc(xv[q], w) : cmul(xv[q], w);
        }
      }
      dft<RAD, INV>(xv);
      uint32_t ob = tq * Ns * RAD + j;
#pragma unroll
      for (int q = 0; q < RAD; ++q) buf[lay.idx(item, ob + q * Ns)] = xv[q];
    }
  }
}

// Full transform of all items (in place, natural order in and out).  The
// register block x is shared by every radix so that the stage dispatch does
// not multiply register pressure.
template <bool INV, class Lay>
__device__ __forceinline__ void fft_smem(double2* __restrict__ buf, const Lay& lay,
                                         const SubFft& p, int tid, int nthr) {
  double2 x[kXMax];
  for (int s = 0; s < p.nst; ++s) {
    const int rad = p.rad[s];
    switch (rad) {
      case 16: stage_load<16>(x, buf, lay, p.R, tid, nthr); break;
      case 8: stage_load<8>(x, buf, lay, p.R, tid, nthr); break;
      case 4: stage_load<4>(x, buf, lay, p.R, tid, nthr); break;
      case 2: stage_load<2>(x, buf, lay, p.R, tid, nthr); break;
      case 3: stage_load<3>(x, buf, lay, p.R, tid, nthr); break;
      case 5: stage_load<5>(x, buf, lay, p.R, tid, nthr); break;
      default: stage_load<7>(x, buf, lay, p.R, tid, nthr); break;
    }
    __syncthreads();
    const uint32_t Ns = p.Ns[s];
    const uint32_t ts = p.twstep[s];
    const FastDiv fd = p.fdNs[s];
    switch (rad) {
      case 16: stage_store<16, INV>(x, buf, lay, p.R, Ns, fd, ts, p.tw, tid, nthr); break;
      case 8: stage_store<8, INV>(x, buf, lay, p.R, Ns, fd, ts, p.tw, tid, nthr); break;
      case 4: stage_store<4, INV>(x, buf, lay, p.R, Ns, fd, ts, p.tw, tid, nthr); break;
      case 2: stage_store<2, INV>(x, buf, lay, p.R, Ns, fd, ts, p.tw, tid, nthr); break;
      case 3: stage_store<3, INV>(x, buf, lay, p.R, Ns, fd, ts, p.tw, tid, nthr); break;
      case 5: stage_store<5, INV>(x, buf, lay, p.R, Ns, fd, ts, p.tw, tid, nthr); break;
      default: stage_store<7, INV>(x, buf, lay, p.R, Ns, fd, ts, p.tw, tid, nthr); break;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Pass driver with external source and sink: the first stage reads its
// butterfly inputs straight from src(item, e) (global memory: every thread
// issues all of its loads before the first use), the last stage hands its
// outputs to sink(item, k, value) (global memory with the inter-pass
// twiddle).  Intermediate stages exchange through shared memory.  With a
// single stage no shared memory is touched.

template <int RAD, class Lay, class Src>
__device__ __forceinline__ void stage_load_src(double2 (&x)[kXMax], const Lay& lay,
                                               uint32_t R, const Src& src, int tid,
                                               int nthr) {
  constexpr int NB = (16 + RAD - 1) / RAD;
  const uint32_t nbf_item = R / RAD;
  const uint32_t nbf = nbf_item * lay.nitems();
#pragma unroll
  for (int it = 0; it < NB; ++it) {
    uint32_t bf = tid + it * nthr;
    if (bf < nbf) {
      uint32_t item, t;
      lay.split(bf, nbf_item, item, t);
#pragma unroll
      for (int q = 0; q < RAD; ++q) x[it * RAD + q] = src(item, t + q * nbf_item);
    }
  }
}

template <int RAD, bool INV, class Lay, class Sink>
__device__ __forceinline__ void stage_store_sink(double2 (&x)[kXMax], const Lay& lay,
                                                 uint32_t R, uint32_t Ns,
                                                 const FastDiv& fdNs, uint32_t twstep,
                                                 const double2* __restrict__ tw,
                                                 const Sink& sink, int tid, int nthr) {
  constexpr int NB = (16 + RAD - 1) / RAD;
  const uint32_t nbf_item = R / RAD;
  const uint32_t nbf = nbf_item * lay.nitems();
#pragma unroll
  for (int it = 0; it < NB; ++it) {
    uint32_t bf = tid + it * nthr;
    if (bf < nbf) {
      uint32_t item, t;
      lay.split(bf, nbf_item, item, t);
      uint32_t tq = fdiv(t, fdNs);
      uint32_t j = t - tq * Ns;
      double2* xv = x + it * RAD;
      if (j != 0) {
        uint32_t step = j * twstep;
#pragma unroll
        for (int q = 1; q < RAD; ++q) {
          double2 w = __ldg(tw + step * q);
          xv[q] = INV ? cmulc(xv[q], w) : cmul(xv[q], w);
        }
      }
      dft<RAD, INV>(xv);
      uint32_t ob = tq * Ns * RAD + j;
#pragma unroll
      for (int q = 0; q < RAD; ++q) sink(item, ob + q * Ns, xv[q]);
    }
  }
}

#define TMG_RADIX_SWITCH(rad, CALL) \
  switch (rad) {                    \
    case 16: CALL(16); break;       \
    case 8: CALL(8); break;         \
    case 4: CALL(4); break;         \
    case 2: CALL(2); break;         \
    case 3: CALL(3); break;         \
    case 5: CALL(5); break;         \
    default: CALL(7); break;        \
  }

template <bool INV, class Lay, class Src, class Sink>
__device__ __forceinline__ void fft_pass(double2* __restrict__ buf, const Lay& lay,
                                         const SubFft& p, const Src& src,
                                         const Sink& sink, int tid, int nthr) {
  double2 x[kXMax];
  const int last = p.nst - 1;
  {
    const int rad = p.rad[0];
#define TMG_L0(RR) stage_load_src<RR>(x, lay, p.R, src, tid, nthr)
    TMG_RADIX_SWITCH(rad, TMG_L0)
#undef TMG_L0
    __syncthreads();  // src may alias buf
    const FastDiv fd = p.fdNs[0];
    if (last == 0) {
#define TMG_S0(RR) stage_store_sink<RR, INV>(x, lay, p.R, 1u, fd, p.twstep[0], p.tw, sink, tid, nthr)
      TMG_RADIX_SWITCH(rad, TMG_S0)
#undef TMG_S0
      return;
    }
#define TMG_S0B(RR) stage_store<RR, INV>(x, buf, lay, p.R, 1u, fd, p.twstep[0], p.tw, tid, nthr)
    TMG_RADIX_SWITCH(rad, TMG_S0B)
#undef TMG_S0B
    __syncthreads();
  }
  for (int s = 1; s < last; ++s) {
    const int rad = p.rad[s];
#define TMG_LM(RR) stage_load<RR>(x, buf, lay, p.R, tid, nthr)
    TMG_RADIX_SWITCH(rad, TMG_LM)
#undef TMG_LM
    __syncthreads();
    const uint32_t Ns = p.Ns[s];
    const uint32_t ts = p.twstep[s];
    const FastDiv fd = p.fdNs[s];
#define TMG_SM(RR) stage_store<RR, INV>(x, buf, lay, p.R, Ns, fd, ts, p.tw, tid, nthr)
    TMG_RADIX_SWITCH(rad, TMG_SM)
#undef TMG_SM
    __syncthreads();
  }
  {
    const int rad = p.rad[last];
#define TMG_LL(RR) stage_load<RR>(x, buf, lay, p.R, tid, nthr)
    TMG_RADIX_SWITCH(rad, TMG_LL)
#undef TMG_LL
    __syncthreads();  // sink may alias buf
    const uint32_t Ns = p.Ns[last];
    const uint32_t ts = p.twstep[last];
    const FastDiv fd = p.fdNs[last];
#define TMG_SL(RR) stage_store_sink<RR, INV>(x, lay, p.R, Ns, fd, ts, p.tw, sink, tid, nthr)
    TMG_RADIX_SWITCH(rad, TMG_SL)
#undef TMG_SL
  }
}

// Shared-memory source and sink for fft_pass.
template <class Lay>
struct SmemSrc {
  const double2* buf;
  Lay lay;
  __device__ __forceinline__ double2 operator()(uint32_t item, uint32_t e) const {
    return buf[lay.idx(item, e)];
  }
};
template <class Lay>
struct SmemSink {
  double2* buf;
  Lay lay;
  __device__ __forceinline__ void operator()(uint32_t item, uint32_t k, double2 v) const {
    buf[lay.idx(item, k)] = v;
  }
};

// Global twiddle omega_L^x for x < L from a two-level table:
// omega^x = hi[x >> S] * lo[x & (2^S - 1)].
struct TwGlobal {
  const double2* lo;
  const double2* hi;
  uint32_t S;
  __device__ __forceinline__ double2 get(uint32_t x) const {
    double2 a = __ldg(hi + (x >> S));
    double2 b = __ldg(lo + (x & ((1u << S) - 1)));
    return cmul(a, b);
  }
};

}  // namespace tmg
