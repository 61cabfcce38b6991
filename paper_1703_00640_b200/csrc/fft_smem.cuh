// Batched mixed-radix Stockham FFT passes on shared memory (FP64).
//
// Each stage of radix r reads r strided values per butterfly into registers,
// applies the inter-stage twiddles omega_{Ns r}^{j q}, runs the r-point DFT
// in registers and writes the outputs in autosorted (natural) order.  All
// loads of a stage complete before any store (two barriers), so a single
// buffer suffices.  Twiddles come from exact tables (no recurrences: the
// float budget of the reference leaves no room for twiddle drift), staged in
// shared memory as a two-level table omega^x = hi[x >> 6] * lo[x & 63].
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
  uint32_t twstep[kMaxStages];  // (R / (Ns * rad)) * table stride
  FastDiv fdNs[kMaxStages];
  const double2* tw;  // omega_T^x, x in [0, T), forward sign (T = R * stride)
  uint32_t twlen;     // T
  // Per-stage twiddle table, q-major: stage s, butterfly offset j < Ns,
  // q = 1..rad-1 at stab[toff[s] + (q * qmul[s] - 1) * Ns[s] + j] holds
  // omega_{Ns rad}^{j q} exactly (consecutive j -> consecutive entries, so
  // the reads of a warp are bank-conflict free).
  const double2* stab;
  uint32_t stablen;
  uint32_t toff[kMaxStages];
  uint32_t qmul[kMaxStages];
};

// Per-stage accessors used inside stage_store: get(j, q) = omega_{Ns r}^{j q}.
struct TwQStage {
  const double2* base;
  uint32_t Ns, qmul;
  __device__ __forceinline__ double2 get(uint32_t j, uint32_t q) const {
    return base[(q * qmul - 1) * Ns + j];
  }
};
template <class TW>
struct TwQFlat {
  TW tw;
  uint32_t step;
  __device__ __forceinline__ double2 get(uint32_t j, uint32_t q) const { return tw.get(j * q * step); }
};

// Stage table staged in shared memory.
struct TwStage {
  const double2* t;
  __device__ __forceinline__ TwQStage stage(const SubFft& p, int s) const {
    return TwQStage{t + p.toff[s], p.Ns[s], p.qmul[s]};
  }
};
__device__ __forceinline__ TwStage load_tw_stage(double2* dst, const SubFft& p, int tid,
                                                 int nthr) {
  for (uint32_t i = tid; i < p.stablen; i += nthr) dst[i] = __ldg(p.stab + i);
  return TwStage{dst};
}

__device__ __forceinline__ uint32_t padidx(uint32_t i) { return i + (i >> 4); }
__host__ __device__ inline uint32_t padded_len(uint32_t n) {
  return n + (n >> 4) + 1;
}

// Twiddles from a global table (L1/L2 resident).
struct TwTable {
  const double2* t;
  __device__ __forceinline__ double2 get(uint32_t x) const { return __ldg(t + x); }
  __device__ __forceinline__ TwQFlat<TwTable> stage(const SubFft& p, int s) const {
    return TwQFlat<TwTable>{*this, p.twstep[s]};
  }
};

// Full table staged in shared memory (one exact entry per twiddle).
struct TwFull {
  const double2* t;
  __device__ __forceinline__ double2 get(uint32_t x) const { return t[x]; }
  __device__ __forceinline__ TwQFlat<TwFull> stage(const SubFft& p, int s) const {
    return TwQFlat<TwFull>{*this, p.twstep[s]};
  }
};
__device__ __forceinline__ TwFull load_tw_full(double2* dst, const SubFft& p, int tid,
                                               int nthr) {
  for (uint32_t i = tid; i < p.twlen; i += nthr) dst[i] = __ldg(p.tw + i);
  return TwFull{dst};
}

// Two-level shared-memory table: omega^x = hi[x >> 6] * lo[x & 63].
struct TwSmem {
  const double2* lo;
  const double2* hi;
  __device__ __forceinline__ double2 get(uint32_t x) const {
    return cmul(hi[x >> 6], lo[x & 63]);
  }
  __device__ __forceinline__ TwQFlat<TwSmem> stage(const SubFft& p, int s) const {
    return TwQFlat<TwSmem>{*this, p.twstep[s]};
  }
};
__host__ __device__ inline uint32_t tw_smem_len(uint32_t T) { return 64 + (T + 63) / 64; }

// Stage the two-level table of omega_T (T = p.twlen) into dst.
__device__ __forceinline__ TwSmem load_tw_smem(double2* dst, const SubFft& p,
                                               int tid, int nthr) {
  const uint32_t nhi = (p.twlen + 63) / 64;
  for (uint32_t i = tid; i < 64 + nhi; i += nthr)
    dst[i] = (i < 64) ? __ldg(p.tw + (i < p.twlen ? i : 0)) : __ldg(p.tw + 64 * (i - 64));
  return TwSmem{dst, dst + 64};
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

// Loads of one stage: butterfly bf reads elements t + q * R/RAD of its item.
template <int RAD, class Lay, class Src>
__device__ __forceinline__ void stage_load(double2 (&x)[kXMax], const Lay& lay,
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

// Twiddle, DFT and stores of one stage (outputs to sink(item, k, value)).
template <int RAD, bool INV, class Lay, class TWQ, class Sink>
__device__ __forceinline__ void stage_store(double2 (&x)[kXMax], const Lay& lay,
                                            uint32_t R, uint32_t Ns,
                                            const FastDiv& fdNs, const TWQ& twq,
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
#pragma unroll
        for (int q = 1; q < RAD; ++q) {
          double2 w = twq.get(j, uint32_t(q));
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

// Shared-memory source and sink.
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

// One complete transform of every item: the first stage reads from src
// (e.g. global memory: each thread issues all of its loads before the first
// use), the last stage writes to sink (e.g. global memory with the
// inter-pass twiddle); the stages in between exchange through buf.  src and
// sink may alias buf.  The register block x is shared by every radix so
// that the stage dispatch does not multiply register pressure.
template <bool INV, class Lay, class TW, class Src, class Sink>
__device__ __forceinline__ void fft_pass(double2* __restrict__ buf, const Lay& lay,
                                         const SubFft& p, const TW& tw,
                                         const Src& src, const Sink& sink,
                                         int tid, int nthr) {
  double2 x[kXMax];
  const int last = p.nst - 1;
  const SmemSrc<Lay> ssrc{buf, lay};
  const SmemSink<Lay> ssink{buf, lay};
  for (int s = 0; s <= last; ++s) {
    const int rad = p.rad[s];
    if (s == 0) {
#define TMG_L(RR) stage_load<RR>(x, lay, p.R, src, tid, nthr)
      TMG_RADIX_SWITCH(rad, TMG_L)
#undef TMG_L
    } else {
#define TMG_L(RR) stage_load<RR>(x, lay, p.R, ssrc, tid, nthr)
      TMG_RADIX_SWITCH(rad, TMG_L)
#undef TMG_L
    }
    __syncthreads();
    const uint32_t Ns = p.Ns[s];
    const auto twq = tw.stage(p, s);
    const FastDiv fd = p.fdNs[s];
    if (s == last) {
#define TMG_S(RR) stage_store<RR, INV>(x, lay, p.R, Ns, fd, twq, sink, tid, nthr)
      TMG_RADIX_SWITCH(rad, TMG_S)
#undef TMG_S
    } else {
#define TMG_S(RR) stage_store<RR, INV>(x, lay, p.R, Ns, fd, twq, ssink, tid, nthr)
      TMG_RADIX_SWITCH(rad, TMG_S)
#undef TMG_S
      __syncthreads();
    }
  }
}

// Whole transform in shared memory with one radix dispatch per stage: the
// code holds each radix's load / twiddle / DFT / store once (the fft_pass
// form inlines them separately for the first, middle and last stage of each
// source and sink type).  Expects the data in buf and a barrier before the
// call; ends with a barrier.
template <bool INV, class Lay, class TW>
__device__ __forceinline__ void fft_smem_compact(double2* __restrict__ buf, const Lay lay,
                                              const SubFft& p, const TW tw, int tid, int nthr) {
  double2 x[kXMax];
  const SmemSrc<Lay> ssrc{buf, lay};
  const SmemSink<Lay> ssink{buf, lay};
  for (int s = 0; s < p.nst; ++s) {
    const uint32_t Ns = p.Ns[s];
    const auto twq = tw.stage(p, s);
    const FastDiv fd = p.fdNs[s];
#define TMG_ST(RR)                                                              \
  stage_load<RR>(x, lay, p.R, ssrc, tid, nthr);                                 \
  __syncthreads();                                                              \
  stage_store<RR, INV>(x, lay, p.R, Ns, fd, twq, ssink, tid, nthr);             \
  __syncthreads();
    TMG_RADIX_SWITCH(p.rad[s], TMG_ST)
#undef TMG_ST
  }
}

// ---------------------------------------------------------------------------
// Ping-pong transform for the column passes: stage s reads buffer a and
// writes buffer b (then they swap), so loads and stores of a stage never
// conflict -- one barrier per stage -- and a thread holds one butterfly of
// at most 8 values at a time (radix <= 8 schedules), which lets a CTA run
// 1024 threads at 64 registers.  Stage twiddles are read through L1 from
// the global stage table (q-major, same layout and values as TwStage).
// Returns the buffer holding the result; expects a barrier before the call
// and ends with one.
template <int RAD, bool INV, class Lay>
__device__ __forceinline__ void stage_pp(const double2* __restrict__ a, double2* __restrict__ b,
                                         const Lay& lay, const SubFft& p, int s, int tid,
                                         int nthr) {
  const uint32_t R = p.R, Ns = p.Ns[s];
  const uint32_t nbi = R / RAD;
  const uint32_t nbf = nbi * lay.nitems();
  const FastDiv fd = p.fdNs[s];
  const double2* __restrict__ st = p.stab + p.toff[s];
  const uint32_t qm = p.qmul[s];
  for (uint32_t bf = tid; bf < nbf; bf += nthr) {
    uint32_t item, t;
    lay.split(bf, nbi, item, t);
    double2 x[RAD];
#pragma unroll
    for (int q = 0; q < RAD; ++q) x[q] = a[lay.idx(item, t + q * nbi)];
    const uint32_t tq = fdiv(t, fd);
    const uint32_t j = t - tq * Ns;
    if (j != 0) {
#pragma unroll
      for (int q = 1; q < RAD; ++q) {
        const double2 w = __ldg(st + (uint32_t(q) * qm - 1) * Ns + j);
        x[q] = INV ? cmulc(x[q], w) : cmul(x[q], w);
      }
    }
    dft<RAD, INV>(x);
    const uint32_t ob = tq * Ns * RAD + j;
#pragma unroll
    for (int q = 0; q < RAD; ++q) b[lay.idx(item, ob + q * Ns)] = x[q];
  }
}

template <bool INV, class Lay>
__device__ __forceinline__ double2* fft_pp(double2* a, double2* b, const Lay lay,
                                           const SubFft& p, int tid, int nthr) {
  for (int s = 0; s < p.nst; ++s) {
    switch (p.rad[s]) {
      case 8: stage_pp<8, INV>(a, b, lay, p, s, tid, nthr); break;
      case 4: stage_pp<4, INV>(a, b, lay, p, s, tid, nthr); break;
      case 2: stage_pp<2, INV>(a, b, lay, p, s, tid, nthr); break;
      case 3: stage_pp<3, INV>(a, b, lay, p, s, tid, nthr); break;
      case 5: stage_pp<5, INV>(a, b, lay, p, s, tid, nthr); break;
      default: stage_pp<7, INV>(a, b, lay, p, s, tid, nthr); break;
    }
    __syncthreads();
    double2* t = a;
    a = b;
    b = t;
  }
  return a;
}

// Whole transform in shared memory (natural order in and out), ends with a
// barrier.
template <bool INV, class Lay, class TW>
__device__ __forceinline__ void fft_smem(double2* __restrict__ buf, const Lay& lay,
                                         const SubFft& p, const TW& tw, int tid,
                                         int nthr) {
  fft_pass<INV>(buf, lay, p, tw, SmemSrc<Lay>{buf, lay}, SmemSink<Lay>{buf, lay}, tid, nthr);
  __syncthreads();
}

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
