// Compile-time column-pass stages shared by k_multipass.cu and k_f1d.cu:
// cc_stages walks a Sched<> radix schedule over a tile of 2^LOGC columns
// (stage 0 from a source, the last stage into a sink), F1SinkQ is the first
// column pass's twiddled sink, digit_at re-derives one balanced digit.
#pragma once

#include "kernels.cuh"
#include "fft_ct.cuh"

namespace tmg {

__device__ __forceinline__ int cbit(const uint32_t* cb, int64_t j) {
  return int((__ldg(cb + (j >> 5)) >> (j & 31)) & 1u);
}

// Single digit re-derived from the limbs and its carry-in bit (the carry
// bits are all zero for the unbalanced split).
__device__ __forceinline__ double digit_at(const uint64_t* limbs,
                                           int64_t nlimbs, int b, int64_t lead,
                                           int64_t count, const uint32_t* cb,
                                           int64_t j, bool balanced = true) {
  uint64_t w = window_bits(limbs, nlimbs, j * b - lead, b);
  return double(split_digit(w, cbit(cb, j), b, j == count - 1 || !balanced));
}

// gamma-dagger fold of the high split's top coefficient into pre-mapped
// coefficient j < nfold + lambda (maps_f64.cpp:337-347).
__device__ __forceinline__ void high_top_fold(const MapConsts& mc, int64_t j, int64_t N, double topu,
                                              double topv, double2& v) {
  const int lam = mc.lambda;
  RowLoop<kMaxLambda>::run([&](auto rc) {
    constexpr int r = decltype(rc)::value;
    if (r < lam) {
      int64_t k = j - r;
      if (k < 0) k += N;
      if (k < mc.nfold) {
        const double g = mc.fold[k] * coef_r<r>(2, double(k), double(N), mc.cpre[r]);
        v.x += topu * g;
        v.y += topv * g;
      }
    }
  });
}

// ---------------------------------------------------------------------------
// Column passes with compile-time radix schedules (the column analogue of
// k_mid_4096).  A CTA owns c = 2^LOGC consecutive columns of length R
// (interleaved in shared memory, LayCols).  Every stage's butterflies are
// spread over the NTHR threads, NB = ceil(c R / (RAD NTHR)) per thread, with
// strides, butterfly counts and stage-table offsets known at compile time.
// The first stage loads straight from global memory (all of a thread's
// loads in flight together), the last stores straight to global memory, so
// the tile never makes a separate staging pass through shared memory.
// Numerics are those of the generic passes (same stage tables, same
// in-register DFTs).
template <int RAD, int NB, uint32_t R, int LOGC, int NTHR, int P, class Src>
__device__ __forceinline__ void cc_load(double2 (&x)[P], const Src& src, int tid) {
  constexpr uint32_t nbi = R / RAD, nbf = nbi << LOGC;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const uint32_t bf = uint32_t(tid) + uint32_t(i) * NTHR;
    if (nbf % NTHR == 0 || bf < nbf) {
      const uint32_t item = bf & ((1u << LOGC) - 1), t = bf >> LOGC;
#pragma unroll
      for (int q = 0; q < RAD; ++q) x[i * RAD + q] = src(item, t + q * nbi);
    }
  }
}

template <int RAD, int NB, bool INV, uint32_t R, uint32_t NS, int LOGC, int NTHR, int P, class Sink>
__device__ __forceinline__ void cc_store(double2 (&x)[P], const double2* __restrict__ stab,
                                         uint32_t qmul, const Sink& sink, int tid) {
  constexpr uint32_t nbi = R / RAD, nbf = nbi << LOGC;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const uint32_t bf = uint32_t(tid) + uint32_t(i) * NTHR;
    if (nbf % NTHR == 0 || bf < nbf) {
      const uint32_t item = bf & ((1u << LOGC) - 1), t = bf >> LOGC;
      const uint32_t tq = t / NS, j = t - tq * NS;
      const uint32_t ob = tq * NS * RAD + j;
      double2* xv = x + i * RAD;
      if constexpr (SinkPrep<Sink>::value) {
        const auto pre = sink.prep(item, ob);
        if (NS > 1 && j != 0) {
#pragma unroll
          for (int q = 1; q < RAD; ++q) {
            const double2 w = stab[(uint32_t(q) * qmul - 1) * NS + j];
            xv[q] = INV ? cmulc(xv[q], w) : cmul(xv[q], w);
          }
        }
        dft<RAD, INV>(xv);
#pragma unroll
        for (int q = 0; q < RAD; ++q) sink.put(item, ob + q * NS, uint32_t(q), xv[q], pre);
      } else {
        if (NS > 1 && j != 0) {
#pragma unroll
          for (int q = 1; q < RAD; ++q) {
            const double2 w = stab[(uint32_t(q) * qmul - 1) * NS + j];
            xv[q] = INV ? cmulc(xv[q], w) : cmul(xv[q], w);
          }
        }
        dft<RAD, INV>(xv);
#pragma unroll
        for (int q = 0; q < RAD; ++q) sink(item, ob + q * NS, xv[q]);
      }
    }
  }
}

// hook (NoHook, fft_ct.cuh): called by every thread once the last stage has
// taken its inputs from the tile (behind that stage's barrier): the tile's
// shared memory is free from there on, e.g. for staging the next tile.
template <bool INV, class SC, int S, int LOGC, int NTHR, int P, class Src, class Sink, class Hook = NoHook>
__device__ __forceinline__ void cc_stages(double2 (&x)[P], double2* __restrict__ buf,
                                          const LayCols& lay, const double2* __restrict__ stab,
                                          const SubFft& p, const Src& src, const Sink& sink,
                                          int tid, const Hook& hook = Hook{}) {
  constexpr int RAD = SC::rad(S);
  constexpr uint32_t NS = SC::ns(S);
  constexpr uint32_t R = SC::R;
  constexpr uint32_t nbf = (R / RAD) << LOGC;
  constexpr int NB = int((nbf + NTHR - 1) / NTHR);
  static_assert(NB * RAD <= P, "register block");
  constexpr bool last = S + 1 == SC::nst;
  if constexpr (S == 0) {
    cc_load<RAD, NB, R, LOGC, NTHR, P>(x, src, tid);
  } else {
    cc_load<RAD, NB, R, LOGC, NTHR, P>(x, SmemSrc<LayCols>{buf, lay}, tid);
  }
  __syncthreads();
  const double2* st = stab + p.toff[S];
  if constexpr (last) {
    hook();
    cc_store<RAD, NB, INV, R, NS, LOGC, NTHR, P>(x, st, p.qmul[S], sink, tid);
  } else {
    cc_store<RAD, NB, INV, R, NS, LOGC, NTHR, P>(x, st, p.qmul[S], SmemSink<LayCols>{buf, lay}, tid);
    __syncthreads();
    cc_stages<INV, SC, S + 1, LOGC, NTHR, P>(x, buf, lay, stab, p, src, sink, tid, hook);
  }
}

// First column pass's sink: T[k][col] = v omega_L^{col k} with
// omega_L^{col (ob + q NS)} = omega_L^{col ob} * omega_L^{col NS q}; the
// first factor is fetched before the last stage's DFT (prep), the second
// comes from a per-CTA table qt[item * RADL + q].
template <uint32_t RADL>
struct F1SinkQ {
  double2* out;
  uint32_t ncols, col0;
  TwGlobal tw;
  const double2* qt;
  __device__ __forceinline__ double2 prep(uint32_t item, uint32_t ob) const {
    const uint32_t x = (col0 + item) * ob;
    return x ? tw.get(x) : make_double2(1.0, 0.0);
  }
  __device__ __forceinline__ void put(uint32_t item, uint32_t k, uint32_t q, double2 v,
                                      double2 b) const {
    out[int64_t(k) * ncols + col0 + item] = cmul(v, cmul(b, qt[item * RADL + q]));
  }
};
template <uint32_t RADL>
struct SinkPrep<F1SinkQ<RADL>> {
  static constexpr bool value = true;
};

template <class SC>
__host__ __device__ constexpr uint32_t ct_last_rad() { return uint32_t(SC::rad(SC::nst - 1)); }
template <class SC>
__host__ __device__ constexpr uint32_t ct_last_ns() { return SC::ns(SC::nst - 1); }

}  // namespace tmg
