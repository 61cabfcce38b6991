// Compile-time radix schedules for the hot transform shapes.
//
// The generic passes of fft_smem.cuh dispatch every stage on a runtime radix
// and read the stage geometry from the kernel parameters; for the shapes the
// product sizes hit most (rows of 4096 = 16 x 16 x 16 forward and
// 2048 = 16 x 16 x 8 inverse) the whole schedule is known at compile time:
// butterfly counts, strides, Ns and the twiddle-table offsets become
// immediates, every loop unrolls, and the kernel carries only the code of the
// stages it runs.  Numerics are those of the generic pass (same stage tables,
// same in-register DFTs, same order of operations).
#pragma once

#include "fft_smem.cuh"

namespace tmg {

template <int R0, int R1 = 0, int R2 = 0, int R3 = 0>
struct Sched {
  static constexpr int nst = R1 == 0 ? 1 : R2 == 0 ? 2 : R3 == 0 ? 3 : 4;
  __host__ __device__ static constexpr int rad(int s) {
    return s == 0 ? R0 : s == 1 ? R1 : s == 2 ? R2 : R3;
  }
  __host__ __device__ static constexpr uint32_t ns(int s) {
    return s == 0 ? 1u : uint32_t(rad(s - 1)) * ns(s - 1);
  }
  static constexpr uint32_t R = uint32_t(R0) * (R1 ? R1 : 1) * (R2 ? R2 : 1) * (R3 ? R3 : 1);
  // offset of stage s in the q-major stage table (make_subfft, plan.cu)
  __host__ __device__ static constexpr uint32_t toff(int s) {
    return s <= 1 ? 0u : toff(s - 1) + ns(s - 1) * uint32_t(rad(s - 1) - 1);
  }
};

// Row layout with one or two rows (a conjugate pair) of compile-time length.
struct RowPair {
  uint32_t rowstride, nrows;
  __device__ __forceinline__ uint32_t idx(uint32_t item, uint32_t e) const {
    return item * rowstride + padidx(e);
  }
};

// Each row of the pair is owned by one half of the CTA (threads
// [0, NTHR/2) row 0, [NTHR/2, NTHR) row 1), which syncs on its own named
// barrier: the halves run their stages independently and overlap each
// other's stalls; only the spectral step couples the rows.
template <int NTHR>
__device__ __forceinline__ void ct_sync(int tid) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + (tid >= NTHR / 2 ? 1 : 0)), "r"(NTHR / 2) : "memory");
}

template <int RAD, uint32_t R, int NTHR, class Src>
__device__ __forceinline__ void ct_load(double2 (&x)[16], const RowPair& lay, const Src& src,
                                        int tid) {
  constexpr uint32_t nbi = R / RAD;
  static_assert(nbi <= uint32_t(NTHR / 2), "one butterfly per thread and stage");
  const uint32_t item = tid >= NTHR / 2 ? 1u : 0u;
  const uint32_t t = uint32_t(tid) - item * (NTHR / 2);
  if (t < nbi && item < lay.nrows) {
#pragma unroll
    for (int q = 0; q < RAD; ++q) x[q] = src(item, t + q * nbi);
  }
}

// Sinks that take a per-butterfly factor (SinkPrep<Sink>::value) get
// pre = sink.prep(item, ob) before the stage's twiddles and DFT, so its
// loads overlap them, and put(item, ob + q NS, q, v, pre) per output.
template <class Sink>
struct SinkPrep {
  static constexpr bool value = false;
};

// TMUL: stage-table index stride (2: a length-R/2 inverse reading the
// forward stage table of length R at every second entry).
template <int RAD, bool INV, uint32_t R, uint32_t NS, int NTHR, class Sink, uint32_t TMUL = 1>
__device__ __forceinline__ void ct_store(double2 (&x)[16], const RowPair& lay,
                                         const double2* __restrict__ stab, uint32_t qmul,
                                         const Sink& sink, int tid) {
  constexpr uint32_t nbi = R / RAD;
  const uint32_t item = tid >= NTHR / 2 ? 1u : 0u;
  const uint32_t t = uint32_t(tid) - item * (NTHR / 2);
  {
    if (t < nbi && item < lay.nrows) {
      const uint32_t tq = t / NS;
      const uint32_t j = t - tq * NS;
      const uint32_t ob = tq * NS * RAD + j;
      double2* xv = x;
      if constexpr (SinkPrep<Sink>::value) {
        const auto pre = sink.prep(item, ob);
        if (NS > 1 && j != 0) {
#pragma unroll
          for (int q = 1; q < RAD; ++q) {
            const double2 w = stab[TMUL * ((uint32_t(q) * qmul - 1) * NS + j)];
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
            const double2 w = stab[TMUL * ((uint32_t(q) * qmul - 1) * NS + j)];
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

// Stages S .. nst-1 of schedule SC, through the caller's register block x
// (one block for every stage: separate per-stage arrays defeat ptxas's
// register promotion and land in local memory).  Stage 0 reads src, the last stage
// writes sink, the others exchange through buf (RowPair layout).  toff and
// qmul of each stage come from the plan (the inverse of a row pass reads the
// forward table through the qmul mapping, plan.cu map_stages).
// hook: called by every thread of a half once the last stage has taken its
// inputs (behind that stage's barrier of the half): the half's row buffer is
// free from there on.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};
template <bool INV, class SC, int S, int NTHR, class Src, class Sink, uint32_t TMUL = 1, class Hook = NoHook>
__device__ __forceinline__ void ct_stages(double2 (&x)[16], double2* __restrict__ buf,
                                          const RowPair& lay, const double2* __restrict__ stab,
                                          const SubFft& p, const Src& src, const Sink& sink,
                                          int tid, const Hook& hook = Hook{}) {
  constexpr int RAD = SC::rad(S);
  constexpr uint32_t NS = SC::ns(S);
  constexpr uint32_t R = SC::R;
  constexpr bool last = S + 1 == SC::nst;
  if constexpr (S == 0) {
    ct_load<RAD, R, NTHR>(x, lay, src, tid);
  } else {
    ct_load<RAD, R, NTHR>(x, lay, SmemSrc<RowPair>{buf, lay}, tid);
  }
  ct_sync<NTHR>(tid);
  const double2* st = stab + p.toff[S];
  if constexpr (last) {
    hook();
    ct_store<RAD, INV, R, NS, NTHR, Sink, TMUL>(x, lay, st, p.qmul[S], sink, tid);
  } else {
    ct_store<RAD, INV, R, NS, NTHR, SmemSink<RowPair>, TMUL>(x, lay, st, p.qmul[S], SmemSink<RowPair>{buf, lay},
                                                             tid);
    ct_sync<NTHR>(tid);
    ct_stages<INV, SC, S + 1, NTHR, Src, Sink, TMUL, Hook>(x, buf, lay, stab, p, src, sink, tid, hook);
  }
}

// L2 prefetch of a contiguous global range (bytes multiple of 16).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

}  // namespace tmg
