// Chunk extraction (balanced split), ring-change series coefficients and the
// pre/post maps of the low and high products, as device functions.
//
// Reference semantics:
//   split            split.cpp:66-102 (chunk_store: windows of u*2^lead,
//                    balanced digits in (-2^{b-1}, 2^{b-1}], unbalanced top)
//   series coeffs    series.cpp:146-170 (alpha/beta/gamma/delta closed forms)
//   alpha*, gamma+   maps_f64.cpp:48-136, 317-348
//   beta*, delta+    maps_f64.cpp:140-188, 269-281, 350-384
#pragma once

#include <type_traits>

#include "common.cuh"

namespace tmg {

// Parameters of the ring-change maps, built on the host (plan.cu).
constexpr int kMaxLambda = 8;
constexpr int kMaxFold = 24;
constexpr int kMaxRootTerms = 32;

struct MapConsts {
  int32_t mode;      // 0 full, 1 low, 2 high
  int32_t b;
  int64_t N;         // chunk count of the transform (low/high) or N (full)
  int32_t lambda;
  int32_t balanced;          // signed (balanced) split, products.hpp:43-44
  double cpre[kMaxLambda];   // pre-map (alpha or gamma) row scale
  double cpost[kMaxLambda];  // post-map (beta or delta) row scale
  double step;               // 2^-b
  double scale_out;          // 2^b (low/high) or 1 (full)
  // high product only (maps_f64.cpp:192-245)
  int32_t nfold;             // fold_row length
  double fold[kMaxFold];     // 2^b / root^{i+1}
  int32_t nroot;             // terms of the root-channel sums
  double ipow[kMaxRootTerms];  // inv_root^d, d = 0..nroot-1 (ipow[0] = 1)
  int32_t nhrho;             // terms of hrho (d = 1..nhrho)
  double root_neg_n;
  double cofactor_scaled;
};

// Bits [pos, pos + b) of the operand held in `limbs` (nlimbs words);
// positions below 0 or at/after nlimbs*64 read as zero.
__device__ __forceinline__ uint64_t window_bits(const uint64_t* __restrict__ limbs,
                                                int64_t nlimbs, int64_t pos,
                                                int b) {
  const uint64_t mask = (b >= 64) ? ~0ull : ((1ull << b) - 1);
  int64_t idx = pos >> 6;  // floor
  uint32_t sh = uint32_t(pos & 63);
  uint64_t lo = 0, hi = 0;
  if (idx >= 0 && idx < nlimbs) lo = __ldg(limbs + idx);
  if (idx + 1 >= 0 && idx + 1 < nlimbs) hi = __ldg(limbs + idx + 1);
  uint64_t w = (sh == 0) ? lo : ((lo >> sh) | (hi << (64 - sh)));
  return w & mask;
}

// Sequential reader of consecutive b-bit windows of u * 2^lead.
template <class Ld>
struct WindowReader {
  Ld ld;
  int64_t idx;
  uint32_t sh;
  uint64_t cur, nxt;
  int b;
  uint64_t mask;
  __device__ __forceinline__ void init(const Ld& l, int64_t pos, int bb) {
    ld = l;
    b = bb;
    mask = (1ull << bb) - 1;
    idx = pos >> 6;
    sh = uint32_t(pos & 63);
    cur = ld(idx);
    nxt = ld(idx + 1);
  }
  __device__ __forceinline__ uint64_t next() {
    uint64_t w = sh ? ((cur >> sh) | (nxt << (64 - sh))) : cur;
    sh += b;
    if (sh >= 64) {
      sh -= 64;
      cur = nxt;
      ++idx;
      nxt = ld(idx + 1);
    }
    return w & mask;
  }
};

struct GlobalLimbs {
  const uint64_t* limbs;
  int64_t nlimbs;
  __device__ __forceinline__ uint64_t operator()(int64_t i) const {
    return (i >= 0 && i < nlimbs) ? __ldg(limbs + i) : 0ull;
  }
};


// Transfer code of a chunk for the balanced-split carry chain
// (split.cpp:88-95): generate if window > 2^{b-1}, propagate if equal.
__device__ __forceinline__ uint32_t split_tf(uint64_t w, int b) {
  const uint64_t half = 1ull << (b - 1);
  return w > half ? tf_const(1) : (w == half ? kTfIdentity : tf_const(0));
}

// Balanced digit of a chunk with window w and incoming carry cin.
__device__ __forceinline__ int64_t split_digit(uint64_t w, int cin, int b,
                                               bool top) {
  int64_t x = int64_t(w) + cin;
  if (!top && x > (int64_t(1) << (b - 1))) x -= (int64_t(1) << b);
  return x;
}

// Series coefficient of family row r at residue k (series.cpp:146-170):
//   alpha: (-1)^r k prod_{i<r-1} (k + r - N(i+1)) / (r! N^r 2^{rb})
//   beta :         prod_{i<r}   (k + iN)          / (r! N^r 2^{rb})
//   gamma:       k prod_{i<r-1} (k + r + N(i+1)) / (r! N^r 2^{rb})
//   delta: (-1)^r  prod_{i<r}   (k - iN)          / (r! N^r 2^{rb})
// The signed scale sgn/(r! N^r 2^{rb}) arrives precomputed in c.
// fam: 0 alpha, 1 beta, 2 gamma, 3 delta.
__device__ __forceinline__ double series_coef(int fam, int r, double k,
                                              double N, double c) {
  if (r == 0) return 1.0;
  double p;
  if (fam == 0 || fam == 2) {
    p = k;
    const double sgn = (fam == 0) ? -1.0 : 1.0;
    for (int i = 0; i < r - 1; ++i) p *= (k + double(r) + sgn * N * double(i + 1));
  } else {
    const double sgn = (fam == 1) ? 1.0 : -1.0;
    p = k;
    for (int i = 1; i < r; ++i) p *= (k + sgn * N * double(i));
  }
  return p * c;
}

// Same coefficient with the row r known at compile time: the r integer
// factors are exact doubles (|k + iN| < 2^53) stepped by +-N, so only the
// products round.
template <int R>
__device__ __forceinline__ double coef_r(int fam, double k, double N, double c) {
  if constexpr (R == 0) {
    return 1.0;
  } else {
    double p = k;
    if (fam == 0 || fam == 2) {
      const double st = (fam == 0) ? -N : N;
      double f = k + double(R) + st;
#pragma unroll
      for (int i = 0; i < R - 1; ++i) {
        p *= f;
        f += st;
      }
    } else {
      const double st = (fam == 1) ? N : -N;
      double f = k + st;
#pragma unroll
      for (int i = 1; i < R; ++i) {
        p *= f;
        f += st;
      }
    }
    return p * c;
  }
}

// coef_r with the row known only after unrolling (r is a loop constant of a
// fully unrolled loop): the same multiplications as coef_r<R>.
__device__ __forceinline__ double coef_rt(int fam, int R, double k, double N, double c) {
  double p = k;
  if (fam == 0 || fam == 2) {
    const double st = (fam == 0) ? -N : N;
    double f = k + double(R) + st;
#pragma unroll
    for (int i = 0; i < kMaxLambda - 1; ++i) {
      if (i < R - 1) {
        p *= f;
        f += st;
      }
    }
  } else {
    const double st = (fam == 1) ? N : -N;
    double f = k + st;
#pragma unroll
    for (int i = 1; i < kMaxLambda; ++i) {
      if (i < R) {
        p *= f;
        f += st;
      }
    }
  }
  return p * c;
}

// Compile-time loop r = 0 .. R-1 calling f(std::integral_constant<int, r>).
template <int R>
struct RowLoop {
  template <class F>
  __device__ __forceinline__ static void run(F&& f) {
    RowLoop<R - 1>::run(f);
    f(std::integral_constant<int, R - 1>{});
  }
};
template <>
struct RowLoop<0> {
  template <class F>
  __device__ __forceinline__ static void run(F&&) {}
};

// r = R-1 .. 0: the series maps accumulate their small high-order rows
// first so that only the last term (row 0, the largest) rounds at the
// magnitude of the result.
template <int R>
struct RowLoopDown {
  template <class F>
  __device__ __forceinline__ static void run(F&& f) {
    f(std::integral_constant<int, R - 1>{});
    RowLoopDown<R - 1>::run(f);
  }
};
template <>
struct RowLoopDown<0> {
  template <class F>
  __device__ __forceinline__ static void run(F&&) {}
};

}  // namespace tmg
