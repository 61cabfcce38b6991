// In-register small DFT butterflies (radix 2, 3, 4, 5, 7, 8, 16) in FP64.
//
// Forward transforms use e^{-2 pi i jk / r}; INV selects e^{+2 pi i jk / r}.
// No scaling is applied.  These replace FFTW's codelets, which the reference
// reaches through fftw_execute_dft_r2c / _c2r (convolution.cpp:175-195).
#pragma once

#include "common.cuh"

namespace tmg {

// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 mul_mi(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2,
                                     double2& x3) {
  double2 t0 = cadd(x0, x2), t1 = csub(x0, x2);
  double2 t2 = cadd(x1, x3), t3 = mul_mi<INV>(csub(x1, x3));
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd(t1, t3);
  x3 = csub(t1, t3);
}

// Multiplying by an irrational constant: every constant is carried as an
// unevaluated pair hi + lo (lo = the rounding error of hi, from 70-digit
// evaluations), so the product rounds once against the exact constant.  The
// nearest doubles of cos/sin(2 pi j/P) are biased (e.g. 1/sqrt2 rounds up by
// 0.44 ulp), and a butterfly network that multiplies by them at every stage
// accumulates a coherent gain error of several 2^-53 -- large enough to
// matter for structured operands at the reference's chunk widths.
__device__ __forceinline__ double mul_hl(double x, double hi, double lo) {
  return fma(x, hi, x * lo);
}

// Odd prime radix via the symmetric pair formulation:
//   X_k = x0 + sum_j cos(2pi jk/p) t_j  -/+ i sum_j sin(2pi jk/p) s_j
// with t_j = x_j + x_{p-j}, s_j = x_j - x_{p-j}.
template <int P>
struct OddTrig;
template <>
struct OddTrig<3> {
  __device__ static constexpr double c(int) { return -0.5; }
  __device__ static constexpr double cl(int) { return 0.0; }
  __device__ static constexpr double s(int) { return 0.8660254037844386; }
  __device__ static constexpr double sl(int) { return 5.0175421109034514e-17; }
};
template <>
struct OddTrig<5> {
  __device__ static constexpr double c(int j) {
    return j == 1 ? 0.30901699437494745 : -0.8090169943749475;
  }
  __device__ static constexpr double cl(int j) {
    return j == 1 ? -2.716057601841253e-17 : 2.716057601841253e-17;
  }
  __device__ static constexpr double s(int j) {
    return j == 1 ? 0.9510565162951535 : 0.5877852522924731;
  }
  __device__ static constexpr double sl(int j) {
    return j == 1 ? 4.0934500900087295e-17 : -7.93475083819002e-18;
  }
};
template <>
struct OddTrig<7> {
  __device__ static constexpr double c(int j) {
    return j == 1 ? 0.6234898018587335 : j == 2 ? -0.2225209339563144 : -0.9009688679024191;
  }
  __device__ static constexpr double cl(int j) {
    return j == 1 ? 4.716099920540896e-17
                  : j == 2 ? -1.1412494827220627e-17 : 1.9762646853069492e-17;
  }
  __device__ static constexpr double s(int j) {
    return j == 1 ? 0.7818314824680298 : j == 2 ? 0.9749279121818236 : 0.4338837391175581;
  }
  __device__ static constexpr double sl(int j) {
    return j == 1 ? 5.074320362582868e-18
                  : j == 2 ? -1.232383765062425e-17 : 7.407189078946677e-20;
  }
};

template <int P, bool INV>
__device__ __forceinline__ void dft_odd(double2* x) {
  constexpr int H = (P - 1) / 2;
  double2 t[H], s[H];
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    t[j - 1] = cadd(x[j], x[P - j]);
    s[j - 1] = csub(x[j], x[P - j]);
  }
  const double2 x0 = x[0];
  double2 sum = x0;
#pragma unroll
  for (int j = 0; j < H; ++j) sum = cadd(sum, t[j]);
  x[0] = sum;
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    // cos/sin(2 pi j k / P) with jk reduced into the first half-turn
    double cj[H], cjl[H], sj[H], sjl[H];
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      const int m = (j * k) % P;
      const bool lo = m <= H;
      const int mm = lo ? m : P - m;
      cj[j - 1] = OddTrig<P>::c(mm);
      cjl[j - 1] = OddTrig<P>::cl(mm);
      sj[j - 1] = lo ? OddTrig<P>::s(mm) : -OddTrig<P>::s(mm);
      sjl[j - 1] = lo ? OddTrig<P>::sl(mm) : -OddTrig<P>::sl(mm);
    }
    double2 a, b;
    if constexpr (P == 3) {
      a = make_double2(fma(-0.5, t[0].x, x0.x), fma(-0.5, t[0].y, x0.y));
      b = make_double2(mul_hl(s[0].x, sj[0], sjl[0]), mul_hl(s[0].y, sj[0], sjl[0]));
    } else {
      // the lo parts first (small), then the hi products, then x0
      a = make_double2(cjl[0] * t[0].x, cjl[0] * t[0].y);
      b = make_double2(sjl[0] * s[0].x, sjl[0] * s[0].y);
#pragma unroll
      for (int j = 1; j < H; ++j) {
        a.x = fma(cjl[j], t[j].x, a.x);
        a.y = fma(cjl[j], t[j].y, a.y);
        b.x = fma(sjl[j], s[j].x, b.x);
        b.y = fma(sjl[j], s[j].y, b.y);
      }
#pragma unroll
      for (int j = 0; j < H; ++j) {
        a.x = fma(cj[j], t[j].x, a.x);
        a.y = fma(cj[j], t[j].y, a.y);
        b.x = fma(sj[j], s[j].x, b.x);
        b.y = fma(sj[j], s[j].y, b.y);
      }
      a = cadd(a, x0);
    }
    // forward: X_k = a - i b ; X_{P-k} = a + i b
    const double2 ib = make_double2(-b.y, b.x);
    if (INV) {
      x[k] = cadd(a, ib);
      x[P - k] = csub(a, ib);
    } else {
      x[k] = csub(a, ib);
      x[P - k] = cadd(a, ib);
    }
  }
}

constexpr double kR2 = 0.7071067811865476, kR2l = -4.833646656726457e-17;  // 1/sqrt2
constexpr double kC1 = 0.9238795325112867, kC1l = 1.7645047084336677e-17;  // cos pi/8
constexpr double kS1 = 0.3826834323650898, kS1l = -1.0050772696461588e-17; // sin pi/8

// omega_8^k multipliers (forward: e^{-i pi k/4})
template <bool INV>
__device__ __forceinline__ double2 w8_1(double2 a) {
  // forward: (1 - i)/sqrt2 * a ; inverse: (1 + i)/sqrt2 * a
  return INV ? make_double2(mul_hl(a.x - a.y, kR2, kR2l), mul_hl(a.x + a.y, kR2, kR2l))
             : make_double2(mul_hl(a.x + a.y, kR2, kR2l), mul_hl(a.y - a.x, kR2, kR2l));
}
template <bool INV>
__device__ __forceinline__ double2 w8_3(double2 a) {
  // forward: (-1 - i)/sqrt2 * a ; inverse: (-1 + i)/sqrt2 * a
  return INV ? make_double2(mul_hl(-a.x - a.y, kR2, kR2l), mul_hl(a.x - a.y, kR2, kR2l))
             : make_double2(mul_hl(a.y - a.x, kR2, kR2l), mul_hl(-a.x - a.y, kR2, kR2l));
}

template <bool INV>
__device__ __forceinline__ void dft8(double2* x) {
  // DIT: even/odd radix-4 then combine
  double2 e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6];
  double2 o0 = x[1], o1 = x[3], o2 = x[5], o3 = x[7];
  dft4<INV>(e0, e1, e2, e3);
  dft4<INV>(o0, o1, o2, o3);
  o1 = w8_1<INV>(o1);
  o2 = mul_mi<INV>(o2);
  o3 = w8_3<INV>(o3);
  x[0] = cadd(e0, o0);
  x[4] = csub(e0, o0);
  x[1] = cadd(e1, o1);
  x[5] = csub(e1, o1);
  x[2] = cadd(e2, o2);
  x[6] = csub(e2, o2);
  x[3] = cadd(e3, o3);
  x[7] = csub(e3, o3);
}

// (a.x + i a.y)(c - i s) with c = ch + cl, s = sh + sl
__device__ __forceinline__ double2 rot_hl(double2 a, double ch, double cl, double sh,
                                          double sl) {
  double re = fma(a.x, cl, a.y * sl);
  re = fma(a.y, sh, re);
  re = fma(a.x, ch, re);
  double im = fma(a.y, cl, -a.x * sl);
  im = fma(-a.x, sh, im);
  im = fma(a.y, ch, im);
  return make_double2(re, im);
}

// omega_16^j * a for j = 0..9 (compile-time j)
template <bool INV>
__device__ __forceinline__ double2 w16(double2 a, int j) {
  const double sg = INV ? -1.0 : 1.0;  // e^{-+2 pi i j/16} = c -+ i s
  switch (j) {
    case 0: return a;
    case 1: return rot_hl(a, kC1, kC1l, sg * kS1, sg * kS1l);
    case 2: return w8_1<INV>(a);
    case 3: return rot_hl(a, kS1, kS1l, sg * kC1, sg * kC1l);
    case 4: return mul_mi<INV>(a);
    case 5: return rot_hl(a, -kS1, -kS1l, sg * kC1, sg * kC1l);
    case 6: return w8_3<INV>(a);
    case 7: return rot_hl(a, -kC1, -kC1l, sg * kS1, sg * kS1l);
    case 8: return make_double2(-a.x, -a.y);
    default: return rot_hl(a, -kC1, -kC1l, -sg * kS1, -sg * kS1l);  // 9
  }
}

template <bool INV>
__device__ __forceinline__ void dft16(double2* x) {
  // 4 x radix-4 (DIT): F_m(k1) = DFT4(x_m, x_{m+4}, x_{m+8}, x_{m+12})
  double2 f[4][4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    f[m][0] = x[m];
    f[m][1] = x[m + 4];
    f[m][2] = x[m + 8];
    f[m][3] = x[m + 12];
    dft4<INV>(f[m][0], f[m][1], f[m][2], f[m][3]);
  }
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    double2 g0 = f[0][k1];
    double2 g1 = w16<INV>(f[1][k1], k1);
    double2 g2 = w16<INV>(f[2][k1], 2 * k1);
    double2 g3 = w16<INV>(f[3][k1], 3 * k1);
    dft4<INV>(g0, g1, g2, g3);
    x[k1] = g0;
    x[k1 + 4] = g1;
    x[k1 + 8] = g2;
    x[k1 + 12] = g3;
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dft(double2* x);

__host__ __device__ constexpr int inv_mod(int a, int m) {
  int r = 1;
  while ((a * r) % m != 1) ++r;
  return r;
}

// Composite radix P = P1 P2 with gcd(P1, P2) = 1 by the prime-factor
// (Good-Thomas) algorithm: input n = (n1 P2 + n2 P1) mod P, output
// k = (k1 P2 t2 + k2 P1 t1) mod P with t2 = P2^-1 mod P1, t1 = P1^-1 mod P2,
// so omega_P^{nk} = omega_P1^{n1 k1} omega_P2^{n2 k2}: P2 DFTs of length P1,
// then P1 DFTs of length P2, with no twiddle multiplications in between (all
// index maps are compile-time register renames).
template <int P1, int P2, bool INV>
__device__ __forceinline__ void dft_pfa(double2* x) {
  constexpr int P = P1 * P2;
  constexpr int t2 = inv_mod(P2 % P1, P1), t1 = inv_mod(P1 % P2, P2);
  double2 y[P];
#pragma unroll
  for (int n2 = 0; n2 < P2; ++n2) {
    double2 a[P1];
#pragma unroll
    for (int n1 = 0; n1 < P1; ++n1) a[n1] = x[(n1 * P2 + n2 * P1) % P];
    dft<P1, INV>(a);
#pragma unroll
    for (int k1 = 0; k1 < P1; ++k1) y[n2 * P1 + k1] = a[k1];
  }
#pragma unroll
  for (int k1 = 0; k1 < P1; ++k1) {
    double2 c[P2];
#pragma unroll
    for (int n2 = 0; n2 < P2; ++n2) c[n2] = y[n2 * P1 + k1];
    dft<P2, INV>(c);
#pragma unroll
    for (int k2 = 0; k2 < P2; ++k2) x[(k1 * P2 * t2 + k2 * P1 * t1) % P] = c[k2];
  }
}

template <int R, bool INV>
__device__ __forceinline__ void dft(double2* x) {
  if constexpr (R == 6) {
    dft_pfa<2, 3, INV>(x);
  } else if constexpr (R == 10) {
    dft_pfa<2, 5, INV>(x);
  } else if constexpr (R == 12) {
    dft_pfa<4, 3, INV>(x);
  } else if constexpr (R == 14) {
    dft_pfa<2, 7, INV>(x);
  } else if constexpr (R == 15) {
    dft_pfa<3, 5, INV>(x);
  } else if constexpr (R == 2) {
    dft2<INV>(x[0], x[1]);
  } else if constexpr (R == 4) {
    dft4<INV>(x[0], x[1], x[2], x[3]);
  } else if constexpr (R == 8) {
    dft8<INV>(x);
  } else if constexpr (R == 16) {
    dft16<INV>(x);
  } else {
    dft_odd<R, INV>(x);
  }
}

}  // namespace tmg
