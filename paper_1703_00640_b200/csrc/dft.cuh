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

// Odd prime radix via the symmetric pair formulation:
//   X_k = x0 + sum_j cos(2pi jk/p) t_j  -/+ i sum_j sin(2pi jk/p) s_j
// with t_j = x_j + x_{p-j}, s_j = x_j - x_{p-j}.
template <int P>
struct OddTrig;
template <>
struct OddTrig<3> {
  __device__ static constexpr double c(int j) { return -0.5; }
  __device__ static constexpr double s(int j) {
    return 0.8660254037844386467637232;
  }
};
template <>
struct OddTrig<5> {
  __device__ static constexpr double c(int j) {
    return j == 1 ? 0.3090169943749474241022934 : -0.8090169943749474241022934;
  }
  __device__ static constexpr double s(int j) {
    return j == 1 ? 0.9510565162951535721164393 : 0.587785252292473129168706;
  }
};
template <>
struct OddTrig<7> {
  __device__ static constexpr double c(int j) {
    return j == 1   ? 0.6234898018587335305250049
           : j == 2 ? -0.2225209339563144042889026
                    : -0.9009688679024191262361023;
  }
  __device__ static constexpr double s(int j) {
    return j == 1   ? 0.7818314824680298087084445
           : j == 2 ? 0.9749279121818236070181317
                    : 0.4338837391175581204757683;
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
  double2 x0 = x[0];
  double2 sum = x0;
#pragma unroll
  for (int j = 0; j < H; ++j) sum = cadd(sum, t[j]);
  x[0] = sum;
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    double2 a = x0, b = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      // cos/sin(2 pi j k / P): reduce jk mod P into the first half-turn
      constexpr int dummy = 0;
      (void)dummy;
      int m = (j * k) % P;
      double cj, sj;
      if (m <= H) {
        cj = OddTrig<P>::c(m);
        sj = OddTrig<P>::s(m);
      } else {
        cj = OddTrig<P>::c(P - m);
        sj = -OddTrig<P>::s(P - m);
      }
      a.x = fma(cj, t[j - 1].x, a.x);
      a.y = fma(cj, t[j - 1].y, a.y);
      b.x = fma(sj, s[j - 1].x, b.x);
      b.y = fma(sj, s[j - 1].y, b.y);
    }
    // forward: X_k = a - i b ; X_{P-k} = a + i b
    double2 ib = make_double2(-b.y, b.x);
    if (INV) {
      x[k] = cadd(a, ib);
      x[P - k] = csub(a, ib);
    } else {
      x[k] = csub(a, ib);
      x[P - k] = cadd(a, ib);
    }
  }
}

// omega_8^k multipliers (forward: e^{-i pi k/4})
template <bool INV>
__device__ __forceinline__ double2 w8_1(double2 a) {
  constexpr double r = 0.7071067811865475244008444;
  // forward: (1 - i)/sqrt2 * a ; inverse: (1 + i)/sqrt2 * a
  return INV ? make_double2((a.x - a.y) * r, (a.x + a.y) * r)
             : make_double2((a.x + a.y) * r, (a.y - a.x) * r);
}
template <bool INV>
__device__ __forceinline__ double2 w8_3(double2 a) {
  constexpr double r = 0.7071067811865475244008444;
  // forward: (-1 - i)/sqrt2 * a ; inverse: (-1 + i)/sqrt2 * a
  return INV ? make_double2((-a.x - a.y) * r, (a.x - a.y) * r)
             : make_double2((a.y - a.x) * r, (-a.x - a.y) * r);
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

// omega_16^j * a for j = 0..9 (compile-time j)
template <bool INV>
__device__ __forceinline__ double2 w16(double2 a, int j) {
  constexpr double C1 = 0.9238795325112867561281832;
  constexpr double S1 = 0.38268343236508977172846;
  constexpr double R2 = 0.7071067811865475244008444;
  double c, s;  // e^{-2 pi i j/16} = c - i s (forward)
  switch (j) {
    case 0: return a;
    case 1: c = C1; s = S1; break;
    case 2: c = R2; s = R2; break;
    case 3: c = S1; s = C1; break;
    case 4: return mul_mi<INV>(a);
    case 5: c = -S1; s = C1; break;
    case 6: c = -R2; s = R2; break;
    case 7: c = -C1; s = S1; break;
    case 8: return make_double2(-a.x, -a.y);
    default: c = -C1; s = -S1; break;  // 9
  }
  if (INV) s = -s;
  // (a.x + i a.y)(c - i s) = (a.x c + a.y s) + i (a.y c - a.x s)
  return make_double2(fma(a.x, c, a.y * s), fma(a.y, c, -a.x * s));
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
__device__ __forceinline__ void dft(double2* x) {
  if constexpr (R == 2) {
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
