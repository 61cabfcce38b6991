/*
 * CPU oracle for the truncated-product hot path — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's float pipeline
 * (arxiv 1703.00640 artifact, /root/reference/proj/core) used as the checker
 * for the CUDA path: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg are the only callers.  The product
 * path never links or calls this file.
 *
 * The reference itself cannot be built in this image (it needs gmp.h, FFTW3,
 * CMake and vendored CLI11/json/doctest headers that are absent), so the
 * oracle restates it function by function, each citing the file:line it
 * follows.  The FFT convolution (FFTW r2c/c2r in the reference,
 * convolution.cpp:175-195) is done by numpy.fft (pocketfft) in port.py.
 *
 * Differences from the reference that cannot change results:
 *   - series tables are the closed forms evaluated in long double and rounded
 *     to nearest; the reference truncates the exact rational (mpq_get_d), so
 *     entries may differ by one ulp of terms already scaled by 2^-rb.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (the generator of gen_inputs.cpp:76-83)                 */
void orc_mt19937_64(uint64_t seed, uint64_t* out, int64_t count) {
  enum { NN = 312, MM = 156 };
  const uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL;
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  uint64_t mt[NN];
  int mti;
  mt[0] = seed;
  for (mti = 1; mti < NN; mti++)
    mt[mti] = 6364136223846793005ULL * (mt[mti - 1] ^ (mt[mti - 1] >> 62)) + (uint64_t)mti;
  for (int64_t k = 0; k < count; ++k) {
    uint64_t x;
    if (mti >= NN) {
      int i;
      for (i = 0; i < NN - MM; i++) {
        x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + MM] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
      }
      for (; i < NN - 1; i++) {
        x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + (MM - NN)] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
      }
      x = (mt[NN - 1] & UM) | (mt[0] & LM);
      mt[NN - 1] = mt[MM - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
      mti = 0;
    }
    x = mt[mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    out[k] = x;
  }
}

/* ------------------------------------------------------------------------ */
/* split.cpp:66-102 (chunk_store): windows of u * 2^lead, balanced digits in
 * (-2^{b-1}, 2^{b-1}] below the top chunk, which absorbs the carry. */
static uint64_t load_limb(const uint64_t* lp, int64_t nl, int64_t i) {
  return (i >= 0 && i < nl) ? lp[i] : 0;
}

int orc_split(const uint64_t* limbs, int64_t nlimbs, int b, int64_t count,
              int balanced, int64_t lead, double* out) {
  if (b < 1 || b > 62) return -1;
  const uint64_t mask = (((uint64_t)1) << b) - 1;
  const int64_t half = ((int64_t)1) << (b - 1);
  const int64_t body = balanced ? count - 1 : 0;
  int64_t carry = 0;
  for (int64_t i = 0; i < count; ++i) {
    const int64_t pos = i * b - lead;
    const int64_t idx = pos >> 6;
    const unsigned sh = (unsigned)(pos & 63);
    uint64_t w;
    if (idx >= 0) {
      w = load_limb(limbs, nlimbs, idx) >> sh;
      if (sh != 0) w |= load_limb(limbs, nlimbs, idx + 1) << (64u - sh);
      w &= mask;
    } else if (idx == -1 && sh != 0) {
      w = (load_limb(limbs, nlimbs, 0) << (64u - sh)) & mask;
    } else {
      w = 0;
    }
    const int64_t x = (int64_t)w + carry;
    if (i < body) {
      const int64_t d = x > half ? 1 : 0;
      out[i] = (double)(x - (d << b));
      carry = d;
    } else {
      out[i] = (double)x;
      carry = 0;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* series.cpp:146-228: coefficient tables, row r = 0..lam-1, N entries each.
 * fam: 0 alpha, 1 beta, 2 gamma, 3 delta. */
int orc_coeff_table(int fam, int64_t lam, int64_t N, int b, double* out) {
  for (int64_t r = 0; r < lam; ++r) {
    long double den = 1.0L;
    for (int64_t i = 1; i <= r; ++i) den *= (long double)i * (long double)N;
    den = ldexpl(den, (int)(r * b));
    for (int64_t k = 0; k < N; ++k) {
      long double v;
      if (r == 0) {
        v = 1.0L;
      } else if (fam == 0 || fam == 2) {
        long double p = (long double)k;
        const long double sg = fam == 0 ? -1.0L : 1.0L;
        for (int64_t i = 0; i < r - 1; ++i)
          p *= (long double)k + (long double)r + sg * (long double)N * (long double)(i + 1);
        v = p / den;
        if (fam == 0 && (r & 1)) v = -v;
      } else {
        long double p = (long double)k;
        const long double sg = fam == 1 ? 1.0L : -1.0L;
        for (int64_t i = 1; i < r; ++i) p *= (long double)k + sg * (long double)N * (long double)i;
        v = p / den;
        if (fam == 3 && (r & 1)) v = -v;
      }
      out[r * N + k] = (double)v;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* maps_f64.cpp:21-38 (detect_shape) */
typedef struct {
  int identity_row0, linear_row1;
  double slope1;
} Shape;

static Shape detect_shape(const double* t, int64_t R, int64_t N) {
  Shape s = {0, 0, 0.0};
  if (R == 0 || N < 2) return s;
  s.identity_row0 = 1;
  for (int64_t k = 0; k < N; ++k)
    if (t[k] != 1.0) { s.identity_row0 = 0; break; }
  if (R >= 2) {
    const double* r1 = t + N;
    const double c = r1[1];
    int ok = r1[0] == 0.0;
    for (int64_t k = 1; ok && k < N; ++k) ok = (double)k * c == r1[k];
    s.linear_row1 = ok;
    s.slope1 = c;
  }
  return s;
}

/* maps_f64.cpp:48-96 (apply_series) */
static void apply_series(const double* t, int64_t R, Shape sh, int64_t N,
                         const double* in, double* out) {
  if (R == 4 && N >= 4) {
    const double *r0 = t, *r1 = t + N, *r2 = t + 2 * N, *r3 = t + 3 * N;
    for (int64_t j = 0; j < 3; ++j) {
      const int64_t k1 = j - 1 < 0 ? j - 1 + N : j - 1;
      const int64_t k2 = j - 2 < 0 ? j - 2 + N : j - 2;
      const int64_t k3 = j - 3 < 0 ? j - 3 + N : j - 3;
      out[j] = in[j] * r0[j] + in[k1] * r1[k1] + in[k2] * r2[k2] + in[k3] * r3[k3];
    }
    if (sh.identity_row0 && sh.linear_row1) {
      const double c = sh.slope1;
      for (int64_t j = 3; j < N; ++j)
        out[j] = in[j] + in[j - 1] * ((double)(j - 1) * c) + in[j - 2] * r2[j - 2] +
                 in[j - 3] * r3[j - 3];
    } else if (sh.identity_row0) {
      for (int64_t j = 3; j < N; ++j)
        out[j] = in[j] + in[j - 1] * r1[j - 1] + in[j - 2] * r2[j - 2] + in[j - 3] * r3[j - 3];
    } else {
      for (int64_t j = 3; j < N; ++j)
        out[j] = in[j] * r0[j] + in[j - 1] * r1[j - 1] + in[j - 2] * r2[j - 2] +
                 in[j - 3] * r3[j - 3];
    }
    return;
  }
  for (int64_t j = 0; j < N; ++j) {
    double acc = 0.0;
    for (int64_t r = 0; r < R; ++r) {
      int64_t k = (j - r) % N;
      if (k < 0) k += N;
      acc += in[k] * t[r * N + k];
    }
    out[j] = acc;
  }
}

/* maps_f64.cpp:103-136 (apply_series_inplace4) */
static void apply_series_inplace4(const double* t, Shape sh, int64_t N, double* buf) {
  const double *r0 = t, *r1 = t + N, *r2 = t + 2 * N, *r3 = t + 3 * N;
  const double o0 = buf[0] * r0[0] + buf[N - 1] * r1[N - 1] + buf[N - 2] * r2[N - 2] +
                    buf[N - 3] * r3[N - 3];
  const double o1 = buf[1] * r0[1] + buf[0] * r1[0] + buf[N - 1] * r2[N - 1] +
                    buf[N - 2] * r3[N - 2];
  const double o2 = buf[2] * r0[2] + buf[1] * r1[1] + buf[0] * r2[0] + buf[N - 1] * r3[N - 1];
  if (sh.identity_row0 && sh.linear_row1) {
    const double c = sh.slope1;
    for (int64_t j = N - 1; j >= 3; --j)
      buf[j] = buf[j] + buf[j - 1] * ((double)(j - 1) * c) + buf[j - 2] * r2[j - 2] +
               buf[j - 3] * r3[j - 3];
  } else if (sh.identity_row0) {
    for (int64_t j = N - 1; j >= 3; --j)
      buf[j] = buf[j] + buf[j - 1] * r1[j - 1] + buf[j - 2] * r2[j - 2] + buf[j - 3] * r3[j - 3];
  } else {
    for (int64_t j = N - 1; j >= 3; --j)
      buf[j] = buf[j] * r0[j] + buf[j - 1] * r1[j - 1] + buf[j - 2] * r2[j - 2] +
               buf[j - 3] * r3[j - 3];
  }
  buf[0] = o0;
  buf[1] = o1;
  buf[2] = o2;
}

/* maps_f64.cpp:140-188 (apply_series_flat): buf has N + R - 1 entries */
static void apply_series_flat(const double* t, int64_t R, Shape sh, int64_t N,
                              const double* in, double* buf) {
  if (R == 4 && N >= 4) {
    const double *r0 = t, *r1 = t + N, *r2 = t + 2 * N, *r3 = t + 3 * N;
    buf[0] = in[0] * r0[0];
    buf[1] = in[1] * r0[1] + in[0] * r1[0];
    buf[2] = in[2] * r0[2] + in[1] * r1[1] + in[0] * r2[0];
    if (sh.identity_row0 && sh.linear_row1) {
      const double c = sh.slope1;
      for (int64_t j = 3; j < N; ++j)
        buf[j] = in[j] + in[j - 1] * ((double)(j - 1) * c) + in[j - 2] * r2[j - 2] +
                 in[j - 3] * r3[j - 3];
    } else if (sh.identity_row0) {
      for (int64_t j = 3; j < N; ++j)
        buf[j] = in[j] + in[j - 1] * r1[j - 1] + in[j - 2] * r2[j - 2] + in[j - 3] * r3[j - 3];
    } else {
      for (int64_t j = 3; j < N; ++j)
        buf[j] = in[j] * r0[j] + in[j - 1] * r1[j - 1] + in[j - 2] * r2[j - 2] +
                 in[j - 3] * r3[j - 3];
    }
    buf[N] = in[N - 1] * r1[N - 1] + in[N - 2] * r2[N - 2] + in[N - 3] * r3[N - 3];
    buf[N + 1] = in[N - 1] * r2[N - 1] + in[N - 2] * r3[N - 2];
    buf[N + 2] = in[N - 1] * r3[N - 1];
    return;
  }
  for (int64_t j = 0; j < N + R - 1; ++j) {
    double acc = 0.0;
    const int64_t rlo = j - N + 1 > 0 ? j - N + 1 : 0;
    const int64_t rhi = R - 1 < j ? R - 1 : j;
    for (int64_t r = rlo; r <= rhi; ++r) acc += in[j - r] * t[r * N + (j - r)];
    buf[j] = acc;
  }
}

/* maps_f64.cpp:259-267 (alpha_star_inplace_f64) */
int orc_alpha_star_inplace(const double* t, int64_t R, int64_t N, double* buf) {
  Shape sh = detect_shape(t, R, N);
  if (R == 4 && N >= 4) {
    apply_series_inplace4(t, sh, N, buf);
    return 0;
  }
  double* tmp = (double*)malloc(sizeof(double) * (size_t)N);
  if (!tmp) return -1;
  memcpy(tmp, buf, sizeof(double) * (size_t)N);
  apply_series(t, R, sh, N, tmp, buf);
  free(tmp);
  return 0;
}

/* maps_f64.cpp:269-281 (beta_star_view_f64): out gets N entries */
int orc_beta_star(const double* t, int64_t R, int64_t N, int b, const double* in, double* out) {
  Shape sh = detect_shape(t, R, N);
  const int64_t size = N + R - 1;
  double* buf = (double*)malloc(sizeof(double) * (size_t)size);
  if (!buf) return -1;
  apply_series_flat(t, R, sh, N, in, buf);
  const double step = ldexp(1.0, -b);
  for (int64_t j = size - 1; j >= N; --j) {
    const double c = buf[j];
    if (c == 0.0) continue;
    buf[j - N] += c;
    buf[j - N + 1] -= c * step;
  }
  memcpy(out, buf, sizeof(double) * (size_t)N);
  free(buf);
  return 0;
}

/* High-product constants (maps_f64.cpp:209-243). */
typedef struct {
  double root, inv_root, root_neg_n, cofactor_scaled;
  int64_t nfold;
  double fold[128];
} HighConsts;

static void high_consts(int64_t N, int b, HighConsts* h) {
  const int64_t total_bits = N * (int64_t)b;
  h->nfold = 0;
  if (total_bits >= 64) {
    h->root = ldexp(1.0, b);
    h->inv_root = ldexp(1.0, -b);
    const int neg = (int)(total_bits < 1100 ? total_bits : 1100);
    h->root_neg_n = ldexp(1.0, -neg);
    h->cofactor_scaled = 1.0 - (double)N * h->root_neg_n;
    for (int64_t i = 0; i < N && i * b <= 80 && h->nfold < 128; ++i)
      h->fold[h->nfold++] = ldexp(1.0, (int)(-i * b));
  } else {
    /* compute_aux_root (maps.cpp:31-63) by Newton in long double */
    long double top = ldexpl(1.0L, b), x = top;
    for (int it = 0; it < 200; ++it) {
      long double xn = powl(x, (long double)N);
      long double val = xn * (x - top) + top;
      long double slope = powl(x, (long double)(N - 1)) * ((N + 1) * x - N * top);
      if (slope == 0) break;
      long double nx = x - val / slope;
      if (nx > top) nx = top;
      if (fabsl(nx - x) <= ldexpl(fabsl(x), -62)) { x = nx; break; }
      x = nx;
    }
    h->root = (double)x;
    h->inv_root = 1.0 / h->root;
    double ipow = h->inv_root;
    for (int64_t i = 0; i < N && h->nfold < 128; ++i) {
      h->fold[h->nfold++] = ldexp(ipow, b);
      ipow *= h->inv_root;
    }
    double inv_n = 1.0;
    for (int64_t i = 0; i < N; ++i) inv_n *= h->inv_root;
    h->root_neg_n = inv_n;
    h->cofactor_scaled = 1.0 - (double)N * ldexp(inv_n * h->inv_root, b);
  }
}

/* maps_f64.cpp:317-348 (gamma_dagger_inplace_f64): buf holds N + 1 */
int orc_gamma_dagger_inplace(const double* t, int64_t R, int64_t N, int b, double* buf,
                             double* aux) {
  HighConsts h;
  high_consts(N, b, &h);
  Shape sh = detect_shape(t, R, N);
  double acc = 0.0, ipow = 1.0;
  for (int64_t d = 0; d <= N; ++d) {
    acc += buf[N - d] * ipow;
    ipow *= h.inv_root;
    if (ipow < 1e-30) break;
  }
  *aux = acc;
  const double top = buf[N];
  if (R == 4 && N >= 4) {
    apply_series_inplace4(t, sh, N, buf);
  } else {
    double* tmp = (double*)malloc(sizeof(double) * (size_t)N);
    if (!tmp) return -1;
    memcpy(tmp, buf, sizeof(double) * (size_t)N);
    apply_series(t, R, sh, N, tmp, buf);
    free(tmp);
  }
  if (top != 0.0) {
    for (int64_t r = 0; r < R; ++r) {
      const double* row = t + r * N;
      for (int64_t k = 0; k < h.nfold; ++k) {
        const int64_t j = (k + r) % N;
        buf[j] += top * h.fold[k] * row[k];
      }
    }
  }
  return 0;
}

/* maps_f64.cpp:350-384 (delta_dagger_view_f64): out gets N + 1 entries */
int orc_delta_dagger(const double* t, int64_t R, int64_t N, int b, const double* in,
                     double aux, double* out) {
  HighConsts h;
  high_consts(N, b, &h);
  Shape sh = detect_shape(t, R, N);
  const int64_t size = N + R - 1;
  const int64_t bsz = size > N + 1 ? size : N + 1;
  double* buf = (double*)calloc((size_t)bsz, sizeof(double));
  if (!buf) return -1;
  apply_series_flat(t, R, sh, N, in, buf);
  for (int64_t j = size - 1; j >= N; --j) {
    const double c = buf[j];
    if (c == 0.0) continue;
    for (int64_t i = 0; i < h.nfold; ++i) buf[j - N + i] += c * h.fold[i];
  }
  double hrho = 0.0, ipow = h.inv_root;
  for (int64_t d = 1; d <= N; ++d) {
    hrho += buf[N - d] * ipow;
    ipow *= h.inv_root;
    if (ipow < 1e-30) break;
  }
  const double psi = (aux - hrho * h.root_neg_n) / h.cofactor_scaled;
  const double step = ldexp(1.0, -b);
  buf[N] = psi - buf[N - 1] * step;
  for (int64_t i = N - 1; i >= 1; --i) buf[i] = buf[i] - buf[i - 1] * step;
  for (int64_t i = 0; i < h.nfold; ++i) buf[i] -= psi * h.fold[i];
  memcpy(out, buf, sizeof(double) * (size_t)(N + 1));
  free(buf);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* products_f64.cpp:16-102: round vals[i] * 2^scale (tripwire: |x| >= 2^53 or
 * residual above a quarter) and accumulate at bit offset i * b into signed
 * 128-bit lanes, then one carry pass.  Writes the two's-complement limbs of
 * the sum (nout limbs, little endian) and the sign (0 or -1) of the value.
 * Returns 0, 1 (overflow tripwire) or 2 (quarter tripwire). */
int orc_round_accumulate(const double* vals, int64_t count, int scale, int b,
                         uint64_t* out, int64_t nout, int64_t* sign_out,
                         double* max_err, double* max_abs) {
  const int64_t nlanes = (count * (int64_t)b + 128) / 64 + 3;
  i128* lanes = (i128*)calloc((size_t)nlanes, sizeof(i128));
  if (!lanes) return -1;
  const double factor = ldexp(1.0, scale);
  double me = 0.0, ma = 0.0;
  int status = 0;
  for (int64_t i = 0; i < count; ++i) {
    const double x = vals[i] * factor;
    const double ax = fabs(x);
    if (!(ax < 9007199254740992.0)) {
      status = 1;
      ma = 1e308;
      break;
    }
    const double r = nearbyint(x);
    const double e = fabs(x - r);
    if (e > me) me = e;
    if (ax > ma) ma = ax;
    if (e > 0.25 && status == 0) status = 2;
    const int64_t bit = i * (int64_t)b;
    lanes[bit >> 6] += ((i128)(int64_t)r) << (unsigned)(bit & 63);
  }
  *max_err = me;
  *max_abs = ma;
  i128 carry = 0;
  for (int64_t i = 0; i < nlanes; ++i) {
    const i128 s = lanes[i] + carry;
    if (i < nout) out[i] = (uint64_t)s;
    carry = s >> 64;
  }
  for (int64_t i = nlanes; i < nout; ++i) out[i] = (uint64_t)carry;
  *sign_out = carry < 0 ? -1 : 0;
  free(lanes);
  return status;
}

/* ------------------------------------------------------------------------ */
/* oracle.cpp:69-130 (limb_mul): schoolbook below 24 limbs, Karatsuba above,
 * on plain little-endian limb arrays (no shared code with GMP). */
static void school_mul(const uint64_t* a, int64_t na, const uint64_t* b, int64_t nb,
                       uint64_t* r) {
  memset(r, 0, sizeof(uint64_t) * (size_t)(na + nb));
  for (int64_t i = 0; i < na; ++i) {
    if (a[i] == 0) continue;
    uint64_t carry = 0;
    for (int64_t j = 0; j < nb; ++j) {
      u128 cur = (u128)a[i] * b[j] + r[i + j] + carry;
      r[i + j] = (uint64_t)cur;
      carry = (uint64_t)(cur >> 64);
    }
    r[i + nb] = carry;
  }
}

/* r = a + b (na >= nb), returns carry */
static uint64_t add_n(uint64_t* r, const uint64_t* a, int64_t na, const uint64_t* b,
                      int64_t nb) {
  uint64_t c = 0;
  for (int64_t i = 0; i < na; ++i) {
    u128 s = (u128)a[i] + (i < nb ? b[i] : 0) + c;
    r[i] = (uint64_t)s;
    c = (uint64_t)(s >> 64);
  }
  return c;
}
/* a -= b in place (na >= nb, a >= b) */
static void sub_in(uint64_t* a, int64_t na, const uint64_t* b, int64_t nb) {
  uint64_t br = 0;
  for (int64_t i = 0; i < na; ++i) {
    u128 d = (u128)a[i] - (i < nb ? b[i] : 0) - br;
    a[i] = (uint64_t)d;
    br = (uint64_t)(d >> 64) ? 1 : 0;
  }
}
/* acc[off..] += src */
static void add_at(uint64_t* acc, int64_t nacc, const uint64_t* src, int64_t ns, int64_t off) {
  uint64_t c = 0;
  int64_t i = 0;
  for (; i < ns; ++i) {
    u128 s = (u128)acc[off + i] + src[i] + c;
    acc[off + i] = (uint64_t)s;
    c = (uint64_t)(s >> 64);
  }
  for (; c && off + i < nacc; ++i) {
    u128 s = (u128)acc[off + i] + c;
    acc[off + i] = (uint64_t)s;
    c = (uint64_t)(s >> 64);
  }
}

/* balanced Karatsuba for equal lengths n; r has 2n limbs */
static void kara(const uint64_t* a, const uint64_t* b, int64_t n, uint64_t* r) {
  if (n < 24) {
    school_mul(a, n, b, n, r);
    return;
  }
  const int64_t h = n / 2, hh = n - h;  /* low h limbs, high hh limbs */
  uint64_t* sa = (uint64_t*)calloc((size_t)(hh + 1), 8);
  uint64_t* sb = (uint64_t*)calloc((size_t)(hh + 1), 8);
  uint64_t* z1 = (uint64_t*)calloc((size_t)(2 * hh + 2), 8);
  sa[hh] = add_n(sa, a + h, hh, a, h);
  sb[hh] = add_n(sb, b + h, hh, b, h);
  kara(a, b, h, r);                /* z0 -> r[0..2h) */
  kara(a + h, b + h, hh, r + 2 * h); /* z2 -> r[2h..2n) */
  kara(sa, sb, hh + 1, z1);        /* (a0+a1)(b0+b1) */
  sub_in(z1, 2 * hh + 2, r, 2 * h);
  sub_in(z1, 2 * hh + 2, r + 2 * h, 2 * hh);
  add_at(r, 2 * n, z1, 2 * hh + 2 > 2 * n - h ? 2 * n - h : 2 * hh + 2, h);
  free(sa);
  free(sb);
  free(z1);
}

/* r gets na + nb limbs (both operands padded to the longer length inside). */
int orc_limb_mul(const uint64_t* a, int64_t na, const uint64_t* b, int64_t nb, uint64_t* r) {
  const int64_t n = na > nb ? na : nb;
  if (n == 0) return 0;
  uint64_t* pa = (uint64_t*)calloc((size_t)n, 8);
  uint64_t* pb = (uint64_t*)calloc((size_t)n, 8);
  uint64_t* pr = (uint64_t*)calloc((size_t)(2 * n), 8);
  if (!pa || !pb || !pr) return -1;
  memcpy(pa, a, (size_t)na * 8);
  memcpy(pb, b, (size_t)nb * 8);
  kara(pa, pb, n, pr);
  memcpy(r, pr, (size_t)(na + nb) * 8);
  free(pa);
  free(pb);
  free(pr);
  return 0;
}
