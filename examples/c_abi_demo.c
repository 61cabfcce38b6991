/*
 * Calling the B200 products through the C ABI from plain C (no Python, no
 * torch): what a reference maintainer's shim does.
 *
 *   gcc -std=c11 -O2 -Iinclude examples/c_abi_demo.c \
 *       -Lpaper_1703_00640_b200 -ltruncmul_b200 -Wl,-rpath,$PWD/paper_1703_00640_b200 \
 *       -o c_abi_demo && ./c_abi_demo
 *
 * For n = 8192 and 2^17 bits it computes the full, low and high products of
 * two mt19937-style pseudo-random operands with tmg_full/low/high_product
 * (host buffers) and checks them against a schoolbook product computed here;
 * then shows the refusal of an over-wide parameter set
 * (TMG_ERR_PRECISION_FAILURE, the reference's ConvolutionPrecisionFailure)
 * and the escalation that recovers it.  Exit status 0 on success.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "truncmul_b200.h"

static uint64_t splitmix(uint64_t* s) {
  uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* r[0 .. na+nb) = a * b (schoolbook, 128-bit partial products) */
static void school(const uint64_t* a, size_t na, const uint64_t* b, size_t nb, uint64_t* r) {
  memset(r, 0, (na + nb) * sizeof(uint64_t));
  for (size_t i = 0; i < na; ++i) {
    unsigned __int128 c = 0;
    for (size_t j = 0; j < nb; ++j) {
      c += (unsigned __int128)a[i] * b[j] + r[i + j];
      r[i + j] = (uint64_t)c;
      c >>= 64;
    }
    r[i + nb] = (uint64_t)c;
  }
}

#define CHECK(call)                                                        \
  do {                                                                     \
    int rc_ = (call);                                                      \
    if (rc_ != TMG_OK) {                                                   \
      fprintf(stderr, "%s: %d %s\n", #call, rc_, tmg_last_error());        \
      return 1;                                                            \
    }                                                                      \
  } while (0)

static int run(tmg_context* ctx, int64_t n) {
  const size_t nl = (size_t)((n + 63) / 64);
  uint64_t* u = malloc(nl * 8);
  uint64_t* v = malloc(nl * 8);
  uint64_t* P = malloc(2 * nl * 8);
  uint64_t s = 12345 + (uint64_t)n;
  for (size_t i = 0; i < nl; ++i) {
    u[i] = splitmix(&s);
    v[i] = splitmix(&s);
  }
  school(u, nl, v, nl, P);
  int bad = 0;
  const int32_t modes[3] = {TMG_MODE_FULL, TMG_MODE_LOW, TMG_MODE_HIGH};
  for (int m = 0; m < 3; ++m) {
    tmg_params p;
    CHECK(tmg_select_params(n, modes[m], TMG_BACKEND_FFT, 4096, TMG_POLICY_ACCURATE, &p));
    const int64_t ol = tmg_output_limbs(modes[m], n);
    uint64_t* out = calloc((size_t)ol, 8);
    tmg_stats st;
    if (modes[m] == TMG_MODE_FULL) CHECK(tmg_full_product(ctx, &p, u, v, out, &st));
    if (modes[m] == TMG_MODE_LOW) CHECK(tmg_low_product(ctx, &p, u, v, out, &st));
    if (modes[m] == TMG_MODE_HIGH) CHECK(tmg_high_product(ctx, &p, u, v, out, &st));
    int ok = 1;
    if (modes[m] != TMG_MODE_HIGH) {
      for (int64_t i = 0; i < ol; ++i) ok &= out[i] == P[i];
    } else {
      /* n is a multiple of 64 here: w = floor(uv / 2^n) or that + 1 */
      const uint64_t* hi = P + nl;
      int eq = 1, plus1 = 1;
      unsigned carry = 1;
      for (size_t i = 0; i < nl; ++i) {
        eq &= out[i] == hi[i];
        const uint64_t h1 = hi[i] + carry;
        carry = carry && h1 == 0;
        plus1 &= out[i] == h1;
      }
      eq &= out[nl] == 0;
      plus1 &= out[nl] == carry;
      ok = eq || plus1;
    }
    printf("n=%lld %-4s b=%d N=%lld L=%lld residual %.4f %s\n", (long long)n,
           m == 0 ? "full" : m == 1 ? "low" : "high", p.b, (long long)p.N,
           (long long)st.transform_length, st.max_round_err, ok ? "exact" : "WRONG");
    bad |= !ok;
    free(out);
  }
  free(u);
  free(v);
  free(P);
  return bad;
}

int main(void) {
  printf("%s\n", tmg_version());
  tmg_context* ctx = NULL;
  CHECK(tmg_context_create(0, &ctx));
  int bad = run(ctx, 8192) | run(ctx, 1 << 17);

  /* unsigned 30-bit chunks of all-ones operands overflow the float budget:
   * the reference's ConvolutionPrecisionFailure, then recovered by escalation */
  const int64_t n = 3840;
  uint64_t ones[60];
  for (int i = 0; i < 60; ++i) ones[i] = ~0ull;
  tmg_params p = {n, 30, 128, 4, 0, TMG_MODE_LOW, TMG_BACKEND_FFT, 0};
  CHECK(tmg_required_precision(TMG_MODE_LOW, 30, 128, &p.p));
  uint64_t out[60];
  tmg_stats st;
  int rc = tmg_low_product(ctx, &p, ones, ones, out, &st);
  printf("b=30 unsigned: rc=%d (%s)\n", rc, rc ? tmg_last_error() : "ok");
  bad |= rc != TMG_ERR_PRECISION_FAILURE;
  /* b = 24 unsigned refuses the same way; with escalation the context
   * recomputes it at narrower balanced chunks until the tripwire passes */
  tmg_params q = {n, 24, 160, 4, 0, TMG_MODE_LOW, TMG_BACKEND_FFT, 0};
  CHECK(tmg_required_precision(TMG_MODE_LOW, 24, 160, &q.p));
  CHECK(tmg_context_set_escalation(ctx, 8));
  rc = tmg_low_product(ctx, &q, ones, ones, out, &st);
  /* (2^n - 1)^2 mod 2^n = 1 */
  int ok = rc == TMG_OK && out[0] == 1;
  for (int i = 1; i < 60; ++i) ok &= out[i] == 0;
  printf("escalated: rc=%d attempts=%d b=%d residual %.4f %s\n", rc, st.attempts, st.b,
         st.max_round_err, ok ? "exact" : "WRONG");
  bad |= !ok;
  /* the stages of the pipeline as entry points of their own: the documented
   * split of 13 into 2-bit chunks (test_products.cpp:52-64), a cyclic
   * convolution with a shifted delta, and alpha* with one series row (the
   * identity map) */
  {
    tmg_params sp = {6, 2, 3, 0, 8, TMG_MODE_FULL, TMG_BACKEND_EXACT, 0};
    const uint64_t thirteen = 13;
    int64_t chunks[3] = {-1, -1, -1};
    CHECK(tmg_split_low_i64(ctx, &sp, &thirteen, chunks));
    int sok = chunks[0] == 1 && chunks[1] == 3 && chunks[2] == 0;
    enum { CN = 8192 };
    static double f[CN], g[CN], c[CN];
    for (int i = 0; i < CN; ++i) {
      f[i] = (double)((i * 37) % 101 - 50);
      g[i] = 0.0;
    }
    g[3] = 2.0;
    CHECK(tmg_cyclic_convolve_f64(ctx, CN, f, g, c));
    int cok = 1;
    for (int i = 0; i < CN; ++i) {
      const double want = 2.0 * f[(i + CN - 3) % CN], d = c[i] - want;
      cok &= d < 1e-9 && d > -1e-9;
    }
    CHECK(tmg_alpha_star_f64(ctx, CN, 12, 1, f, c));
    int aok = 1;
    for (int i = 0; i < CN; ++i) aok &= c[i] == f[i];
    printf("entry points: split %s, convolution %s, alpha* %s\n", sok ? "ok" : "WRONG",
           cok ? "ok" : "WRONG", aok ? "ok" : "WRONG");
    bad |= !(sok && cok && aok);
  }
  tmg_context_destroy(ctx);
  printf(bad ? "FAILED\n" : "OK\n");
  return bad;
}
