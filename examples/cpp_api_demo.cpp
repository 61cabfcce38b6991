/*
 * The C++ host API (include/truncmul_b200.hpp, the reference's products.hpp
 * names over the C-ABI) from a C++ program: what a reference user switching
 * to the B200 path writes.
 *
 *   g++ -std=c++17 -O2 -Iinclude examples/cpp_api_demo.cpp \
 *       -Lpaper_1703_00640_b200 -ltruncmul_b200 -Wl,-rpath,$PWD/paper_1703_00640_b200 \
 *       -o cpp_api_demo && ./cpp_api_demo
 *
 * With TMG_DEMO_PARAMS_ONLY set it exercises the parameter functions only
 * (no GPU needed) and exits 0 after "params OK"; otherwise it also checks
 * full/low/high products against a schoolbook product computed here and
 * the reference's exception classes, and prints "OK".
 */
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "truncmul_b200.hpp"

namespace tb = truncmul_b200;

static std::uint64_t splitmix(std::uint64_t& s) {
  std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static tb::Limbs school(const tb::Limbs& a, const tb::Limbs& b) {
  tb::Limbs r(a.size() + b.size(), 0);
  for (size_t i = 0; i < a.size(); ++i) {
    unsigned __int128 c = 0;
    for (size_t j = 0; j < b.size(); ++j) {
      c += static_cast<unsigned __int128>(a[i]) * b[j] + r[i + j];
      r[i + j] = static_cast<std::uint64_t>(c);
      c >>= 64;
    }
    r[i + b.size()] = static_cast<std::uint64_t>(c);
  }
  return r;
}

#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAILED %s (line %d)\n", #c, __LINE__);           \
      return 1;                                                    \
    }                                                              \
  } while (0)

int main() {
  // parameters: no device needed
  const std::int64_t n = 1 << 17;
  const tb::Params pf = tb::select_params(n, tb::Mode::kFull);
  const tb::Params pl = tb::select_params(n, tb::Mode::kLow);
  const tb::Params ph = tb::select_params(n, tb::Mode::kHigh);
  tb::validate_params(pf);
  tb::validate_params(pl);
  tb::validate_params(ph);
  CHECK(pf.lambda == 0 && pl.lambda > 0 && ph.lambda > 0);
  CHECK(tb::required_precision(pl.mode, pl.b, pl.N) == pl.p);
  CHECK(tb::select_params(1000, tb::Mode::kLow).mode == tb::Mode::kOracleFallback);
  // the default policy is the reference's params.cpp (test_products.cpp:179-197,
  // products.hpp:60-61); the accurate policy is an explicit opt-in
  {
    const tb::Params r = tb::select_params(1000000, tb::Mode::kLow, tb::Backend::kFft);
    CHECK(r.b == 14 && r.N == 71680 && r.lambda == 4 && r.p == 65);
    const tb::Params a = tb::select_params(1000000, tb::Mode::kLow, tb::Backend::kFft,
                                           tb::kDefaultFallbackCutoff, tb::Policy::kAccurate);
    CHECK(a.b == 13);
  }
  bool threw = false;
  try {
    tb::Params bad = pl;
    bad.N = 3;  // does not cover n
    tb::validate_params(bad);
  } catch (const tb::InputOutOfRange&) {
    threw = true;
  } catch (const tb::UnsupportedLength&) {
    threw = true;
  }
  CHECK(threw);
  std::printf("params OK (n = %lld: full b=%d N=%lld, low b=%d N=%lld lambda=%lld)\n",
              static_cast<long long>(n), pf.b, static_cast<long long>(pf.N), pl.b,
              static_cast<long long>(pl.N), static_cast<long long>(pl.lambda));
  if (std::getenv("TMG_DEMO_PARAMS_ONLY")) return 0;

  // products on the GPU
  std::uint64_t seed = 42;
  const size_t nl = static_cast<size_t>((n + 63) / 64);
  tb::Limbs u(nl), v(nl);
  for (size_t i = 0; i < nl; ++i) {
    u[i] = splitmix(seed);
    v[i] = splitmix(seed);
  }
  const tb::Limbs P = school(u, v);
  tb::Context ctx(0);
  const tb::Limbs full = ctx.full_product(u, v, pf);
  CHECK(full.size() == 2 * nl);
  for (size_t i = 0; i < full.size(); ++i) CHECK(full[i] == P[i]);
  const tb::Limbs low = tb::low_product(u, v, pl);  // free function, default context
  CHECK(low.size() == nl);
  for (size_t i = 0; i < nl; ++i) CHECK(low[i] == P[i]);
  const tb::Limbs high = ctx.high_product(u, v, ph);
  // |uv - 2^n w| < 2^n with n a multiple of 64: w = P >> n or P >> n plus one
  CHECK(high.size() == nl + 1);
  bool eq = true;
  for (size_t i = 0; i < nl; ++i) eq = eq && high[i] == P[nl + i];
  tb::Limbs w1(P.begin() + nl, P.end());
  w1.push_back(0);
  unsigned __int128 c = 1;
  for (auto& x : w1) {
    c += x;
    x = static_cast<std::uint64_t>(c);
    c >>= 64;
  }
  bool eq1 = true;
  for (size_t i = 0; i <= nl; ++i) eq1 = eq1 && high[i] == w1[i];
  CHECK((eq && high[nl] == 0) || eq1);
  std::printf("products OK (n = %lld: max round err full %.4f, high %.4f)\n",
              static_cast<long long>(n), ctx.last_stats().max_round_err,
              ctx.last_stats().max_round_err);

  // the machine-word splitters (products.hpp:77-79): the reference's documented
  // examples (test_products.cpp:52-78), and a low split of u reassembled
  {
    tb::Params sp;
    sp.n = 6; sp.b = 2; sp.N = 3; sp.mode = tb::Mode::kFull; sp.backend = tb::Backend::kExact;
    sp.signed_split = false;  // like the reference tests' manual_params
    const std::vector<std::int64_t> w = ctx.split_low_i64(tb::Limbs{13}, sp);
    CHECK(w.size() == 3 && w[0] == 1 && w[1] == 3 && w[2] == 0);
    tb::Params hp;
    hp.n = 10; hp.b = 4; hp.N = 3; hp.mode = tb::Mode::kHigh; hp.backend = tb::Backend::kExact;
    hp.signed_split = false;
    const std::vector<std::int64_t> h = tb::split_high_i64(tb::Limbs{1023}, hp);
    CHECK(h.size() == 4 && h[0] == 0 && h[1] == 12 && h[2] == 15 && h[3] == 15);
    const std::vector<std::int64_t> z = ctx.split_low_i64(u, pl);
    CHECK(static_cast<std::int64_t>(z.size()) == pl.N);
    // sum_i z_i 2^{i b} == u, accumulated limb by limb with signed carries
    tb::Limbs back(nl + 1, 0);
    for (size_t i = 0; i < z.size(); ++i) {
      const std::int64_t pos = static_cast<std::int64_t>(i) * pl.b;
      __int128 val = static_cast<__int128>(z[i]) << (pos & 63);
      for (size_t m = static_cast<size_t>(pos >> 6); m <= nl && val != 0; ++m) {
        const __int128 t = static_cast<__int128>(back[m]) + static_cast<std::uint64_t>(val);
        back[m] = static_cast<std::uint64_t>(t);
        val = (val >> 64) + static_cast<__int128>(t >> 64);
      }
    }
    for (size_t i = 0; i < nl; ++i) CHECK(back[i] == u[i]);
    std::printf("splits OK\n");
  }

  // the reference's exceptions
  threw = false;
  try {
    tb::Limbs big = u;
    big.pop_back();
    ctx.low_product(big, v, pl);
  } catch (const tb::InputOutOfRange&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    tb::Params wide = pl;
    wide.b = 30;  // far beyond the float budget: the rounding tripwire fires
    wide.N = (n + wide.b - 1) / wide.b;
    wide.p = tb::required_precision(wide.mode, wide.b, wide.N);
    wide.lambda = tb::default_lambda(wide.mode, wide.backend, wide.b, wide.p);
    ctx.low_product(u, v, wide);
  } catch (const tb::ConvolutionPrecisionFailure&) {
    threw = true;
  } catch (const tb::UnsupportedLength&) {
    threw = true;  // no 2357-smooth length at that N
  }
  CHECK(threw);
  std::printf("OK\n");
  return 0;
}
