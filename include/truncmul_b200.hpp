// C++ host API of the B200 truncated-product path, mirroring the reference's
// proj/core interface (include/truncmul/products.hpp, errors.hpp) over the
// C-ABI of truncmul_b200.h.  Header-only: every function is a thin inline
// wrapper that converts types, calls the C entry point and turns a TMG_ERR_*
// return code into the exception class the reference throws.
//
//   reference (products.hpp)                 here
//   Mode / Backend / Params (25-34)          Mode / Backend / Params
//   required_precision (40)                  required_precision
//   default_lambda (44-45)                   default_lambda
//   validate_params (52)                     validate_params
//   select_params (60-61)                    select_params (+ Policy)
//   full/low/high_product (91-93)            full/low/high_product on
//     BigInt operands                          little-endian uint64 limb
//                                              vectors (BigInt::to_limbs,
//                                              bigint.hpp:113-115)
//   errors.hpp:9-67 exception classes         same names, same messages
//
// The products run on a Context (one CUDA device, one stream, a reusable
// workspace); the free functions use a thread-local default context on
// device 0, as the reference's functions need no handle.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "truncmul_b200.h"

namespace truncmul_b200 {

// ---- errors (errors.hpp) ----
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& m) : std::runtime_error(m) {}
};
class InputOutOfRange : public Error {
 public:
  using Error::Error;
};
class NoValidParams : public Error {
 public:
  using Error::Error;
};
class UnsupportedLength : public Error {
 public:
  using Error::Error;
};
class ConvolutionPrecisionFailure : public Error {
 public:
  using Error::Error;
};
class PlanMismatch : public Error {
 public:
  using Error::Error;
};
// Not in the reference: a parameter set the GPU path refuses (the exact
// backend), and CUDA runtime failures.
class Unsupported : public Error {
 public:
  using Error::Error;
};
class CudaError : public Error {
 public:
  using Error::Error;
};

inline void check(int rc) {
  if (rc == TMG_OK) return;
  const std::string m = tmg_last_error();
  switch (rc) {
    case TMG_ERR_INPUT_OUT_OF_RANGE: throw InputOutOfRange(m);
    case TMG_ERR_NO_VALID_PARAMS: throw NoValidParams(m);
    case TMG_ERR_UNSUPPORTED_LENGTH: throw UnsupportedLength(m);
    case TMG_ERR_PRECISION_FAILURE: throw ConvolutionPrecisionFailure(m);
    case TMG_ERR_PLAN_MISMATCH: throw PlanMismatch(m);
    case TMG_ERR_UNSUPPORTED: throw Unsupported(m);
    case TMG_ERR_CUDA: throw CudaError(m);
    default: throw Error(m);
  }
}

// ---- parameters (products.hpp:14-61) ----
enum class Mode : std::int32_t { kFull = 0, kLow = 1, kHigh = 2, kOracleFallback = 3 };
enum class Backend : std::int32_t { kExact = TMG_BACKEND_EXACT, kFft = TMG_BACKEND_FFT };
// kReference (the default, as products.hpp:60-61) reproduces the reference's
// params.cpp; kAccurate is an opt-in that adds the predicted-error bound and
// the GPU cost model (Numerics).
enum class Policy : std::int32_t { kReference = TMG_POLICY_REFERENCE, kAccurate = TMG_POLICY_ACCURATE };

inline constexpr std::int64_t kDefaultFallbackCutoff = 4096;

struct Params {
  std::int64_t n = 0;
  std::int32_t b = 0;
  std::int64_t N = 0;
  std::int64_t lambda = 0;
  std::int32_t p = 0;
  Mode mode = Mode::kFull;
  Backend backend = Backend::kFft;
  bool signed_split = true;

  tmg_params to_c() const {
    tmg_params q{};
    q.n = n;
    q.b = b;
    q.N = N;
    q.lambda = lambda;
    q.p = p;
    q.mode = static_cast<std::int32_t>(mode);
    q.backend = static_cast<std::int32_t>(backend);
    q.signed_split = signed_split ? 1 : 0;
    return q;
  }
  static Params from_c(const tmg_params& q) {
    Params r;
    r.n = q.n;
    r.b = q.b;
    r.N = q.N;
    r.lambda = q.lambda;
    r.p = q.p;
    r.mode = static_cast<Mode>(q.mode);
    r.backend = static_cast<Backend>(q.backend);
    r.signed_split = q.signed_split != 0;
    return r;
  }
};

inline std::int32_t required_precision(Mode mode, std::int32_t b, std::int64_t N) {
  std::int32_t out = 0;
  check(tmg_required_precision(static_cast<std::int32_t>(mode), b, N, &out));
  return out;
}

inline std::int64_t default_lambda(Mode mode, Backend backend, std::int32_t b, std::int32_t p) {
  std::int64_t out = 0;
  check(tmg_default_lambda(static_cast<std::int32_t>(mode), static_cast<std::int32_t>(backend), b, p,
                           &out));
  return out;
}

inline void validate_params(const Params& params) {
  const tmg_params q = params.to_c();
  check(tmg_validate_params(&q));
}

inline Params select_params(std::int64_t n, Mode mode, Backend backend = Backend::kFft,
                            std::int64_t fallback_cutoff = kDefaultFallbackCutoff,
                            Policy policy = Policy::kReference) {
  tmg_params q{};
  check(tmg_select_params(n, static_cast<std::int32_t>(mode), static_cast<std::int32_t>(backend),
                          fallback_cutoff, static_cast<std::int32_t>(policy), &q));
  return Params::from_c(q);
}

// Limbs of a product result: ceil(2n/64) full, ceil(n/64) low, ceil((n+1)/64) high.
inline std::int64_t output_limbs(Mode mode, std::int64_t n) {
  return tmg_output_limbs(static_cast<std::int32_t>(mode), n);
}

using Limbs = std::vector<std::uint64_t>;  // little-endian 64-bit limbs
using Stats = tmg_stats;

// ---- products ----
class Context {
 public:
  explicit Context(int device = 0) { check(tmg_context_create(device, &h_)); }
  ~Context() { tmg_context_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  tmg_context* handle() const { return h_; }
  // run on a caller-owned cudaStream_t (passed as void*)
  void set_stream(void* stream) { check(tmg_context_set_stream(h_, stream)); }
  // recompute a refused product at chunk width b - 1, up to k times (off = 0)
  void set_escalation(int k) { check(tmg_context_set_escalation(h_, k)); }
  void synchronize() { check(tmg_synchronize(h_)); }

  // u v exactly (products.hpp:91)
  Limbs full_product(const Limbs& u, const Limbs& v, const Params& p) {
    return run(tmg_full_product, Mode::kFull, u, v, p);
  }
  // u v mod 2^n (products.hpp:92)
  Limbs low_product(const Limbs& u, const Limbs& v, const Params& p) {
    return run(tmg_low_product, Mode::kLow, u, v, p);
  }
  // w with |u v - 2^n w| < 2^n and 0 <= w <= 2^n (products.hpp:93)
  Limbs high_product(const Limbs& u, const Limbs& v, const Params& p) {
    return run(tmg_high_product, Mode::kHigh, u, v, p);
  }

  // FP64 cyclic convolution of two sequences of one {2,3,5,7}-smooth length
  // (cyclic_convolve_f64 on an FFT plan, convolution.hpp:64-67)
  std::vector<double> cyclic_convolve_f64(const std::vector<double>& f,
                                          const std::vector<double>& g) {
    if (f.size() != g.size()) throw PlanMismatch("cyclic_convolve_f64: operand lengths differ");
    std::vector<double> out(f.size());
    check(tmg_cyclic_convolve_f64(h_, static_cast<std::int64_t>(f.size()), f.data(), g.data(),
                                  out.data()));
    return out;
  }

  // The ring-change maps on FP64 sequences (maps_f64.hpp): alpha* and beta*
  // (N -> N), gamma-dagger (N + 1 -> N and the root channel), delta-dagger
  // (N and aux -> N + 1), for the series tables of (N, b, lambda).
  std::vector<double> alpha_star_f64(std::int64_t N, std::int32_t b, std::int64_t lambda,
                                     const std::vector<double>& in) {
    need(in, N, "alpha_star_f64");
    std::vector<double> out(static_cast<size_t>(N));
    check(tmg_alpha_star_f64(h_, N, b, lambda, in.data(), out.data()));
    return out;
  }
  std::vector<double> beta_star_f64(std::int64_t N, std::int32_t b, std::int64_t lambda,
                                    const std::vector<double>& in) {
    need(in, N, "beta_star_f64");
    std::vector<double> out(static_cast<size_t>(N));
    check(tmg_beta_star_f64(h_, N, b, lambda, in.data(), out.data()));
    return out;
  }
  std::vector<double> gamma_dagger_f64(std::int64_t N, std::int32_t b, std::int64_t lambda,
                                       const std::vector<double>& in, double* aux) {
    need(in, N + 1, "gamma_dagger_f64");
    std::vector<double> out(static_cast<size_t>(N));
    check(tmg_gamma_dagger_f64(h_, N, b, lambda, in.data(), out.data(), aux));
    return out;
  }
  std::vector<double> delta_dagger_f64(std::int64_t N, std::int32_t b, std::int64_t lambda,
                                       const std::vector<double>& in, double aux) {
    need(in, N, "delta_dagger_f64");
    std::vector<double> out(static_cast<size_t>(N + 1));
    check(tmg_delta_dagger_f64(h_, N, b, lambda, in.data(), aux, out.data()));
    return out;
  }

  // The machine-word splitters (products.hpp:77-79): N chunks of u, or the
  // N + 1 chunks of the top-aligned u 2^sigma, sigma = (N + 1) b - n.
  std::vector<std::int64_t> split_low_i64(const Limbs& u, const Params& p) {
    return split(tmg_split_low_i64, u, p, p.N);
  }
  std::vector<std::int64_t> split_high_i64(const Limbs& u, const Params& p) {
    return split(tmg_split_high_i64, u, p, p.N + 1);
  }

  // Device-pointer variant: enqueue `count` products on the context stream;
  // device-side errors surface at the next check().
  void product_device(const Params& p, const std::uint64_t* d_u, const std::uint64_t* d_v,
                      std::uint64_t* d_out, std::int64_t count = 1) {
    const tmg_params q = p.to_c();
    check(tmg_product_device(h_, &q, d_u, d_v, d_out, count));
  }
  Stats check_device() {
    Stats s{};
    truncmul_b200::check(tmg_check(h_, &s));
    return s;
  }

  const Stats& last_stats() const { return stats_; }

 private:
  using Fn = int (*)(tmg_context*, const tmg_params*, const std::uint64_t*, const std::uint64_t*,
                     std::uint64_t*, tmg_stats*);
  Limbs run(Fn fn, Mode mode, const Limbs& u, const Limbs& v, const Params& p) {
    const std::int64_t nl = (p.n + 63) / 64;
    if (static_cast<std::int64_t>(u.size()) != nl || static_cast<std::int64_t>(v.size()) != nl)
      throw InputOutOfRange("operands must hold ceil(n/64) limbs");
    Limbs out(static_cast<size_t>(output_limbs(mode, p.n)));
    const tmg_params q = p.to_c();
    check(fn(h_, &q, u.data(), v.data(), out.data(), &stats_));
    return out;
  }

  static void need(const std::vector<double>& v, std::int64_t count, const char* what) {
    if (count < 0 || static_cast<std::int64_t>(v.size()) != count)
      throw PlanMismatch(std::string(what) + ": wrong input length");
  }
  using SplitFn = int (*)(tmg_context*, const tmg_params*, const std::uint64_t*, std::int64_t*);
  std::vector<std::int64_t> split(SplitFn fn, const Limbs& u, const Params& p, std::int64_t count) {
    if (p.n >= 1 && static_cast<std::int64_t>(u.size()) != (p.n + 63) / 64)
      throw InputOutOfRange("operands must hold ceil(n/64) limbs");
    std::vector<std::int64_t> out(static_cast<size_t>(count > 0 ? count : 0));
    const tmg_params q = p.to_c();
    check(fn(h_, &q, u.data(), out.data()));
    return out;
  }

  tmg_context* h_ = nullptr;
  Stats stats_{};
};

// Free functions of products.hpp on a thread-local context on device 0.
inline Context& default_context() {
  thread_local Context ctx(0);
  return ctx;
}
inline Limbs full_product(const Limbs& u, const Limbs& v, const Params& p) {
  return default_context().full_product(u, v, p);
}
inline Limbs low_product(const Limbs& u, const Limbs& v, const Params& p) {
  return default_context().low_product(u, v, p);
}
inline Limbs high_product(const Limbs& u, const Limbs& v, const Params& p) {
  return default_context().high_product(u, v, p);
}

inline std::vector<double> cyclic_convolve_f64(const std::vector<double>& f,
                                               const std::vector<double>& g) {
  return default_context().cyclic_convolve_f64(f, g);
}
inline std::vector<std::int64_t> split_low_i64(const Limbs& u, const Params& p) {
  return default_context().split_low_i64(u, p);
}
inline std::vector<std::int64_t> split_high_i64(const Limbs& u, const Params& p) {
  return default_context().split_high_i64(u, p);
}
}  // namespace truncmul_b200
