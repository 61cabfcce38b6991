// Shared device-side definitions for the truncated-product pipeline.
//
// Domain vocabulary follows the reference (arxiv 1703.00640 artifact,
// /root/reference/proj/core): limbs are little-endian uint64 words of an
// operand, chunks are the b-bit pieces the operand is split into
// (split.cpp:66-102), coefficients are the rounded convolution outputs that
// recombination sums at bit offsets i*b (products_f64.cpp:29-102).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tmg {

// ---------------------------------------------------------------------------
// Status word written by the kernels and read by the host after a product.
// The flag bits map onto the reference's exception types (errors.hpp):
//   kFlagTripwire / kFlagOverflow -> ConvolutionPrecisionFailure
//       ("rounding tripwire: residual above a quarter" /
//        "coefficient overflowed the exact-integer range",
//        products_f64.cpp:16-27)
//   kFlagLowNotDivisible -> ConvolutionPrecisionFailure
//       ("low product recombination is not divisible by the chunk base",
//        products_f64.cpp:137-140)
//   kFlagHighRange -> ConvolutionPrecisionFailure
//       ("high product left its admissible range", products_f64.cpp:167-169)
//   kFlagNegative -> ConvolutionPrecisionFailure
//       ("full product recombined negative", products_f64.cpp:117-119)
//   kFlagInputRange -> InputOutOfRange ("split: operand outside [0, 2^n)",
//       split.cpp:13-20)
enum : uint32_t {
  kFlagTripwire = 1u << 0,
  kFlagOverflow = 1u << 1,
  kFlagLowNotDivisible = 1u << 2,
  kFlagHighRange = 1u << 3,
  kFlagNegative = 1u << 4,
  kFlagInputRange = 1u << 5,
  kFlagCarryRange = 1u << 6,   // internal: a limb carry left {-1,0,1}
  kFlagFullOverflow = 1u << 7, // full product had bits above 2n
};

struct DevStatus {
  unsigned long long max_err_bits;  // max |x - round(x)| as double bits
  unsigned long long max_abs_bits;  // max |x| as double bits
  unsigned int flags;
  unsigned int high_topbit;  // high product: bit n of w was set
  unsigned int high_lownz;   // high product: some bit below n was set
  unsigned int high_sticky;  // high product: t has a set bit below s-1
};

// ---------------------------------------------------------------------------
// Programmatic dependent launch (sm_90+).  Kernels of a product are launched
// with the programmatic-serialization attribute (api.cu launch()): the next
// kernel may be scheduled once every CTA of the current one has executed
// pdl_trigger(), runs its prologue (constant tables, arguments), and
// pdl_wait() blocks until the predecessor grid has completed and its memory
// is visible.  Launched without the attribute both are no-ops.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Complex helpers (double2 as complex double).
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cconj(double2 a) {
  return make_double2(a.x, -a.y);
}
__device__ __forceinline__ double2 cscale(double2 a, double s) {
  return make_double2(a.x * s, a.y * s);
}

// ---------------------------------------------------------------------------
// Carry transfer functions.  A limb (or chunk) maps an incoming carry
// c in {-1, 0, +1} to an outgoing carry f(c) in {-1, 0, +1}; composing these
// maps is associative, which is what makes carry propagation a parallel
// prefix.  Encoding: one byte per input, holding f(c)+1, for c = -1, 0, +1
// in bytes 0, 1, 2 -- so that composition is one byte permute.
__host__ __device__ __forceinline__ uint32_t tf_const(int c) {
  return uint32_t(c + 1) * 0x010101u;
}
constexpr uint32_t kTfIdentity = 0x020100u;
// g o f: apply f first, then g.  Byte c of the result is byte f(c)+1 of g:
// PRMT with f's bytes as selector nibbles.
__device__ __forceinline__ uint32_t tf_compose(uint32_t f, uint32_t g) {
  const uint32_t sel = (f & 0xFu) | ((f >> 4) & 0xF0u) | ((f >> 8) & 0xF00u);
  return __byte_perm(g, 0u, sel) & 0xFFFFFFu;
}
__device__ __forceinline__ int tf_apply(uint32_t f, int c) {
  return int((f >> (8 * (c + 1))) & 0xFFu) - 1;
}

// Small fast divider for runtime-constant uint32 divisors (n < 2^31).
struct FastDiv {
  uint32_t d, m, s;
};
inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  uint32_t s = 0;
  while ((1ull << s) < d) ++s;
  f.s = s;
  // m = floor(2^32 * (2^s - d) / d) + 1
  f.m = uint32_t(((1ull << 32) * ((1ull << s) - d)) / d + 1);
  return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t x, const FastDiv& f) {
  if (f.s == 0) return x;  // d == 1
  uint32_t t = __umulhi(x, f.m);
  return (t + ((x - t) >> 1)) >> (f.s - 1);
}

// Bulk global -> shared copy completing on an mbarrier (cp.async.bulk; the
// sizes and addresses are multiples of 16 bytes).
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  const uint32_t a = uint32_t(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  const uint32_t a = uint32_t(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  const uint32_t d = uint32_t(__cvta_generic_to_shared(dst));
  const uint32_t b = uint32_t(__cvta_generic_to_shared(bar));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
// 16-byte asynchronous global -> shared copies (cp.async, no registers).
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  const uint32_t d = uint32_t(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = uint32_t(__cvta_generic_to_shared(bar));
  asm volatile(
      "{\n .reg .pred p;\n"
      "MBW%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MBW%=;\n}" ::"r"(a), "r"(phase) : "memory");
}

}  // namespace tmg
