// Stand-alone FP64 cyclic convolution (cyclic_convolve_f64,
// convolution.hpp:64-67, convolution.cpp:175-203): out = f (*) g of length n.
//
// Lengths above 4096 run the products' own transform passes (first column
// pass, row pass with the spectral product, inverse column pass; api.cu
// enqueue_fft_passes) on z_j = f_j + i g_j: k_conv_pack interleaves the two
// real sequences into the packed complex input those passes read (16 n bytes
// written, 16 n read).  A packed transform separates the two spectra by
// differences, so its error follows ||f||^2 + ||g||^2 and not ||f|| ||g||:
// k_conv_absmax finds max |f| and max |g| first, and the pack multiplies g by
// the power of two that brings them together (exact; the last pass's output
// scale takes it out again).  Shorter lengths, and lengths that are not a
// multiple of 4 up to 32768, are summed directly (k_conv_direct: one output
// per thread, n fused multiply-adds each, both operands through L1).
#include <algorithm>

#include "kernels.cuh"

namespace tmg {

namespace {

// mx[0] = max |f_j|, mx[1] = max |g_j| as bit patterns (non-negative doubles
// order like their bits; a NaN lands above every number).  mx zeroed before.
__global__ void __launch_bounds__(256)
k_conv_absmax(const double* __restrict__ f, const double* __restrict__ g, int64_t n,
              unsigned long long* __restrict__ mx) {
  unsigned long long mf = 0, mg = 0;
  auto see = [&](double2 a, double2 b) {
    mf = max(mf, (unsigned long long)__double_as_longlong(fmax(fabs(a.x), fabs(a.y))));
    mg = max(mg, (unsigned long long)__double_as_longlong(fmax(fabs(b.x), fabs(b.y))));
    // fmax drops a NaN next to a number: keep it visible
    if (a.x != a.x || a.y != a.y) mf = ~0ull;
    if (b.x != b.x || b.y != b.y) mg = ~0ull;
  };
  // pairs (16-byte loads), four per thread and trip in flight
  const int64_t np = n >> 1, stride = int64_t(gridDim.x) * 256;
  const double2* f2 = reinterpret_cast<const double2*>(f);
  const double2* g2 = reinterpret_cast<const double2*>(g);
  int64_t j = int64_t(blockIdx.x) * 256 + threadIdx.x;
  for (; j + 3 * stride < np; j += 4 * stride) {
    const double2 a0 = f2[j], a1 = f2[j + stride], a2 = f2[j + 2 * stride], a3 = f2[j + 3 * stride];
    const double2 b0 = g2[j], b1 = g2[j + stride], b2 = g2[j + 2 * stride], b3 = g2[j + 3 * stride];
    see(a0, b0);
    see(a1, b1);
    see(a2, b2);
    see(a3, b3);
  }
  for (; j < np; j += stride) see(f2[j], g2[j]);
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0)
    see(make_double2(f[n - 1], 0.0), make_double2(g[n - 1], 0.0));
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mf = max(mf, __shfl_xor_sync(0xffffffffu, mf, o));
    mg = max(mg, __shfl_xor_sync(0xffffffffu, mg, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (mf) atomicMax(mx, mf);
    if (mg) atomicMax(mx + 1, mg);
  }
}

__global__ void __launch_bounds__(256)
k_conv_pack(const double* __restrict__ f, const double* __restrict__ g, int64_t n, double gs,
            double2* __restrict__ z) {
  // two elements per thread: 16-byte loads of f and g, 32 bytes stored
  const int64_t j = 2 * (int64_t(blockIdx.x) * 256 + threadIdx.x);
  if (j + 1 < n) {
    const double2 a = *reinterpret_cast<const double2*>(f + j);
    const double2 b = *reinterpret_cast<const double2*>(g + j);
    z[j] = make_double2(a.x, b.x * gs);
    z[j + 1] = make_double2(a.y, b.y * gs);
  } else if (j < n) {
    z[j] = make_double2(f[j], g[j] * gs);
  }
}

__global__ void __launch_bounds__(256)
k_conv_direct(const double* __restrict__ f, const double* __restrict__ g, int n,
              double* __restrict__ out) {
  const int k = blockIdx.x * 256 + threadIdx.x;
  if (k >= n) return;
  // out_k = sum_j f_j g_{(k - j) mod n}: j = 0 .. k reads g downwards from k,
  // j = k + 1 .. n - 1 downwards from n - 1
  double acc = 0.0;
  for (int j = 0; j <= k; ++j) acc = fma(__ldg(f + j), __ldg(g + (k - j)), acc);
  for (int j = k + 1; j < n; ++j) acc = fma(__ldg(f + j), __ldg(g + (n + k - j)), acc);
  out[k] = acc;
}

}  // namespace

void launch_conv_absmax(const double* d_f, const double* d_g, int64_t n, uint64_t* d_mx,
                        int num_sms, cudaStream_t st) {
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, int64_t(num_sms) * 8);
  k_conv_absmax<<<dim3(unsigned(blocks)), dim3(256), 0, st>>>(
      d_f, d_g, n, reinterpret_cast<unsigned long long*>(d_mx));
}

void launch_conv_pack(const double* d_f, const double* d_g, int64_t n, double gscale,
                      double2* d_z, cudaStream_t st) {
  const int64_t blocks = ((n + 1) / 2 + 255) / 256;
  k_conv_pack<<<dim3(unsigned(blocks)), dim3(256), 0, st>>>(d_f, d_g, n, gscale, d_z);
}

void launch_conv_direct(const double* d_f, const double* d_g, int64_t n, double* d_out,
                        cudaStream_t st) {
  k_conv_direct<<<dim3(unsigned((n + 255) / 256)), dim3(256), 0, st>>>(d_f, d_g, int(n), d_out);
}

}  // namespace tmg
