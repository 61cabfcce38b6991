// Schoolbook product for operands below the pipeline cutoff (the reference's
// ORACLE_FALLBACK mode, products.hpp:14-15 and truncmul_cli.cpp:115-131).
#include "kernels.cuh"

namespace tmg {

__global__ void k_basecase(BaseArgs a) {
  // column sums as 192-bit accumulators, then one sequential carry pass
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(smem_raw);
  const int64_t nl = a.nlimbs;
  const int64_t nc = 2 * nl;
  for (int64_t k = threadIdx.x; k < nc; k += blockDim.x) {
    unsigned long long lo = 0, mid = 0, hi = 0;
    int64_t i0 = k - (nl - 1);
    if (i0 < 0) i0 = 0;
    for (int64_t i = i0; i <= k && i < nl; ++i) {
      unsigned long long x = a.u[i], y = a.v[k - i];
      unsigned long long pl = x * y, ph = __umul64hi(x, y);
      unsigned long long t = lo + pl;
      unsigned long long c1 = t < lo;
      lo = t;
      t = mid + ph;
      unsigned long long c2 = t < mid;
      mid = t + c1;
      c2 += (mid < t);
      hi += c2;
    }
    acc[3 * k] = lo;
    acc[3 * k + 1] = mid;
    acc[3 * k + 2] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long c0 = 0, c1 = 0;  // running carry (128-bit)
    for (int64_t k = 0; k < nc; ++k) {
      unsigned long long lo = acc[3 * k], mid = acc[3 * k + 1], hi = acc[3 * k + 2];
      unsigned long long t = lo + c0;
      unsigned long long cy = t < lo;
      a.prod[k] = t;
      // new carry = mid + hi*2^64 + c1*2^64 + cy
      unsigned long long n0 = mid + c1;
      unsigned long long k1 = n0 < mid;
      unsigned long long n0b = n0 + cy;
      k1 += n0b < n0;
      c0 = n0b;
      c1 = hi + k1;
    }
  }
}

}  // namespace tmg
