// The paper's ring-change maps as entry points of their own: alpha*, beta*
// (low product) and gamma-dagger, delta-dagger (high product) on FP64
// sequences -- maps_f64.hpp's alpha_star_f64, beta_star_f64,
// gamma_dagger_f64 and delta_dagger_f64 (maps_f64.cpp:245-384).
//
// One output per thread, through the same device helpers the products use
// (pipeline.cuh: premap, root_channel, postmap_low, high_psi, postmap_high),
// with the series coefficients computed on the fly from the row scales in
// MapConsts (the reference reads them from tables built by series.cpp; the
// two agree to the last few ulps of a coefficient).  The products fuse
// these maps into the first column pass and the carry; here they are plain
// elementwise kernels over lambda-wide windows of the input: 8 bytes read
// (through L1, lambda taps) and 8 written per point.
#include "kernels.cuh"
#include "pipeline.cuh"

namespace tmg {

namespace {

constexpr int kMapThreads = 256;

struct SeqSrc {
  const double* p;
  __device__ __forceinline__ double operator()(int64_t k) const { return __ldg(p + k); }
};

// alpha* (mode low) or gamma-dagger (mode high: in has N + 1 entries, the top
// one folded in; aux receives the root channel)
__global__ void __launch_bounds__(kMapThreads)
k_map_pre(const __grid_constant__ MapConsts mc, const double* __restrict__ in,
          double* __restrict__ out, double* __restrict__ aux) {
  const int64_t j = int64_t(blockIdx.x) * kMapThreads + threadIdx.x;
  const SeqSrc D{in};
  const double top = (mc.mode == kModeHigh) ? __ldg(in + mc.N) : 0.0;
  if (mc.mode == kModeHigh && j == 0) *aux = root_channel(mc, D, top);
  if (j < mc.N) out[j] = premap(mc, D, j, top);
}

// beta* (mode low: N outputs) or delta-dagger (mode high: N + 1 outputs)
__global__ void __launch_bounds__(kMapThreads)
k_map_post(const __grid_constant__ MapConsts mc, const double* __restrict__ in, double aux,
           double* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * kMapThreads + threadIdx.x;
  const SeqSrc W{in};
  if (mc.mode == kModeLow) {
    if (i < mc.N) out[i] = postmap_low(mc, W, i);
    return;
  }
  __shared__ double s_psi;
  if (threadIdx.x == 0) s_psi = high_psi(mc, W, aux);
  __syncthreads();
  if (i <= mc.N) out[i] = postmap_high(mc, W, i, s_psi);
}

}  // namespace

void launch_map_pre(const MapConsts& mc, const double* d_in, double* d_out, double* d_aux,
                    cudaStream_t st) {
  const int64_t blocks = (mc.N + kMapThreads - 1) / kMapThreads;
  k_map_pre<<<dim3(unsigned(blocks)), dim3(kMapThreads), 0, st>>>(mc, d_in, d_out, d_aux);
}

void launch_map_post(const MapConsts& mc, const double* d_in, double aux, double* d_out,
                     cudaStream_t st) {
  const int64_t outs = mc.N + (mc.mode == kModeHigh ? 1 : 0);
  const int64_t blocks = (outs + kMapThreads - 1) / kMapThreads;
  k_map_post<<<dim3(unsigned(blocks)), dim3(kMapThreads), 0, st>>>(mc, d_in, aux, d_out);
}

}  // namespace tmg
