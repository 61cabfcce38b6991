// FP64 issue-rate microbenchmark: DFMA / DADD / DMUL / mixed chains at ILP 8,
// one CTA per SM, 4..32 warps.  Prints thread-instructions per clock per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_rate fp64_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, long long* clk) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) a[i] = fma(a[i], b, c);
      if (OP == 1) a[i] = a[i] + c;
      if (OP == 2) a[i] = a[i] * b;
      if (OP == 3) { if (i & 1) a[i] = a[i] + c; else a[i] = fma(a[i], b, c); }
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
int main() {
  double* out; long long* clk;
  cudaMalloc(&out, 148 * 1024 * 8); cudaMalloc(&clk, 148 * 8);
  const int iters = 4096;
  const char* names[] = {"DFMA", "DADD", "DMUL", "DADD+DFMA"};
  for (int op = 0; op < 4; ++op)
    for (int warps : {4, 8, 16, 32}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (op == 0) k<0><<<148, warps * 32>>>(out, iters, clk);
        if (op == 1) k<1><<<148, warps * 32>>>(out, iters, clk);
        if (op == 2) k<2><<<148, warps * 32>>>(out, iters, clk);
        if (op == 3) k<3><<<148, warps * 32>>>(out, iters, clk);
      }
      cudaDeviceSynchronize();
      long long h[148]; cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
      printf("%s warps/SM %d: %.1f thread-instr/clk/SM\n", names[op], warps, double(iters) * 8 * warps * 32 / avg);
    }
  return 0;
}
