// DFMA rate with three distinct 64-bit register operands per instruction (no operand reuse),
// as in the stencil's y pass, against the reuse-friendly form of dfma_peak.cu.
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP, int MODE>
__global__ void k(double* out, const double* in, int iters) {
  double v[ILP], a[ILP], b[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { v[i] = threadIdx.x + i; a[i] = in[i]; b[i] = in[ILP + i]; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      if (MODE == 0) v[i] = fma(a[i], b[i], v[i]);               // 3 distinct regs
      else if (MODE == 1) v[i] = fma(a[i], b[0], v[i]);          // one shared operand
      else if (MODE == 2) v[i] = fma(a[0], b[0], v[i]);          // two shared
      else v[i] = fma(a[i], b[(i + 1) % ILP], v[(i + 3) % ILP]); // shuffled, distinct
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ILP, int MODE>
void run(int warps_per_sm) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out, *in; cudaMalloc(&out, 8ull * sms * 2048); cudaMalloc(&in, 8 * 64);
  double h[64]; for (int i = 0; i < 64; ++i) h[i] = 1.0 + 1e-9 * i; cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  const int iters = 20000, threads = 32 * warps_per_sm;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<ILP, MODE><<<sms, threads>>>(out, in, 100);
  cudaEventRecord(e0);
  k<ILP, MODE><<<sms, threads>>>(out, in, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fmas = (double)sms * threads * ILP * iters;
  printf("mode %d ILP %2d warps/SM %2d: %.2f T DFMA/s, %.2f cycles per warp DFMA per SMSP\n", MODE, ILP, warps_per_sm,
         fmas / ms * 1e-9, 1.965e9 / (fmas / ms * 1e3 / 32 / (sms * 4)));
  cudaFree(out); cudaFree(in);
}
int main() {
  run<8, 0>(8); run<8, 1>(8); run<8, 2>(8); run<8, 3>(8);
  run<16, 0>(8); run<16, 1>(8); run<16, 3>(8); run<16, 0>(16); run<16, 3>(4);
  return 0;
}
