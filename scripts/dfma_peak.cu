// FP64 FMA issue rate of the SM's vector pipe: independent DFMA chains per thread, all SMs.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/dfma_peak.cu -o scripts/dfma_peak
#include <cstdio>
#include <cuda_runtime.h>
template <int ILP>
__global__ void k(double* out, double a, double b, int iters) {
  double v[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) v[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) v[i] = fma(v[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ILP>
void run(int warps_per_sm) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, 8ull * sms * 2048);
  const int iters = 20000;
  const int threads = 32 * warps_per_sm;  // one CTA per SM
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<ILP><<<sms, threads>>>(out, 1.0000001, 1e-9, 100);
  cudaEventRecord(e0);
  k<ILP><<<sms, threads>>>(out, 1.0000001, 1e-9, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fmas = (double)sms * threads * ILP * iters;
  printf("ILP %2d warps/SM %2d: %.2f T DFMA/s (%.1f TFLOP/s), %.1f DFMA/clk/SM at 1.965 GHz\n", ILP, warps_per_sm,
         fmas / ms * 1e-9, 2 * fmas / ms * 1e-9, fmas / ms * 1e-6 / sms / 1.965e3);
  cudaFree(out);
}
int main() {
  run<8>(4); run<8>(8); run<8>(16); run<8>(32); run<16>(8); run<16>(16); run<4>(32); run<2>(32); run<1>(32); run<1>(4); 
  return 0;
}
