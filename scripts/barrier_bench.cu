// Grid-barrier latency on the B200: a persistent kernel (one CTA per SM) doing
// only barriers, in the variants the block tridiagonal solve could use.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void arrive_fence(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) { __threadfence(); atomicAdd(bar, 1u); }
}
__device__ __forceinline__ void arrive_release(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}
__device__ __forceinline__ void wait_acq(unsigned* bar, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned v;
    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while (v < target);
  }
  __syncthreads();
}
__device__ __forceinline__ void wait_relaxed(unsigned* bar, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned v;
    do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while (v < target);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

template <int V>
__global__ void k_bar(unsigned* bar, int steps, double* sink) {
  unsigned phase = 0;
  double acc = 0;
  for (int i = 0; i < steps; ++i) {
    if (V == 0) { arrive_fence(bar); if (threadIdx.x == 0) { __threadfence(); } wait_acq(bar, ++phase * gridDim.x); }
    if (V == 1) { arrive_release(bar); wait_acq(bar, ++phase * gridDim.x); }
    if (V == 2) { arrive_release(bar); wait_relaxed(bar, ++phase * gridDim.x); }
    acc += phase;
  }
  if (acc < 0) *sink = acc;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned* bar;
  double* sink;
  cudaMalloc(&bar, 4);
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int steps = 2000;
  for (int threads : {128, 384}) for (int grid : {nsm, 90, 32}) {
    for (int v = 0; v < 3; ++v) {
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(bar, 0, 4);
        cudaEventRecord(a);
        if (v == 0) k_bar<0><<<grid, threads>>>(bar, steps, sink);
        if (v == 1) k_bar<1><<<grid, threads>>>(bar, steps, sink);
        if (v == 2) k_bar<2><<<grid, threads>>>(bar, steps, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("threads %d grid %d variant %d: %.3f us per barrier\n", threads, grid, v, best * 1e3 / steps);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
