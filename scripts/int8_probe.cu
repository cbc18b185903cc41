// Probe: cuBLAS int8 (IMMA, int32 accumulate) vs FP64 DGEMM on the C5 E-solve
// shapes (M = 800, N = 1600, K = 800 * (d + 1)), for an Ozaki-style FP64 emulation.
#include <cstdio>
#include <cstdint>
#include <cublas_v2.h>
#include <cuda_runtime.h>

int main() {
  const int M = 800, N = 1600, K0 = 800;
  cublasHandle_t h;
  cublasCreate(&h);
  int8_t *A, *B;
  int32_t* C;
  double *dA, *dB, *dC;
  cudaMalloc(&A, (size_t)M * K0 * 8);
  cudaMalloc(&B, (size_t)K0 * 8 * N);
  cudaMalloc(&C, (size_t)M * N * 4);
  cudaMalloc(&dA, (size_t)M * K0 * 8);
  cudaMalloc(&dB, (size_t)K0 * N * 8);
  cudaMalloc(&dC, (size_t)M * N * 8);
  cudaMemset(A, 1, (size_t)M * K0 * 8);
  cudaMemset(B, 1, (size_t)K0 * 8 * N);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int32_t one = 1, zero = 0;
  for (int d = 0; d < 8; ++d) {
    const int K = K0 * (d + 1);
    float best = 1e9;
    cublasStatus_t st = CUBLAS_STATUS_SUCCESS;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      st = cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, M, N, K, &one, A, CUDA_R_8I, K, B, CUDA_R_8I, K, &zero, C,
                        CUDA_R_32I, M, CUBLAS_COMPUTE_32I, CUBLAS_GEMM_DEFAULT);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("int8 K=%5d: %8.2f us  %7.1f TOPS  status %d\n", K, best * 1e3, 2.0 * M * N * K / (best * 1e-3) / 1e12, st);
  }
  const double o = 1.0, z = 0.0;
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, M, N, K0, &o, dA, K0, dB, K0, &z, dC, M);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  printf("dgemm K=%d: %8.2f us  %7.2f TFLOPS\n", K0, best * 1e3, 2.0 * M * N * K0 / (best * 1e-3) / 1e12);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
