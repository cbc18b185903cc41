// cuBLASLt algorithm sweep for the E-solve DGEMM shapes (n = 800 at C5):
//   op(A) n x n, B n x 2n  (TN and NN),  C n x 2n.
// Prints the time of cublasDgemm and of every heuristic cuBLASLt algorithm.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a lt_tune.cu -lcublasLt -lcublas -o lt_tune
#include <cublasLt.h>
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                             \
  do {                                                                    \
    auto e_ = (x);                                                        \
    if (e_ != 0) {                                                        \
      std::printf("%s failed (%d) at %d\n", #x, (int)e_, __LINE__);       \
      std::exit(1);                                                       \
    }                                                                     \
  } while (0)

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 800;
  const int m = n, k = n, nn = 2 * n;
  double *A, *B, *C;
  CK(cudaMalloc(&A, sizeof(double) * m * k));
  CK(cudaMalloc(&B, sizeof(double) * k * nn));
  CK(cudaMalloc(&C, sizeof(double) * m * nn));
  CK(cudaMemset(A, 0, sizeof(double) * m * k));
  CK(cudaMemset(B, 0, sizeof(double) * k * nn));
  cublasHandle_t h;
  CK(cublasCreate(&h));
  cublasLtHandle_t lt;
  CK(cublasLtCreate(&lt));
  void* ws;
  const size_t wsz = 64u << 20;
  CK(cudaMalloc(&ws, wsz));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double one = 1.0, zero = 0.0;
  const double flops = 2.0 * m * nn * k;
  for (int ta = 0; ta < 2; ++ta) {
    const cublasOperation_t opA = ta ? CUBLAS_OP_T : CUBLAS_OP_N;
    // cublasDgemm reference
    for (int w = 0; w < 3; ++w) cublasDgemm(h, opA, CUBLAS_OP_N, m, nn, k, &one, A, n, B, k, &zero, C, m);
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) cublasDgemm(h, opA, CUBLAS_OP_N, m, nn, k, &one, A, n, B, k, &zero, C, m);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("op %s cublasDgemm: %.2f us  %.1f TF/s\n", ta ? "T" : "N", ms * 1e3 / 20, flops / (ms * 1e-3 / 20) / 1e12);
    cublasLtMatmulDesc_t op;
    CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_64F, CUDA_R_64F));
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &opA, sizeof(opA)));
    cublasLtMatrixLayout_t la, lb, lc;
    CK(cublasLtMatrixLayoutCreate(&la, CUDA_R_64F, ta ? k : m, ta ? m : k, n));
    CK(cublasLtMatrixLayoutCreate(&lb, CUDA_R_64F, k, nn, k));
    CK(cublasLtMatrixLayoutCreate(&lc, CUDA_R_64F, m, nn, m));
    cublasLtMatmulPreference_t pref;
    CK(cublasLtMatmulPreferenceCreate(&pref));
    CK(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof(wsz)));
    std::vector<cublasLtMatmulHeuristicResult_t> res(64);
    int got = 0;
    CK(cublasLtMatmulAlgoGetHeuristic(lt, op, la, lb, lc, lc, pref, 64, res.data(), &got));
    std::printf("  %d heuristic algorithms\n", got);
    for (int i = 0; i < got; ++i) {
      bool ok = true;
      for (int w = 0; w < 3 && ok; ++w)
        ok = cublasLtMatmul(lt, op, &one, A, la, B, lb, &zero, C, lc, C, lc, &res[i].algo, ws, wsz, 0) == 0;
      if (!ok) continue;
      cudaEventRecord(e0);
      for (int r = 0; r < 20; ++r)
        cublasLtMatmul(lt, op, &one, A, la, B, lb, &zero, C, lc, C, lc, &res[i].algo, ws, wsz, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      int tile = -1, stages = -1, splitk = -1;
      size_t sz;
      cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_TILE_ID, &tile, sizeof(tile), &sz);
      cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_STAGES_ID, &stages, sizeof(stages), &sz);
      cublasLtMatmulAlgoConfigGetAttribute(&res[i].algo, CUBLASLT_ALGO_CONFIG_SPLITK_NUM, &splitk, sizeof(splitk), &sz);
      std::printf("  algo %2d tile %3d stages %3d splitk %2d ws %8zu: %.2f us  %.1f TF/s\n", i, tile, stages, splitk,
                  res[i].workspaceSize, ms * 1e3 / 20, flops / (ms * 1e-3 / 20) / 1e12);
    }
  }
  return 0;
}
