// cuBLASLt algorithm sweep for the folded E-solve DGEMMs (n = 800, n2 = 400 at C5),
// all strided-batched over the two parities:
//   X: op(A) n2 x n2 (T for the forward transform, N for the inverse), B n2 x 2n
//   Y: A (4 n2) x n2, op(B) n2 x n2 (N forward, T inverse)
// Prints cublasDgemmStridedBatched and every heuristic cuBLASLt algorithm.
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a lt_fold.cu -lcublasLt -lcublas -o lt_fold
#include <cublasLt.h>
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                       \
  do {                                                              \
    auto e_ = (x);                                                  \
    if (e_ != 0) {                                                  \
      std::printf("%s failed (%d) at %d\n", #x, (int)e_, __LINE__); \
      std::exit(1);                                                 \
    }                                                               \
  } while (0)

struct Shape {
  const char* name;
  cublasOperation_t ta, tb;
  int m, n, k, lda, ldb, ldc;
  long long sa, sb, sc;
};

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 800, n2 = n / 2;
  const long long nn = (long long)n2 * n2, hc = (long long)n2 * 2 * n;
  const Shape shapes[] = {
      {"X fwd (T,N) n2 x 2n x n2", CUBLAS_OP_T, CUBLAS_OP_N, n2, 2 * n, n2, n2, n2, n2, nn, hc, hc},
      {"Y fwd (N,N) 4n2 x n2 x n2", CUBLAS_OP_N, CUBLAS_OP_N, 4 * n2, n2, n2, 4 * n2, n2, 4 * n2, 4 * nn, nn, 4 * nn},
      {"Y inv (N,T) 4n2 x n2 x n2", CUBLAS_OP_N, CUBLAS_OP_T, 4 * n2, n2, n2, 4 * n2, n2, 4 * n2, 4 * nn, nn, 4 * nn},
      {"X inv (N,N) n2 x 2n x n2", CUBLAS_OP_N, CUBLAS_OP_N, n2, 2 * n, n2, n2, n2, n2, nn, hc, hc},
  };
  double *A, *B, *C;
  const size_t big = (size_t)8 * nn + 16;
  CK(cudaMalloc(&A, sizeof(double) * big));
  CK(cudaMalloc(&B, sizeof(double) * big));
  CK(cudaMalloc(&C, sizeof(double) * big));
  CK(cudaMemset(A, 0, sizeof(double) * big));
  CK(cudaMemset(B, 0, sizeof(double) * big));
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
  for (const Shape& s : shapes) {
    const double flops = 2.0 * 2 * s.m * s.n * s.k;
    for (int w = 0; w < 3; ++w)
      cublasDgemmStridedBatched(h, s.ta, s.tb, s.m, s.n, s.k, &one, A, s.lda, s.sa, B, s.ldb, s.sb, &zero, C, s.ldc,
                                s.sc, 2);
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r)
      cublasDgemmStridedBatched(h, s.ta, s.tb, s.m, s.n, s.k, &one, A, s.lda, s.sa, B, s.ldb, s.sb, &zero, C, s.ldc,
                                s.sc, 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::printf("%s  cublasDgemmStridedBatched: %.2f us  %.1f TF/s\n", s.name, ms * 1e3 / 20,
                flops / (ms * 1e-3 / 20) / 1e12);
    cublasLtMatmulDesc_t op;
    CK(cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_64F, CUDA_R_64F));
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &s.ta, sizeof(s.ta)));
    CK(cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &s.tb, sizeof(s.tb)));
    cublasLtMatrixLayout_t la, lb, lc;
    const bool tA = s.ta == CUBLAS_OP_T, tB = s.tb == CUBLAS_OP_T;
    CK(cublasLtMatrixLayoutCreate(&la, CUDA_R_64F, tA ? s.k : s.m, tA ? s.m : s.k, s.lda));
    CK(cublasLtMatrixLayoutCreate(&lb, CUDA_R_64F, tB ? s.n : s.k, tB ? s.k : s.n, s.ldb));
    CK(cublasLtMatrixLayoutCreate(&lc, CUDA_R_64F, s.m, s.n, s.ldc));
    const int bc = 2;
    for (auto [l, st] : {std::pair{la, s.sa}, std::pair{lb, s.sb}, std::pair{lc, s.sc}}) {
      CK(cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_BATCH_COUNT, &bc, sizeof(bc)));
      CK(cublasLtMatrixLayoutSetAttribute(l, CUBLASLT_MATRIX_LAYOUT_STRIDED_BATCH_OFFSET, &st, sizeof(st)));
    }
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
      for (int r = 0; r < 20; ++r) cublasLtMatmul(lt, op, &one, A, la, B, lb, &zero, C, lc, C, lc, &res[i].algo, ws, wsz, 0);
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
