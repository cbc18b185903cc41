// Stand-alone A/B of the fine-level stencil: k_stencil2d (cp.async ring, one
// column per lane) against k_stencil2d_tma (tensor-copy boxes, two columns per
// lane) -- bitwise comparison of every mode and per-launch CUDA-event times
// with the L2 flushed between launches.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -I paper_2010_10232_b200/csrc scripts/stencil_tma_bench.cu -o /tmp/stencil_tma_bench
//   /tmp/stencil_tma_bench [n=1601] [reps=20]
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "stencil.cuh"
#include "stencil_tma.cuh"

using namespace hd;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
  if (!f || q != cudaDriverEntryPointSuccess) {
    std::fprintf(stderr, "cuTensorMapEncodeTiled unavailable\n");
    std::exit(1);
  }
  return reinterpret_cast<EncodeFn>(f);
}

// 3D map over doubles: (2n, n rows, nvec), box (2 cols, rows, 1)
static CUtensorMap make_map(const double2* base, int n, int nvec, int box_cols, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)2 * n, (cuuint64_t)n, (cuuint64_t)nvec};
  cuuint64_t strides[2] = {(cuuint64_t)16 * n, (cuuint64_t)16 * n * n};
  cuuint32_t box[3] = {(cuuint32_t)2 * box_cols, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    std::fprintf(stderr, "cuTensorMapEncodeTiled failed: %d\n", (int)r);
    std::exit(1);
  }
  return m;
}

static int pick_rows_old(int n, int rows, int slots, int B) {
  const int colblocks = (n + kSW * kSWarps - 1) / (kSW * kSWarps);
  static const int cand[] = {8, 12, 16, 20, 24, 28, 32, 40, 48, 56, 64, 80, 96, 112, 128};
  int best = 32;
  double best_score = -1.0;
  for (int ry : cand) {
    const long tiles = (long)colblocks * ((rows + ry - 1) / ry);
    const long waves = (tiles + slots - 1) / slots;
    const double util = (double)tiles / ((double)waves * slots);
    const double score = util * ry / (ry + 2.0 * B);
    if (score > best_score + 1e-9) best_score = score, best = ry;
  }
  return best;
}

// strip height of the tensor-copy kernel: whole waves of resident warps, discounted by the halo rows
static int pick_rows_tma(int n, int warp_slots, int B, int* strips_x, int* ntasks) {
  const int sx = (n + kTW - 1) / kTW;
  int best = 32;
  double best_score = -1.0;
  for (int ry = 8; ry <= 256; ++ry) {
    const long tasks = (long)sx * ((n + ry - 1) / ry);
    const long waves = (tasks + warp_slots - 1) / warp_slots;
    const double util = (double)tasks / ((double)waves * warp_slots);
    const double score = util * ry / (ry + 2.0 * B);
    if (score > best_score + 1e-9) best_score = score, best = ry;
  }
  *strips_x = sx;
  *ntasks = sx * ((n + best - 1) / best);
  return best;
}

template <int B, int MODE>
static void run_mode(int n, int reps, const char* name) {
  constexpr int NB = 2 * B + 1;
  const size_t N = (size_t)n * n;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<double> hS((size_t)n * NB), hM((size_t)n * NB);
  srand(7);
  auto rnd = [] { return 2.0 * rand() / RAND_MAX - 1.0; };
  for (auto& v : hS) v = rnd();
  for (auto& v : hM) v = rnd() + 3.0;
  const int nvec = 3, jv = 2;
  std::vector<double2> hx(N * nvec), hb(N);
  for (auto& v : hx) v = make_double2(rnd(), rnd());
  for (auto& v : hb) v = make_double2(rnd(), rnd());
  double *dS, *dM;
  double2 *dx, *db, *o1, *o2, *p1, *p2, *part, *ct;
  unsigned* cnt;
  double* dst;
  int* didx;
  CK(cudaMalloc(&dS, hS.size() * 8));
  CK(cudaMalloc(&dM, hM.size() * 8));
  CK(cudaMalloc(&dx, N * nvec * 16));
  CK(cudaMalloc(&db, N * 16));
  CK(cudaMalloc(&o1, N * 16));
  CK(cudaMalloc(&o2, N * 16));
  CK(cudaMalloc(&p1, N * 16));
  CK(cudaMalloc(&p2, N * 16));
  CK(cudaMalloc(&part, 65536 * 16));
  CK(cudaMalloc(&cnt, 4));
  CK(cudaMalloc(&dst, 16));
  CK(cudaMalloc(&didx, 4));
  CK(cudaMemset(cnt, 0, 4));
  CK(cudaMemcpy(dS, hS.data(), hS.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dM, hM.data(), hM.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dx, hx.data(), N * nvec * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, hb.data(), N * 16, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(didx, &jv, 4, cudaMemcpyHostToDevice));
  const int ct_rows = n + 2 * B + kTSR;
  CK(cudaMalloc(&ct, (size_t)ct_rows * (NB + 1) * 16));
  LevelDev L{dS, dM, n, B, make_double2(0.7, -0.3), make_double2(0, 0), nullptr};
  k_build_ct<<<64, 256>>>(L, ct, ct_rows);
  CK(cudaGetLastError());
  void* flush;
  CK(cudaMalloc(&flush, 256u << 20));
  const double omega = 2.0 / 3.0;
  const double2 c2 = make_double2(0.7, 0.35);
  RedOut red{part, cnt, dst, 2.0, 0};
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));

  // --- old kernel
  const size_t sm_old_max = stencil_smem<B, MODE>(kSRowsMax);
  CK(cudaFuncSetAttribute(k_stencil2d<B, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_old_max));
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_stencil2d<B, MODE>, kSW * kSWarps, sm_old_max));
  const int ry = pick_rows_old(n, n, per * sms, B);
  dim3 g_old((n + kSW * kSWarps - 1) / (kSW * kSWarps), (n + ry - 1) / ry);
  std::vector<float> t_old, t_new;
  double r_old = 0, r_new = 0;
  for (int r = 0; r < reps; ++r) {
    CK(cudaMemsetAsync(flush, r, 256u << 20));
    CK(cudaEventRecord(e0));
    k_stencil2d<B, MODE><<<g_old, kSW * kSWarps, stencil_smem<B, MODE>(ry)>>>(L, dx, db, o1, omega, ry, red, didx, N, 0, n,
                                                                             o2, c2);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    t_old.push_back(ms * 1e3f);
  }
  CK(cudaMemcpy(&r_old, dst, 8, cudaMemcpyDeviceToHost));

  // --- tensor-copy kernel
  using Lay = TmaLayout<B, MODE>;
  auto kern = k_stencil2d_tma<B, MODE>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lay::total));
  int per2 = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, kern, 32 * kTWarps, Lay::total));
  int strips_x = 0, ntasks = 0;
  const int ry2 = pick_rows_tma(n, per2 * kTWarps * sms, B, &strips_x, &ntasks);
  const CUtensorMap tmx = make_map(dx, n, nvec, tma_xc<B>(), kTSR);
  const CUtensorMap tmb = make_map(db, n, 1, kTBC, kTSR);
  const int grid2 = (ntasks + kTWarps - 1) / kTWarps;
  for (int r = 0; r < reps; ++r) {
    CK(cudaMemsetAsync(flush, r, 256u << 20));
    CK(cudaEventRecord(e0));
    kern<<<grid2, 32 * kTWarps, Lay::total>>>(tmx, tmb, L, ct, p1, omega, ry2, strips_x, ntasks, red,
                                                                 didx, p2, c2);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    t_new.push_back(ms * 1e3f);
  }
  CK(cudaMemcpy(&r_new, dst, 8, cudaMemcpyDeviceToHost));

  // --- compare
  size_t bad = 0, bad2 = 0;
  if (MODE != OP_RESNORM) {
    std::vector<double2> a(N), b(N);
    CK(cudaMemcpy(a.data(), o1, N * 16, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), p1, N * 16, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < N; ++i) bad += std::memcmp(&a[i], &b[i], 16) != 0;
    if (MODE == OP_APPLYJ0) {
      CK(cudaMemcpy(a.data(), o2, N * 16, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(b.data(), p2, N * 16, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < N; ++i) bad2 += std::memcmp(&a[i], &b[i], 16) != 0;
    }
  }
  std::sort(t_old.begin(), t_old.end());
  std::sort(t_new.begin(), t_new.end());
  const double P = 16.0 * N;
  const double bytes = (MODE == OP_APPLY || MODE == OP_RESNORM) ? 2 * P : 3 * P;
  std::printf("%-8s n=%d B=%d | old: ry=%d grid=%dx%d per=%d  med %.1f us (%.0f GB/s) | tma: ry=%d tasks=%d per=%d smem=%zu  "
              "med %.1f us min %.1f (%.0f GB/s) | mismatches %zu %zu | resnorm %.17g %.17g\n",
              name, n, B, ry, g_old.x, g_old.y, per, t_old[reps / 2], bytes / t_old[reps / 2] * 1e-3, ry2, ntasks, per2,
              (size_t)Lay::total, t_new[reps / 2], t_new[0], bytes / t_new[reps / 2] * 1e-3, bad, bad2, r_old, r_new);
  cudaFree(dS); cudaFree(dM); cudaFree(dx); cudaFree(db); cudaFree(o1); cudaFree(o2); cudaFree(p1); cudaFree(p2);
  cudaFree(part); cudaFree(cnt); cudaFree(dst); cudaFree(didx); cudaFree(ct); cudaFree(flush);
}

template <int B>
static void run_all(int n, int reps) {
  run_mode<B, OP_APPLY>(n, reps, "APPLY");
  run_mode<B, OP_APPLYJ0>(n, reps, "APPLYJ0");
  run_mode<B, OP_RESID>(n, reps, "RESID");
  run_mode<B, OP_JACOBI>(n, reps, "JACOBI");
  run_mode<B, OP_RESNORM>(n, reps, "RESNORM");
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 1601;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 20;
  const int B = argc > 3 ? std::atoi(argv[3]) : 3;
  if (B == 3) run_all<3>(n, reps);
  else if (B == 2) run_all<2>(n, reps);
  else if (B == 1) run_all<1>(n, reps);
  else run_all<4>(n, reps);
  return 0;
}
