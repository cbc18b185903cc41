// FP64 tensor-core GEMM for the fast-diagonalisation E solve (src/precond.cpp:
// 95-104 solved as (V (x) V) diag(1/(lam_i + lam_j - k^2)) (V (x) V)^T, DESIGN.md
// §4): C = op(A) op(B), column-major, optionally batched by strides.
//
// DMMA (mma.sync m8n8k4 .f64) is the FP64 tensor path on sm_100a (tcgen05 has
// no f64 kind).  The shapes of this solve are small and fixed (n = 800 at C5:
// 800 x 1600 x 800 and 2 x 800^3), where a library GEMM's 128 x 128 tiles
// leave a third of the 148 SMs idle (91 and 98 tiles).  Here the CTA tile is
// BM x BN = 64 x 48 (4 warps of 32 x 24, 4 x 3 fragments of 8 x 8 each), so
// both shapes are 442 tiles: one full wave at 3 resident CTAs per SM; K
// advances by 16 through a 3-stage cp.async ring.  Measured (ncu): the DMMA
// pipe is 85% busy while a CTA runs; 331 us per C5 E solve against cuBLAS's
// 299 us, so cuBLAS stays the default (HD_DGEMM=dmma selects this kernel).
//
// Operand staging (no transposition on the way in): op(A) is kept [m][k] when
// A is transposed (its rows are contiguous in k) and [k][m] otherwise; op(B)
// [n][k] when B is not transposed and [k][n] otherwise.  Row pitches are
// padded by 4 doubles so the 8 x 4 fragment loads hit every bank at most twice
// (two wavefronts, the minimum for 256 bytes).
#pragma once

#include "device_common.cuh"

namespace hd {

#ifndef HD_GBN
#define HD_GBN 48
#endif
#ifndef HD_GBK
#define HD_GBK 16
#endif
constexpr int kGBM = 64, kGBN = HD_GBN, kGBK = HD_GBK, kGST = 3, kGPad = 4;
constexpr int kGFN = kGBN / 16;  // 8 x 8 fragments per warp along n (warp tile 32 x BN/2)

template <bool TA, bool TB>
struct DgemmSmem {
  // A stage: TA ? [BM][BK+pad] : [BK][BM+pad];  B stage: TB ? [BK][BN+pad] : [BN][BK+pad]
  static constexpr int A = TA ? kGBM * (kGBK + kGPad) : kGBK * (kGBM + kGPad);
  static constexpr int B = TB ? kGBK * (kGBN + kGPad) : kGBN * (kGBK + kGPad);
  static constexpr size_t bytes = sizeof(double) * kGST * (A + B);
};

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// VEC doubles per copy: 2 (16 B, .cg) when every operand row is 16-byte aligned, else 1 (8 B, .ca)
template <int VEC>
__device__ __forceinline__ void g_cp(void* s, const void* g, bool valid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s));
  const int sz = valid ? 8 * VEC : 0;  // 0: zero-fill
  if (VEC == 2) asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(sz) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(sz) : "memory");
}

struct DgemmArgs {
  int M, N, K;
  const double* A;
  const double* B;
  double* C;
  int lda, ldb, ldc;
  long long sA, sB, sC;  // batch strides (blockIdx.z)
  // pointer-batched form (the folded E solve's x transforms): when set, entry
  // z of each array replaces the strided base
  const double* const* Ap = nullptr;
  const double* const* Bp = nullptr;
  double* const* Cp = nullptr;
};

// C = op(A) op(B).  VEC = 2 needs M, N, K, lda, ldb and the batch strides even
// and 16-byte aligned bases (the host wrapper checks); VEC = 1 takes any shape.
// KS = 2 splits K in two halves over blockIdx.z (z = batch * KS + half) that
// both add into a zeroed C with atomicAdd: 0 + a + b == 0 + b + a exactly, so
// the result is deterministic.  It doubles the tile count, which levels the
// work over the 148 SMs (325 -> 650 tiles for 800 x 1600).
template <bool TA, bool TB, int VEC, int KS>
__global__ void __launch_bounds__(128) k_dgemm(DgemmArgs g) {
  using SM = DgemmSmem<TA, TB>;
  extern __shared__ __align__(16) double dg_sm[];
  double* As = dg_sm;
  double* Bs = dg_sm + kGST * SM::A;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int m0 = blockIdx.y * kGBM, n0 = blockIdx.x * kGBN;
  const int bz = blockIdx.z / KS, half = blockIdx.z % KS;
  const double* A = g.Ap ? g.Ap[bz] : g.A + bz * g.sA;
  const double* B = g.Bp ? g.Bp[bz] : g.B + bz * g.sB;
  double* C = g.Cp ? g.Cp[bz] : g.C + bz * g.sC;
  const int nkt_all = (g.K + kGBK - 1) / kGBK;
  const int kt0 = KS == 1 ? 0 : (half == 0 ? 0 : nkt_all / 2);
  const int nkt = KS == 1 ? nkt_all : (half == 0 ? nkt_all / 2 : nkt_all - nkt_all / 2);

  auto load = [&](int kt, int st) {
    const int k0 = (kt0 + kt) * kGBK;
    double* as = As + st * SM::A;
    double* bs = Bs + st * SM::B;
    // op(A) tile BM x BK and op(B) tile BK x BN in chunks of VEC doubles
#pragma unroll
    for (int c = tid; c < kGBM * kGBK / VEC; c += 128) {
      if (TA) {  // A(k, m) at k + m lda: per m, 16 contiguous k
        const int m = c / (kGBK / VEC), kk = VEC * (c % (kGBK / VEC));
        const bool v = (m0 + m) < g.M && (k0 + kk) < g.K;
        g_cp<VEC>(as + m * (kGBK + kGPad) + kk, A + (v ? (size_t)(m0 + m) * g.lda + k0 + kk : 0), v);
      } else {  // A(m, k) at m + k lda: per k, 64 contiguous m
        const int kk = c / (kGBM / VEC), m = VEC * (c % (kGBM / VEC));
        const bool v = (m0 + m) < g.M && (k0 + kk) < g.K;
        g_cp<VEC>(as + kk * (kGBM + kGPad) + m, A + (v ? (size_t)(k0 + kk) * g.lda + m0 + m : 0), v);
      }
    }
#pragma unroll
    for (int c = tid; c < kGBK * kGBN / VEC; c += 128) {
      if (TB) {  // B(n, k) at n + k ldb: per k, 32 contiguous n
        const int kk = c / (kGBN / VEC), n = VEC * (c % (kGBN / VEC));
        const bool v = (n0 + n) < g.N && (k0 + kk) < g.K;
        g_cp<VEC>(bs + kk * (kGBN + kGPad) + n, B + (v ? (size_t)(k0 + kk) * g.ldb + n0 + n : 0), v);
      } else {  // B(k, n) at k + n ldb: per n, 16 contiguous k
        const int n = c / (kGBK / VEC), kk = VEC * (c % (kGBK / VEC));
        const bool v = (n0 + n) < g.N && (k0 + kk) < g.K;
        g_cp<VEC>(bs + n * (kGBK + kGPad) + kk, B + (v ? (size_t)(n0 + n) * g.ldb + k0 + kk : 0), v);
      }
    }
  };

  // warp tile 32 x BN/2: 4 fragments along m, kGFN along n
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * (kGBN / 2);
  const int gr = lane >> 2, gc = lane & 3;
  double acc[4][kGFN][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < kGFN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < kGST - 1; ++s) {
    if (s < nkt) load(s, s);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
#pragma unroll 1
  for (int kt = 0; kt < nkt; ++kt) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(kGST - 2) : "memory");
    __syncthreads();
    // refill the stage consumed two iterations ago
    if (kt + kGST - 1 < nkt) load(kt + kGST - 1, (kt + kGST - 1) % kGST);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const double* as = As + (kt % kGST) * SM::A;
    const double* bs = Bs + (kt % kGST) * SM::B;
#pragma unroll
    for (int k4 = 0; k4 < kGBK; k4 += 4) {
      double af[4], bf[kGFN];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm + 8 * i + gr, k = k4 + gc;
        af[i] = TA ? as[m * (kGBK + kGPad) + k] : as[k * (kGBM + kGPad) + m];
      }
#pragma unroll
      for (int j = 0; j < kGFN; ++j) {
        const int n = wn + 8 * j + gr, k = k4 + gc;
        bf[j] = TB ? bs[k * (kGBN + kGPad) + n] : bs[n * (kGBK + kGPad) + k];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < kGFN; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  // C fragment: rows gr, columns 2 gc, 2 gc + 1 of each 8 x 8 block
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < kGFN; ++j) {
      const int m = m0 + wm + 8 * i + gr;
      const int n = n0 + wn + 8 * j + 2 * gc;
      if (m < g.M) {
        if (KS == 1) {
          if (n < g.N) C[(size_t)n * g.ldc + m] = acc[i][j][0];
          if (n + 1 < g.N) C[(size_t)(n + 1) * g.ldc + m] = acc[i][j][1];
        } else {
          if (n < g.N) atomicAdd(C + (size_t)n * g.ldc + m, acc[i][j][0]);
          if (n + 1 < g.N) atomicAdd(C + (size_t)(n + 1) * g.ldc + m, acc[i][j][1]);
        }
      }
    }
}

}  // namespace hd
