// Exact solve of a 2D level operator that is not a Kronecker sum as a block
// tridiagonal system, standing in for the reference's Eigen::SparseLU: the
// deflation matrix E = Z^T A Z of the wedge and layered fields (real;
// src/precond.cpp:95-99, 103) and the whole shifted operator of C_ex on those
// fields (complex; src/precond.cpp:204-211).
//
// Ordering the unknowns lexicographically (x fastest) and grouping q = b grid
// rows (b = the stencil's half-width in y) into one "super-row" of m = q*n
// unknowns makes E block tridiagonal with nb = ceil(n/q) diagonal blocks D_i
// and couplings B_i = E[i, i+1], C_i = E[i, i-1].  Block LU at setup (cuBLAS /
// cuSOLVER, partial pivoting inside each diagonal block):
//
//   S_0 = D_0,  S_i = D_i - G_i B_{i-1},  G_i = C_i S_{i-1}^-1,  H_i = S_i^-1 B_i,
//
// and per solve (real operator: the re and im planes are two real right-hand
// sides; complex operator: one complex right-hand side, planar):
//
//   y_i = r_i - G_i y_{i-1}          (nb sequential steps)
//   w_i = S_i^-1 y_i                 (all blocks in parallel)
//   x_i = w_i - H_i x_{i+1}          (nb sequential steps).
//
// k_btri_solve runs this in one persistent kernel (one CTA per SM, a grid
// barrier between dependent steps; w_{i-1} is formed alongside y_i).  A
// barrier-free variant that ordered the steps by dataflow on self-validating
// vector slots (sentinel-filled buffers polled by the consumers) was correct
// but 2x slower: 720 warps polling L2 starve the producers' stores.  Each
// warp owns matrix rows; the matrices are stored row-major (a warp streams one
// contiguous row).  Padding rows (n not a multiple of q) carry an identity
// diagonal and a zero right-hand side.
#pragma once

#include "layered.cuh"

namespace hd {

// scalar helpers over double (real operator) and double2 (complex operator)
__device__ __forceinline__ double bt_zero(double) { return 0.0; }
__device__ __forceinline__ double2 bt_zero(double2) { return cmk(0.0, 0.0); }
__device__ __forceinline__ void bt_set(double& d, double2 v) { d = v.x; }
__device__ __forceinline__ void bt_set(double2& d, double2 v) { d = v; }
__device__ __forceinline__ double bt_one(double) { return 1.0; }
__device__ __forceinline__ double2 bt_one(double2) { return cmk(1.0, 0.0); }
// acc (re, im) += a * (vr + i vi)
__device__ __forceinline__ void bt_fma(double a, double vr, double vi, double& sr, double& si) {
  sr = fma(a, vr, sr);
  si = fma(a, vi, si);
}
__device__ __forceinline__ void bt_fma(double2 a, double vr, double vi, double& sr, double& si) {
  sr = fma(a.x, vr, fma(-a.y, vi, sr));
  si = fma(a.x, vi, fma(a.y, vr, si));
}

// warps per CTA by the registers a row needs per lane (doubles per lane)
__host__ __device__ constexpr int btri_threads(int regs) { return regs <= 16 ? 512 : (regs <= 32 ? 384 : 256); }

struct BtriArgs {
  int n, q, m, nb;     // grid side, rows per block, block size m = q*n, blocks
  size_t NN;           // n^2 (unknowns); padded length nb*m
  const void* GT;      // nb blocks, row-major: G_i (block 0 unused)      [double or double2]
  const void* SinvT;   // nb blocks, row-major: S_i^-1
  const void* HT;      // nb blocks, row-major: H_i (block nb-1 unused)
  double* y;           // 2 planes x nb*m
  double* w;           // 2 planes x nb*m
  double* x;           // 2 planes x nb*m
  double* io;          // in/out planar (re plane NN, im plane NN)
  unsigned* bar;       // grid barrier counter, zeroed before the launch
};

// Column-major m x m blocks D_i, B_i (= E[i, i+1]), C_i (= E[i, i-1]) of the
// level operator (T = double: its real part; the coefficients must be real).
template <class T>
__global__ void k_btri_blocks(GenLevel L, int q, int m, int nb, T* __restrict__ D, T* __restrict__ Bu,
                              T* __restrict__ Cl) {
  const int n = L.n;
  const size_t mm = (size_t)m * m, tot = (size_t)nb * mm;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / mm);
    const size_t rem = e % mm;
    const int a = (int)(rem % m), c = (int)(rem / m);  // column-major (row a, column c)
    const int iy = i * q + a / n, ix = a % n;
    T d = bt_zero(T()), bu = bt_zero(T()), cl = bt_zero(T());
    if (iy < n) {
      // diagonal block: column c is unknown (i*q + c/n, c%n)
      const int jy = i * q + c / n, jx = c % n;
      const int dy = jy - iy, dx = jx - ix;
      if (jy < n && dy >= -L.b && dy <= L.b && dx >= -L.b && dx <= L.b) bt_set(d, gen_entry(L, iy, ix, dy, dx));
      const int jyu = (i + 1) * q + c / n, dyu = jyu - iy;
      if (jyu < n && dyu <= L.b && dx >= -L.b && dx <= L.b) bt_set(bu, gen_entry(L, iy, ix, dyu, dx));
      const int jyl = (i - 1) * q + c / n, dyl = jyl - iy;
      if (i > 0 && dyl >= -L.b && dx >= -L.b && dx <= L.b) bt_set(cl, gen_entry(L, iy, ix, dyl, dx));
    } else if (a == c) {
      d = bt_one(T());  // padding unknown
    }
    D[e] = d;
    Bu[e] = bu;
    Cl[e] = cl;
  }
}

// One matrix row (m entries, lane-strided into KR registers).
template <class T, int KR>
__device__ __forceinline__ void btri_row_load(const T* __restrict__ row, int m, T (&r)[KR]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int c = lane + 32 * k;
    r[k] = c < m ? __ldcs(row + c) : bt_zero(T());
  }
}

__device__ __forceinline__ void btri_arrive(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
  }
}

__device__ __forceinline__ void btri_wait(unsigned* bar, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar));
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

// The step's input vector (planar: re plane at v, im plane at v + plane),
// written by other CTAs before the last barrier, staged once per CTA into
// shared memory (vs: m re values, then m im values).
__device__ __forceinline__ void btri_stage(const double* v, size_t plane, int m, double* vs) {
  for (int c = threadIdx.x; c < m; c += blockDim.x) {
    vs[c] = __ldcg(v + c);
    vs[m + c] = __ldcg(v + plane + c);
  }
  __syncthreads();
}

// Row dot with the staged vector.
template <class T, int KR>
__device__ __forceinline__ double2 btri_row_dot(const T (&r)[KR], const double* vs, int m) {
  const int lane = threadIdx.x & 31;
  double sr0 = 0.0, si0 = 0.0, sr1 = 0.0, si1 = 0.0;
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int c = lane + 32 * k;
    if (c < m) {
      const double vr = vs[c], vi = vs[m + c];
      if (k & 1) bt_fma(r[k], vr, vi, sr1, si1);
      else bt_fma(r[k], vr, vi, sr0, si0);
    }
  }
  double sr = sr0 + sr1, si = si0 + si1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, o);
    si += __shfl_xor_sync(0xffffffffu, si, o);
  }
  return cmk(sr, si);
}

// Persistent solve.  Sequential steps, one grid barrier each (2 nb in total):
//   F_i (i = 0..nb-1):  y_i = r_i - G_i y_{i-1}  and  w_{i-1} = S_{i-1}^-1 y_{i-1}
//                       (2m independent row tasks: both need only y_{i-1})
//   B_{nb-1}:           x_{nb-1} = S_{nb-1}^-1 y_{nb-1}
//   B_i (i = nb-2..0):  x_i = w_i - H_i x_{i+1}
// A warp's first task of the next step has a fixed matrix row, which it loads
// into registers between arriving at and waiting on the barrier, so the HBM
// fetch of the step matrices overlaps the barrier (as do its right-hand-side
// reads); further tasks (2m > warps) load after the wait.
template <class T, int KR>
__global__ void __launch_bounds__(btri_threads(KR * (int)(sizeof(T) / 8)), 1) k_btri_solve(BtriArgs a) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int gw = blockIdx.x * wpb + (threadIdx.x >> 5);
  const int W = gridDim.x * wpb;
  const int m = a.m, nb = a.nb;
  const size_t mm = (size_t)m * m, P = (size_t)nb * m;
  const unsigned G = gridDim.x;
  const T* GT = static_cast<const T*>(a.GT);
  const T* SinvT = static_cast<const T*>(a.SinvT);
  const T* HT = static_cast<const T*>(a.HT);
  unsigned phase = 0;
  T r[KR];
  extern __shared__ double vs[];  // 2m: the staged step vector
  auto frow = [&](int i, int t) -> const T* {
    return t < m ? GT + i * mm + (size_t)t * m : SinvT + (i - 1) * mm + (size_t)(t - m) * m;
  };
  // ---- forward ----
  for (int i = 0; i < nb; ++i) {
    const int ntask = i > 0 ? 2 * m : m;
    if (i > 0 && blockIdx.x * wpb < ntask) btri_stage(a.y + (size_t)(i - 1) * m, P, m, vs);
    for (int t = gw; t < ntask; t += W) {
      const bool yrow = t < m;
      const int row = yrow ? t : t - m;
      const size_t gi = (size_t)i * m + row;
      double rr = 0.0, ri = 0.0;
      if (yrow && lane == 0 && gi < a.NN) {
        rr = a.io[gi];
        ri = a.io[a.NN + gi];
      }
      double2 acc = cmk(0.0, 0.0);
      if (i > 0) {
        if (t != gw) btri_row_load<T, KR>(frow(i, t), m, r);
        acc = btri_row_dot<T, KR>(r, vs, m);
      }
      if (lane == 0) {
        double* dst = yrow ? a.y + gi : a.w + gi - m;
        dst[0] = yrow ? rr - acc.x : acc.x;
        dst[P] = yrow ? ri - acc.y : acc.y;
      }
    }
    btri_arrive(a.bar);
    if (i + 1 < nb) {
      if (gw < 2 * m) btri_row_load<T, KR>(frow(i + 1, gw), m, r);
    } else if (gw < m) {
      btri_row_load<T, KR>(SinvT + (nb - 1) * mm + (size_t)gw * m, m, r);
    }
    btri_wait(a.bar, ++phase * G);
  }
  // ---- backward (x in its own buffer) ----
  for (int i = nb - 1; i >= 0; --i) {
    if (blockIdx.x * wpb < m) btri_stage(i == nb - 1 ? a.y + (size_t)i * m : a.x + (size_t)(i + 1) * m, P, m, vs);
    for (int row = gw; row < m; row += W) {
      const size_t gi = (size_t)i * m + row;
      double xr, xi;
      if (i == nb - 1) {
        if (row != gw) btri_row_load<T, KR>(SinvT + i * mm + (size_t)row * m, m, r);
        const double2 acc = btri_row_dot<T, KR>(r, vs, m);
        xr = acc.x;
        xi = acc.y;
      } else {
        const double wr = lane == 0 ? __ldcg(a.w + gi) : 0.0, wi = lane == 0 ? __ldcg(a.w + P + gi) : 0.0;
        if (row != gw) btri_row_load<T, KR>(HT + i * mm + (size_t)row * m, m, r);
        const double2 acc = btri_row_dot<T, KR>(r, vs, m);
        xr = wr - acc.x;
        xi = wi - acc.y;
      }
      if (lane == 0) {
        a.x[gi] = xr;
        a.x[P + gi] = xi;
        if (gi < a.NN) {
          a.io[gi] = xr;
          a.io[a.NN + gi] = xi;
        }
      }
    }
    if (i > 0) {
      btri_arrive(a.bar);
      if (gw < m) btri_row_load<T, KR>(HT + (i - 1) * mm + (size_t)gw * m, m, r);
      btri_wait(a.bar, ++phase * G);
    }
  }
}

}  // namespace hd
