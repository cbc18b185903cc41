// Layered wave-number field (reference layered_medium_2d, src/problems.cpp:25-32,
// 68-74; K2 assembly src/assembly.cpp:234-246):
//
//   K2 = sum_{by,bx} (k m_{by,bx})^2  B_by (x) B_bx ,   B_b = mass on [b/4, (b+1)/4]
//
// Grouped by the y factor, every level operator of the hierarchy is a sum of
// G <= 6 Kronecker products with banded 1D factors,
//
//   L = My (x) Sx + Sy (x) Mx + sum_by gamma_by  B_by (x) W_by ,
//   W_by = sum_bx m_{by,bx}^2 B_bx ,  gamma = -k^2 (A) or -k^2 (1 - i beta2) (shifted),
//
// and Galerkin coarsening keeps that form factor by factor (z^T Y z, z^T X z).
// k_kron2d applies it sum-factorised from shared memory: a CTA stages a
// (16 + 2b) x (32 + 2b) input tile, forms the G x-products of every staged row,
// then combines them along y for its 16 x 32 outputs.  The exact solves of the
// layered hierarchy (deflation E, coarsest level) are dense inverses built by
// k_dense_kron + cuSOLVER getrf/getrs; they are not Kronecker sums, so the fast
// diagonalisation of the constant field does not apply.
//
// Wedge field (BASELINE config 4, non-separable K2): the level operator is the
// Kronecker-sum part My (x) Sx + Sy (x) My (G = 2 groups) plus a stored 2D stencil
//
//   L += kc * K_l ,  K_l = (z (x) z)^T K_{l-1} (z (x) z)   (Galerkin, host),
//
// with kc = -1 (A) or -(1 - i beta2) (shifted).  K_l is held as (2b+1)^2 planes
// of n^2 doubles (plane t = (dy+b)(2b+1) + dx+b), so a warp's loads of one tap are
// coalesced; the kernel adds it from the same staged input tile.
#pragma once

#include "kernels.cuh"

namespace hd {

constexpr int kGenMaxG = 6;
constexpr int kGenTY = 16, kGenTX = 32, kGenThreads = 256;

struct GenLevel {
  int n, b, G;
  const double* Y[kGenMaxG];  // n x (2b+1) band rows (y factor of group g)
  const double* X[kGenMaxG];  // n x (2b+1) band rows (x factor)
  double2 coef[kGenMaxG];
  const double* K;  // stored stencil planes (wedge), or null
  double2 kc;       // coefficient of the stored stencil
};

// Entry (r, s) of the level operator, r = iy*n+ix, s = (iy+dy)*n + ix+dx, |dy|,|dx| <= b.
__device__ __forceinline__ double2 gen_entry(const GenLevel& L, int iy, int ix, int dy, int dx) {
  const int NB = 2 * L.b + 1;
  double2 v = cmk(0.0, 0.0);
  for (int g = 0; g < L.G; ++g)
    v = cadd(v, cscale(L.Y[g][(size_t)iy * NB + dy + L.b] * L.X[g][(size_t)ix * NB + dx + L.b], L.coef[g]));
  if (L.K) {
    const size_t NN = (size_t)L.n * L.n;
    v = cadd(v, cscale(L.K[(size_t)((dy + L.b) * NB + dx + L.b) * NN + (size_t)iy * L.n + ix], L.kc));
  }
  return v;
}

// Sum over the (2B+1)^2 taps of the stored stencil at one point: K planes NN apart, x from the staged tile.
// The taps are accumulated in the order of the runtime loop (dy outer, dx inner), so the result is the same;
// unrolled, the coefficient loads of the point are issued ahead of their use instead of one at a time
// (C4, round 2: 45.6 -> 32 us per fine-level launch, 26.3 -> 23.4 ms per solve.  Also tried: one point per
// thread with all coefficients loaded into registers at kernel start, 190 registers: 26.7 ms; an L2 prefetch
// of the coefficients at kernel start: 24.4 ms).
template <int B>
__device__ __forceinline__ double2 gen_stencil_sum(const double* __restrict__ Kp, size_t NN, const double2* xr, int RW) {
  constexpr int NB = 2 * B + 1;
  double k[NB * NB];
#pragma unroll
  for (int e = 0; e < NB * NB; ++e) k[e] = __ldg(Kp + (size_t)e * NN);
  double2 t = cmk(0.0, 0.0);
#pragma unroll
  for (int dy = 0; dy < NB; ++dy)
#pragma unroll
    for (int dx = 0; dx < NB; ++dx) t = cfma_r(k[dy * NB + dx], xr[dy * RW + dx], t);
  return t;
}

__host__ __device__ constexpr size_t gen_smem(int b, int G) {
  return sizeof(double2) * ((size_t)(kGenTY + 2 * b) * (kGenTX + 2 * b) + (size_t)G * (kGenTY + 2 * b) * kGenTX);
}

// Output rows [rb, re) (a row slab; the whole grid: 0, n), addressed with
// global rows: a slab's pointers are shifted by its origin and its b halo rows
// above and below hold the neighbours' rows, so loads stay inside
// [rb - b, re + b).
template <int MODE>
__global__ void __launch_bounds__(kGenThreads) k_kron2d(GenLevel L, const double2* __restrict__ x,
                                                        const double2* __restrict__ bv, double2* __restrict__ out,
                                                        double omega, RedOut red, const int* xidx, size_t xstride,
                                                        int rb, int re) {
  if (xidx) x += (size_t)(*xidx) * xstride;
  extern __shared__ __align__(16) double2 gsm[];
  __shared__ double2 scratch[32];
  const int n = L.n, b = L.b, NB = 2 * b + 1, G = L.G;
  const int RW = kGenTX + 2 * b, RH = kGenTY + 2 * b;
  double2* xs = gsm;             // RH x RW
  double2* px = gsm + RH * RW;   // G x RH x kGenTX
  const int x0 = blockIdx.x * kGenTX, y0 = rb + blockIdx.y * kGenTY;
  for (int e = threadIdx.x; e < RH * RW; e += blockDim.x) {
    const int rr = e / RW, cc = e % RW;
    const int gy = y0 - b + rr, gx = x0 - b + cc;
    xs[e] = (gy >= 0 && gy < n && gy >= rb - b && gy < re + b && gx >= 0 && gx < n) ? x[(size_t)gy * n + gx]
                                                                                       : cmk(0.0, 0.0);
  }
  __syncthreads();
  // x pass: px[g][rr][c] = sum_j X_g(ix, j) x(row rr, ix + j - b)
  for (int e = threadIdx.x; e < G * RH * kGenTX; e += blockDim.x) {
    const int g = e / (RH * kGenTX), rem = e % (RH * kGenTX);
    const int rr = rem / kGenTX, c = rem % kGenTX;
    const int ix = x0 + c;
    double2 s = cmk(0.0, 0.0);
    if (ix < n) {
      const double* Xr = L.X[g] + (size_t)ix * NB;
      const double2* xr = xs + rr * RW + c;
      for (int j = 0; j < NB; ++j) s = cfma_r(__ldg(Xr + j), xr[j], s);
    }
    px[e] = s;
  }
  __syncthreads();
  double acc = 0.0;
  for (int e = threadIdx.x; e < kGenTY * kGenTX; e += blockDim.x) {
    const int r = e / kGenTX, c = e % kGenTX;
    const int iy = y0 + r, ix = x0 + c;
    if (iy >= re || iy >= n || ix >= n) continue;
    double2 y = cmk(0.0, 0.0);
    for (int g = 0; g < G; ++g) {
      const double* Yr = L.Y[g] + (size_t)iy * NB;
      const double2* pr = px + ((size_t)g * RH + r) * kGenTX + c;
      double2 t = cmk(0.0, 0.0);
      for (int d = 0; d < NB; ++d) t = cfma_r(__ldg(Yr + d), pr[d * kGenTX], t);
      y = cadd(y, cmul(L.coef[g], t));
    }
    const size_t gi = (size_t)iy * n + ix;
    if (L.K) {
      const size_t NN = (size_t)n * n;
      const double* Kp = L.K + gi;
      const double2* xr = xs + r * RW + c;
      double2 t;
      switch (b) {  // warp-uniform; the unrolled forms issue a point's coefficient loads before consuming them
        case 1: t = gen_stencil_sum<1>(Kp, NN, xr, RW); break;
        case 2: t = gen_stencil_sum<2>(Kp, NN, xr, RW); break;
        case 3: t = gen_stencil_sum<3>(Kp, NN, xr, RW); break;
        case 4: t = gen_stencil_sum<4>(Kp, NN, xr, RW); break;
        default: {
          t = cmk(0.0, 0.0);
          for (int dy = 0; dy < NB; ++dy)
            for (int dx = 0; dx < NB; ++dx) t = cfma_r(__ldg(Kp + (size_t)(dy * NB + dx) * NN), xr[dy * RW + dx], t);
        }
      }
      y = cadd(y, cmul(L.kc, t));
    }
    if (MODE == OP_APPLY) {
      out[gi] = y;
    } else if (MODE == OP_RESID) {
      out[gi] = csub(bv[gi], y);
    } else if (MODE == OP_RESNORM) {
      acc += cnorm2(csub(bv[gi], y));
    } else {
      double2 D = cmk(0.0, 0.0);
      for (int g = 0; g < G; ++g)
        D = cadd(D, cscale(__ldg(L.Y[g] + (size_t)iy * NB + b) * __ldg(L.X[g] + (size_t)ix * NB + b), L.coef[g]));
      if (L.K) D = cadd(D, cscale(__ldg(L.K + (size_t)(b * NB + b) * ((size_t)n * n) + gi), L.kc));
      out[gi] = cadd(xs[(r + b) * RW + c + b], cscale(omega, cmul(cinv(D), csub(bv[gi], y))));
    }
  }
  if (MODE == OP_RESNORM) {
    double2 total;
    if (grid_sum2(cmk(acc, 0.0), red.partials, red.counter, scratch, &total))
      *red.dst = red.raw ? total.x : sqrt(total.x) / red.scale;
  }
}

// x = omega D^-1 b (Jacobi sweep from a zero iterate), rows [rb, re)
__global__ void __launch_bounds__(256) k_jacobi0_gen(GenLevel L, const double2* __restrict__ bv,
                                                     double2* __restrict__ out, double omega, int rb, int re) {
  const int n = L.n;
  const size_t g0 = (size_t)rb * n, g1 = (size_t)re * n;
  for (size_t gi = g0 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; gi < g1; gi += (size_t)gridDim.x * blockDim.x) {
    const int iy = (int)(gi / n), ix = (int)(gi % n);
    const double2 D = gen_entry(L, iy, ix, 0, 0);
    out[gi] = cscale(omega, cmul(cinv(D), bv[gi]));
  }
}

// Dense column-major n^2 x n^2 matrix of the Kronecker sum (row = iy*n+ix,
// col = jy*n+jx), for the dense exact solves.
__global__ void k_dense_kron(GenLevel L, double2* __restrict__ A) {
  const int n = L.n, b = L.b, NB = 2 * b + 1;
  const size_t NN = (size_t)n * n, tot = NN * NN;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    const size_t row = e % NN, col = e / NN;
    const int iy = (int)(row / n), ix = (int)(row % n), jy = (int)(col / n), jx = (int)(col % n);
    const int dy = jy - iy, dx = jx - ix;
    A[e] = (dy >= -b && dy <= b && dx >= -b && dx <= b) ? gen_entry(L, iy, ix, dy, dx) : cmk(0.0, 0.0);
  }
}

__global__ void k_identity(double2* __restrict__ B, size_t NN) {
  const size_t tot = NN * NN;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x)
    B[e] = cmk((e % NN) == (e / NN) ? 1.0 : 0.0, 0.0);
}

}  // namespace hd
