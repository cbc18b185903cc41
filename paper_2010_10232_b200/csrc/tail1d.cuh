// 1D multigrid tail: every level from the first one with at most kTailMax
// rows down to the coarsest exact solve, as ONE single-CTA kernel with the
// level vectors in shared memory (src/precond.cpp:136-153 for those levels:
// damped Jacobi from zero, residual, linear restriction, recursion, linear
// prolongation, post-smoothing; the coarsest level by its banded LU).  On the
// 1D configs these levels are a few thousand rows at most, so a per-level
// kernel chain (five launches per level) is launch-latency bound; here the
// phases are separated by __syncthreads only.  tail_vcycle is shared with the
// whole-solve kernel of small1d.cuh.  Same formulas and summation
// order as k_op1d / k_jacobi0_1d / k_restrict<1> / k_prolong<1,0> /
// k_bandlu_solve.
#pragma once

#include "kernels.cuh"

namespace hd {

constexpr int kTailMax = 1024;     // rows of the first tail level
constexpr int kTailLevels = 12;
constexpr int kTailThreads = 512;

struct TailArgs {
  int nl;                          // tail levels (the last is the coarsest)
  int n[kTailLevels], b[kTailLevels];
  const double* S[kTailLevels];
  const double* M[kTailLevels];
  int off[kTailLevels];            // shared-memory offset (double2) of the level's 4 vectors
  double2 c;                       // shifted-operator coefficient (L = S - c M)
  double2 corner;                  // added to L(n-1, n-1) of the first tail level (global level 0 only)
  double omega;
  int nu;                          // smoothing steps
  const double2* Lf;               // coarsest banded LU (k_bandlu_solve layout)
  const double2* Uf;
  const int* piv;
  int kl, ku;
};

__host__ inline size_t tail_smem(const TailArgs& a) {
  size_t t = 0;
  for (int l = 0; l < a.nl; ++l) t += 4 * static_cast<size_t>(a.n[l]);
  return t * sizeof(double2);
}

// y = L x at row i of a tail level
__device__ __forceinline__ double2 tail_apply(const TailArgs& a, int l, const double2* x, int i, double2 corner) {
  const int n = a.n[l], b = a.b[l], NB = 2 * b + 1;
  double2 sxv = cmk(0.0, 0.0), mxv = cmk(0.0, 0.0);
  for (int d = -b; d <= b; ++d) {
    const int j = i + d;
    if (j < 0 || j >= n) continue;
    const double2 xv = x[j];
    sxv = cfma_r(__ldg(a.S[l] + (size_t)i * NB + d + b), xv, sxv);
    mxv = cfma_r(__ldg(a.M[l] + (size_t)i * NB + d + b), xv, mxv);
  }
  double2 y = csub(sxv, cmul(a.c, mxv));
  if (i == n - 1) y = cfma(corner, x[i], y);
  return y;
}

__device__ __forceinline__ double2 tail_diag(const TailArgs& a, int l, int i, double2 corner) {
  const int b = a.b[l], NB = 2 * b + 1;
  double2 D = csub(cmk(__ldg(a.S[l] + (size_t)i * NB + b), 0.0), cscale(__ldg(a.M[l] + (size_t)i * NB + b), a.c));
  if (i == a.n[l] - 1) D = cadd(D, corner);
  return D;
}

// banded LU solve in place (one thread), k_bandlu_solve's arithmetic
__device__ __forceinline__ void tail_lu(double2* w, int n, const double2* Lf, const double2* Uf, const int* piv, int kl,
                                         int ku) {
  if (threadIdx.x == 0) {
    for (int k = 0; k < n; ++k) {
      const int p = piv[k];
      if (p != k) {
        const double2 tmp = w[k];
        w[k] = w[p];
        w[p] = tmp;
      }
      const double2 wk = w[k];
      for (int r = 1; r <= kl && k + r < n; ++r) w[k + r] = csub(w[k + r], cmul(Lf[(size_t)k * kl + r - 1], wk));
    }
    for (int k = n - 1; k >= 0; --k) {
      double2 s = w[k];
      for (int d = 1; d <= ku && k + d < n; ++d) s = csub(s, cmul(Uf[(size_t)k * (ku + 1) + d], w[k + d]));
      w[k] = cdiv(s, Uf[(size_t)k * (ku + 1)]);
    }
  }
  __syncthreads();
}

// One V-cycle of the shifted hierarchy on the shared-memory levels (tail
// layout: per level x, y, b, r).  The fine right-hand side is in level 0's b;
// x_zero: the fine iterate starts from zero (else from level 0's current x,
// *cur0 says which buffer).  Returns the fine iterate's buffer index in *cur0.
__device__ void tail_vcycle(const TailArgs& a, double2* tsm, bool x_zero, int* cur0) {
  const int tid = threadIdx.x, nt = blockDim.x;
  auto X = [&](int l, int k) { return tsm + a.off[l] + k * a.n[l]; };
  int cur[kTailLevels];
  const int last = a.nl - 1;
  for (int l = 0; l < last; ++l) {
    const double2 corner = l == 0 ? a.corner : cmk(0.0, 0.0);
    const int n = a.n[l];
    double2* b = X(l, 2);
    double2* r = X(l, 3);
    int s0 = 0;
    if (l == 0 && !x_zero) {
      cur[l] = *cur0;
    } else {
      cur[l] = 0;
      if (a.nu == 0) {
        for (int i = tid; i < n; i += nt) X(l, 0)[i] = cmk(0.0, 0.0);
      } else {
        for (int i = tid; i < n; i += nt) X(l, 0)[i] = cscale(a.omega, cmul(cinv(tail_diag(a, l, i, corner)), b[i]));
        s0 = 1;
      }
      __syncthreads();
    }
    for (int s = s0; s < a.nu; ++s) {
      const double2* x = X(l, cur[l]);
      double2* y = X(l, cur[l] ^ 1);
      for (int i = tid; i < n; i += nt) {
        const double2 yv = tail_apply(a, l, x, i, corner);
        y[i] = cadd(x[i], cscale(a.omega, cmul(cinv(tail_diag(a, l, i, corner)), csub(b[i], yv))));
      }
      cur[l] ^= 1;
      __syncthreads();
    }
    const double2* x = X(l, cur[l]);
    for (int i = tid; i < n; i += nt) r[i] = csub(b[i], tail_apply(a, l, x, i, corner));
    __syncthreads();
    const int nc = a.n[l + 1];
    double2* bc = X(l + 1, 2);
    for (int q = tid; q < nc; q += nt) {
      double2 acc = cmk(0.0, 0.0);
      for (int o = 0; o < 3; ++o) {
        const int i = 2 * q + o;
        if (i < n) acc = cfma_r(o == 1 ? 1.0 : 0.5, r[i], acc);
      }
      bc[q] = acc;
    }
    __syncthreads();
  }
  {  // coarsest: banded LU
    const int n = a.n[last];
    double2* w = X(last, 0);
    cur[last] = 0;
    for (int i = tid; i < n; i += nt) w[i] = X(last, 2)[i];
    __syncthreads();
    tail_lu(w, n, a.Lf, a.Uf, a.piv, a.kl, a.ku);
  }
  for (int l = last - 1; l >= 0; --l) {
    const double2 corner = l == 0 ? a.corner : cmk(0.0, 0.0);
    const int n = a.n[l], nc = a.n[l + 1];
    double2* x = X(l, cur[l]);
    const double2* e = X(l + 1, cur[l + 1]);
    for (int i = tid; i < n; i += nt) {
      double2 acc = cmk(0.0, 0.0);
      if (i & 1) {
        const int q = (i - 1) / 2;
        if (q < nc) acc = cfma_r(1.0, e[q], acc);
      } else {
        if (i / 2 - 1 >= 0 && i / 2 - 1 < nc) acc = cfma_r(0.5, e[i / 2 - 1], acc);
        if (i / 2 < nc) acc = cfma_r(0.5, e[i / 2], acc);
      }
      x[i] = cadd(x[i], acc);
    }
    __syncthreads();
    const double2* b = X(l, 2);
    for (int s = 0; s < a.nu; ++s) {
      const double2* xs = X(l, cur[l]);
      double2* y = X(l, cur[l] ^ 1);
      for (int i = tid; i < n; i += nt) {
        const double2 yv = tail_apply(a, l, xs, i, corner);
        y[i] = cadd(xs[i], cscale(a.omega, cmul(cinv(tail_diag(a, l, i, corner)), csub(b[i], yv))));
      }
      cur[l] ^= 1;
      __syncthreads();
    }
  }
  *cur0 = cur[0];
}

__global__ void __launch_bounds__(kTailThreads) k_tail1d(TailArgs a, const double2* __restrict__ bin,
                                                         double2* __restrict__ xout) {
  extern __shared__ __align__(16) double2 tsm[];
  double2* b0 = tsm + a.off[0] + 2 * a.n[0];
  for (int i = threadIdx.x; i < a.n[0]; i += blockDim.x) b0[i] = bin[i];
  __syncthreads();
  int cur0 = 0;
  tail_vcycle(a, tsm, true, &cur0);
  const double2* x0 = tsm + a.off[0] + cur0 * a.n[0];
  for (int i = threadIdx.x; i < a.n[0]; i += blockDim.x) xout[i] = x0[i];
}

}  // namespace hd
