// Segmented (SPIKE-style) solve with a banded LU factorisation P A = L U
// (partial pivoting, L: KL sub-diagonals, U: KU = 2 KL super-diagonals) --
// the 1D exact solves (deflation E, C_ex, coarsest level) without the
// n-step sequential chain of the single-lane kernel.
//
// Both sweeps are linear recurrences with fixed coefficients:
//   forward  (LAPACK gbtrs order) on the window w = rows k..k+KL:
//            swap w_0 <-> w_p(k); y_k = w_0; w_q -= l(k+q, k) y_k; shift in b_{k+KL+1}
//   backward x_k = (y_k - sum_{d=1..KU} u(k, k+d) x_{k+d}) / u(k, k)
// The rows are cut into segments of Ls rows.  Every segment runs both sweeps
// locally from a zero boundary (the forward window starts from the raw rhs
// rows), in parallel; by linearity the true values differ from the local ones
// by h_k . Delta_i (forward: Delta_i = true window - raw rhs at the segment
// start) and h'_k . X_{i+1} (backward: X_{i+1} = the true x of the next KU
// rows).  h, h' and the window transfer matrices F_i are fixed and computed at
// setup; the boundary values follow from two short sequential scans over the
// segments:  Delta_{i+1} = D_i + F_i Delta_i,  X_i = X0_i + H'_i X_{i+1}.
// Arithmetic is that of the same factorisation; only the association of the
// sums changes (rounding-level differences).
#pragma once

#include "device_common.cuh"

namespace hd {

struct SegArgs {
  int n, P, Ls;               // rows, segments, rows per segment (last segment may be longer)
  const double2* L;           // n x KL multipliers
  const double2* U;           // n x (KU+1), U[k*(KU+1)] = u(k,k)
  const double2* Uinv;        // 1 / u(k,k)
  const int* piv;             // absolute pivot row
  const double2* hf;          // n x (KL+1): forward influence rows
  const double2* Ff;          // P x (KL+1)^2: forward transfer (row-major, [q][r])
  const double2* hb;          // n x KU: backward influence rows
  double2* y;                 // n: local forward results, then corrected y
  double2* x0;                // n: local backward results
  double2* D;                 // P x (KL+1): window increments
  double2* Dl;                // P x (KL+1): Delta_i
  double2* X0;                // P x KU: local x of the first KU rows of segment i
  double2* Xb;                // (P+1) x KU: true x of the first KU rows of segment i
};

__device__ __forceinline__ int seg_start(const SegArgs& a, int i) { return i * a.Ls; }
__device__ __forceinline__ int seg_end(const SegArgs& a, int i) { return i + 1 == a.P ? a.n : (i + 1) * a.Ls; }

__device__ __forceinline__ double2 seg_rhs(const double2* b, const double* bp, int n, int k) {
  if (k >= n) return cmk(0.0, 0.0);
  return bp ? cmk(bp[k], bp[k + n]) : b[k];
}

// local forward sweep of every segment (thread per segment)
template <int KL>
__global__ void k_seg_fwd(SegArgs a, const double2* __restrict__ b, const double* __restrict__ bp) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.P) return;
  const int s = seg_start(a, i), e = seg_end(a, i);
  double2 w[KL + 1];
#pragma unroll
  for (int q = 0; q <= KL; ++q) w[q] = seg_rhs(b, bp, a.n, s + q);
  for (int k = s; k < e; ++k) {
    const int p = a.piv[k] - k;
    double2 yk = w[0];
#pragma unroll
    for (int q = 1; q <= KL; ++q) yk = p == q ? w[q] : yk;
#pragma unroll
    for (int q = 1; q <= KL; ++q) {
      const double2 wq = p == q ? w[0] : w[q];
      w[q] = csub(wq, cmul(a.L[(size_t)k * KL + q - 1], yk));
    }
    a.y[k] = yk;
#pragma unroll
    for (int q = 0; q < KL; ++q) w[q] = w[q + 1];
    w[KL] = seg_rhs(b, bp, a.n, k + KL + 1);
  }
  // D_i = end window - raw rhs rows e..e+KL
#pragma unroll
  for (int q = 0; q <= KL; ++q) a.D[(size_t)i * (KL + 1) + q] = csub(w[q], seg_rhs(b, bp, a.n, e + q));
}

// Delta_0 = 0, Delta_{i+1} = D_i + F_i Delta_i   (one warp, lane q owns component q)
template <int KL>
__global__ void k_seg_scan_fwd(SegArgs a) {
  const int q = threadIdx.x;
  double2 dl = cmk(0.0, 0.0);
  for (int i = 0; i < a.P; ++i) {
    if (q <= KL) a.Dl[(size_t)i * (KL + 1) + q] = dl;
    double2 nx = q <= KL ? a.D[(size_t)i * (KL + 1) + q] : cmk(0.0, 0.0);
#pragma unroll
    for (int r = 0; r <= KL; ++r) {
      const double2 dr = cmk(__shfl_sync(0xffffffffu, dl.x, r), __shfl_sync(0xffffffffu, dl.y, r));
      if (q <= KL) nx = cfma(a.Ff[((size_t)i * (KL + 1) + q) * (KL + 1) + r], dr, nx);
    }
    dl = nx;
  }
}

// forward correction y_k += h_k . Delta_i, then the local backward sweep
template <int KL>
__global__ void k_seg_bwd(SegArgs a) {
  constexpr int KU = 2 * KL;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.P) return;
  const int s = seg_start(a, i), e = seg_end(a, i);
  double2 dl[KL + 1];
#pragma unroll
  for (int q = 0; q <= KL; ++q) dl[q] = a.Dl[(size_t)i * (KL + 1) + q];
  if (i > 0)
    for (int k = s; k < e; ++k) {
      double2 yk = a.y[k];
#pragma unroll
      for (int q = 0; q <= KL; ++q) yk = cfma(a.hf[(size_t)k * (KL + 1) + q], dl[q], yk);
      a.y[k] = yk;
    }
  double2 xw[KU];  // x_{k+1} .. x_{k+KU}
#pragma unroll
  for (int d = 0; d < KU; ++d) xw[d] = cmk(0.0, 0.0);
  for (int k = e - 1; k >= s; --k) {
    double2 sacc = a.y[k];
#pragma unroll
    for (int d = KU; d >= 1; --d) sacc = csub(sacc, cmul(a.U[(size_t)k * (KU + 1) + d], xw[d - 1]));
    const double2 xk = cmul(sacc, a.Uinv[k]);
#pragma unroll
    for (int d = KU - 1; d >= 1; --d) xw[d] = xw[d - 1];
    xw[0] = xk;
    a.x0[k] = xk;
  }
  // local x of the first KU rows (newest first in xw: xw[d] = x_{s+d})
#pragma unroll
  for (int d = 0; d < KU; ++d) a.X0[(size_t)i * KU + d] = xw[d];
}

// X_P = 0, X_i = X0_i + H'_i X_{i+1}   (H'_i rows: h'_{s+d}, d < KU)
template <int KL>
__global__ void k_seg_scan_bwd(SegArgs a) {
  constexpr int KU = 2 * KL;
  const int d = threadIdx.x;
  double2 xn = cmk(0.0, 0.0);
  if (d < KU) a.Xb[(size_t)a.P * KU + d] = xn;
  for (int i = a.P - 1; i >= 0; --i) {
    const int s = seg_start(a, i);
    double2 v = d < KU ? a.X0[(size_t)i * KU + d] : cmk(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < KU; ++r) {
      const double2 xr = cmk(__shfl_sync(0xffffffffu, xn.x, r), __shfl_sync(0xffffffffu, xn.y, r));
      if (d < KU) v = cfma(a.hb[(size_t)(s + d) * KU + r], xr, v);
    }
    xn = v;
    if (d < KU) a.Xb[(size_t)i * KU + d] = xn;
  }
}

// x_k = x0_k + h'_k . X_{i+1}  (thread per row), output interleaved or planar
template <int KL>
__global__ void k_seg_out(SegArgs a, double2* __restrict__ x, double* __restrict__ xp) {
  constexpr int KU = 2 * KL;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.n; k += gridDim.x * blockDim.x) {
    const int i = min(k / a.Ls, a.P - 1);
    double2 v = a.x0[k];
    if (i + 1 < a.P)
#pragma unroll
      for (int r = 0; r < KU; ++r) v = cfma(a.hb[(size_t)k * KU + r], a.Xb[(size_t)(i + 1) * KU + r], v);
    if (xp) {
      xp[k] = v.x;
      xp[k + a.n] = v.y;
    } else {
      x[k] = v;
    }
  }
}

}  // namespace hd
