// Deflation E solve by partial fast diagonalisation (2D, real shift):
// diagonalise x only, then one real banded LU solve per x mode along y.
//
//   E = E_M (x) E_S + E_S (x) E_M - k^2 E_M (x) E_M   (y outer, x inner)
//   E_S V = E_M V Lambda, V^T E_M V = I   =>   with X = Y V^T,  B V = [ T_m y_m ]_m,
//   T_m = E_S + (lam_m - k^2) E_M   (real, banded, indefinite)
//
// so  C = B V  (one GEMM), T_m y_m = c_m for every mode (LU with partial
// pivoting, factored at setup), X = Y V^T (one GEMM): two GEMMs instead of the
// four of the full diagonalisation.  The per-mode sweeps are the segmented
// (SPIKE-style) recurrences of segsolve.cuh with a mode dimension: every
// (mode, segment) pair runs both sweeps locally over kYL rows in parallel, a
// thread per mode scans the kYS segment boundaries, and a final elementwise
// pass adds the boundary influence.  Both planes (re, im) of a mode share the
// real factors and ride in the same thread.
//
// Layout (np = modes padded to 32; rows padded to kYS * kYL, identity):
//   C, Y, X0  [row][mode] per plane (plane stride nr * np), C = the GEMM output
//   TF [row][field][mode]: l(k+q,k) (KL), pivot offset, h_k (KL+1)
//   TB [row][field][mode]: 1/u_kk, u(k,k+d) (KU), h'_k (KU)
//   FM [seg][q][r][mode] forward window transfer;  HM [seg][d][r][mode] backward boundary map
#pragma once

#include "device_common.cuh"

namespace hd {

constexpr int kYL = 32;  // rows per segment

struct YArgs {
  int n, np, S, nr;      // modes/rows n, padded modes, segments, padded rows (S * kYL)
  const double* TF;
  const double* TB;
  const double* FM;
  const double* HM;
  double* C;             // in: rhs (GEMM output, ld np, planes n*np apart); out: solution
  double* Y;             // [nr][np] x 2 planes
  double* X0;            // [nr][np] x 2 planes
  double* D;             // [S][W][np] x 2
  double* Dl;            // [S][W][np] x 2
  double* XS;            // [S][KU][np] x 2: local x of the first KU rows
  double* XB;            // [S+1][KU][np] x 2: true x of the first KU rows
};

template <int KL>
__global__ void __launch_bounds__(128) k_ys_fwd(YArgs a) {
  HD_PDL_ENTRY();
  constexpr int W = KL + 1, NF = 2 * KL + 2;
  const int m = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  if (m >= a.np) return;
  const size_t np = a.np, pc = (size_t)a.n * np, pn = (size_t)a.nr * np;
  const int s = i * kYL;
  auto rhs = [&](int k, int pl) { return k < a.n ? a.C[pl * pc + (size_t)k * np + m] : 0.0; };
  double wr[W], wi[W];
#pragma unroll
  for (int q = 0; q < W; ++q) {
    wr[q] = rhs(s + q, 0);
    wi[q] = rhs(s + q, 1);
  }
#pragma unroll 4
  for (int r = 0; r < kYL; ++r) {
    const int k = s + r;
    const double* t = a.TF + (size_t)k * NF * np + m;
    const int p = (int)__ldg(t + KL * np);
    double yr = wr[0], yi = wi[0];
#pragma unroll
    for (int q = 1; q <= KL; ++q) {
      yr = p == q ? wr[q] : yr;
      yi = p == q ? wi[q] : yi;
    }
#pragma unroll
    for (int q = 1; q <= KL; ++q) {
      const double l = __ldg(t + (q - 1) * np);
      const double ar = p == q ? wr[0] : wr[q], ai = p == q ? wi[0] : wi[q];
      wr[q] = fma(-l, yr, ar);
      wi[q] = fma(-l, yi, ai);
    }
    a.Y[(size_t)k * np + m] = yr;
    a.Y[pn + (size_t)k * np + m] = yi;
#pragma unroll
    for (int q = 0; q < KL; ++q) {
      wr[q] = wr[q + 1];
      wi[q] = wi[q + 1];
    }
    wr[KL] = rhs(k + KL + 1, 0);
    wi[KL] = rhs(k + KL + 1, 1);
  }
  const size_t sp = (size_t)a.S * W * np;
#pragma unroll
  for (int q = 0; q < W; ++q) {
    const size_t o = ((size_t)i * W + q) * np + m;
    a.D[o] = wr[q] - rhs(s + kYL + q, 0);
    a.D[sp + o] = wi[q] - rhs(s + kYL + q, 1);
  }
}

// Delta_0 = 0, Delta_{i+1} = D_i + F_i Delta_i  (thread per mode)
template <int KL>
__global__ void k_ys_scan_fwd(YArgs a) {
  HD_PDL_ENTRY();
  constexpr int W = KL + 1;
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= a.np) return;
  const size_t np = a.np, sp = (size_t)a.S * W * np;
  double dr[W], di[W];
#pragma unroll
  for (int q = 0; q < W; ++q) dr[q] = di[q] = 0.0;
  for (int i = 0; i < a.S; ++i) {
    double nr[W], ni[W];
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const size_t o = ((size_t)i * W + q) * np + m;
      a.Dl[o] = dr[q];
      a.Dl[sp + o] = di[q];
      nr[q] = a.D[o];
      ni[q] = a.D[sp + o];
    }
#pragma unroll
    for (int q = 0; q < W; ++q)
#pragma unroll
      for (int r = 0; r < W; ++r) {
        const double f = __ldg(a.FM + (((size_t)i * W + q) * W + r) * np + m);
        nr[q] = fma(f, dr[r], nr[q]);
        ni[q] = fma(f, di[r], ni[q]);
      }
#pragma unroll
    for (int q = 0; q < W; ++q) {
      dr[q] = nr[q];
      di[q] = ni[q];
    }
  }
}

// y_k += h_k . Delta_i, then the local backward sweep
template <int KL>
__global__ void __launch_bounds__(128) k_ys_bwd(YArgs a) {
  HD_PDL_ENTRY();
  constexpr int W = KL + 1, KU = 2 * KL, NF = 2 * KL + 2, NB = 2 * KU + 1;
  const int m = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  if (m >= a.np) return;
  const size_t np = a.np, pn = (size_t)a.nr * np, sp = (size_t)a.S * W * np;
  const int s = i * kYL;
  double dr[W], di[W];
#pragma unroll
  for (int q = 0; q < W; ++q) {
    const size_t o = ((size_t)i * W + q) * np + m;
    dr[q] = a.Dl[o];
    di[q] = a.Dl[sp + o];
  }
  double xr[KU], xi[KU];  // x_{k+1} .. x_{k+KU}
#pragma unroll
  for (int d = 0; d < KU; ++d) xr[d] = xi[d] = 0.0;
#pragma unroll 4
  for (int r = kYL - 1; r >= 0; --r) {
    const int k = s + r;
    const double* tf = a.TF + (size_t)k * NF * np + m + (size_t)(KL + 1) * np;  // h_k
    const double* tb = a.TB + (size_t)k * NB * np + m;
    double sr = a.Y[(size_t)k * np + m], si = a.Y[pn + (size_t)k * np + m];
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const double h = __ldg(tf + q * np);
      sr = fma(h, dr[q], sr);
      si = fma(h, di[q], si);
    }
#pragma unroll
    for (int d = KU; d >= 1; --d) {
      const double u = __ldg(tb + d * np);
      sr = fma(-u, xr[d - 1], sr);
      si = fma(-u, xi[d - 1], si);
    }
    const double inv = __ldg(tb);
    sr *= inv;
    si *= inv;
#pragma unroll
    for (int d = KU - 1; d >= 1; --d) {
      xr[d] = xr[d - 1];
      xi[d] = xi[d - 1];
    }
    xr[0] = sr;
    xi[0] = si;
    a.X0[(size_t)k * np + m] = sr;
    a.X0[pn + (size_t)k * np + m] = si;
  }
  const size_t sx = (size_t)a.S * KU * np;
#pragma unroll
  for (int d = 0; d < KU; ++d) {  // xr[d] = x_{s+d}
    const size_t o = ((size_t)i * KU + d) * np + m;
    a.XS[o] = xr[d];
    a.XS[sx + o] = xi[d];
  }
}

// X_S = 0, X_i = XS_i + H_i X_{i+1}  (thread per mode)
template <int KL>
__global__ void k_ys_scan_bwd(YArgs a) {
  HD_PDL_ENTRY();
  constexpr int KU = 2 * KL;
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= a.np) return;
  const size_t np = a.np, sx = (size_t)a.S * KU * np, sb = (size_t)(a.S + 1) * KU * np;
  double xr[KU], xi[KU];
#pragma unroll
  for (int d = 0; d < KU; ++d) {
    xr[d] = xi[d] = 0.0;
    const size_t o = ((size_t)a.S * KU + d) * np + m;
    a.XB[o] = 0.0;
    a.XB[sb + o] = 0.0;
  }
  for (int i = a.S - 1; i >= 0; --i) {
    double vr[KU], vi[KU];
#pragma unroll
    for (int d = 0; d < KU; ++d) {
      const size_t o = ((size_t)i * KU + d) * np + m;
      vr[d] = a.XS[o];
      vi[d] = a.XS[sx + o];
#pragma unroll
      for (int r = 0; r < KU; ++r) {
        const double h = __ldg(a.HM + (((size_t)i * KU + d) * KU + r) * np + m);
        vr[d] = fma(h, xr[r], vr[d]);
        vi[d] = fma(h, xi[r], vi[d]);
      }
    }
#pragma unroll
    for (int d = 0; d < KU; ++d) {
      xr[d] = vr[d];
      xi[d] = vi[d];
      const size_t o = ((size_t)i * KU + d) * np + m;
      a.XB[o] = xr[d];
      a.XB[sb + o] = xi[d];
    }
  }
}

// x_k = x0_k + h'_k . X_{i+1}  -> C  (thread per (row, mode))
template <int KL>
__global__ void k_ys_out(YArgs a) {
  HD_PDL_ENTRY();
  constexpr int KU = 2 * KL, NB = 2 * KU + 1;
  const int m = blockIdx.x * blockDim.x + threadIdx.x, k = blockIdx.y;
  if (m >= a.np) return;
  const size_t np = a.np, pn = (size_t)a.nr * np, pc = (size_t)a.n * np, sb = (size_t)(a.S + 1) * KU * np;
  const int i = k / kYL;
  const double* hb = a.TB + (size_t)k * NB * np + m + (size_t)(KU + 1) * np;
  double vr = a.X0[(size_t)k * np + m], vi = a.X0[pn + (size_t)k * np + m];
#pragma unroll
  for (int d = 0; d < KU; ++d) {
    const double h = __ldg(hb + d * np);
    const size_t o = ((size_t)(i + 1) * KU + d) * np + m;
    vr = fma(h, a.XB[o], vr);
    vi = fma(h, a.XB[sb + o], vi);
  }
  a.C[(size_t)k * np + m] = vr;
  a.C[pc + (size_t)k * np + m] = vi;
}

}  // namespace hd
