// sm_100a kernels of the deflated multigrid-CSLP GMRES path, FP64 complex.
//
//   operator apply  k_op2d / k_op1d   A x, b - M x, damped Jacobi, ||f - A x||
//                                      (reference: every `(*A) * v` / `m * x` of
//                                      src/precond.cpp:107,140,147,238,262)
//   transfers       k_restrict* / k_prolong*   Z^T r, x += Z e, w - Z e
//                                      (linear MG stencil src/precond.cpp:57-76,
//                                       Bezier deflation stencil :34-55)
//   Krylov vectors  k_dot / k_axpy_dot / k_axpy_norm / k_iterate / k_givens
//                                      (src/linalg.cpp:40-90)
//   exact solvers   k_fd_small / k_fd_scale / k_bandlu_solve
//                                      (coarsest MG level src/precond.cpp:133,145
//                                       and deflation E solve :95-104)
//
// 2D operators are Kronecker sums of banded 1D factors,
//   L = My (x) Sx + Sy (x) Mx - c My (x) Mx,
// applied sum-factorised (x pass, then y pass) from 1D band tables -- the 2D
// matrix (125 M nonzeros at C5) is never stored or streamed.
#pragma once

#include "device_common.cuh"

namespace hd {

struct LevelDev {
  const double* S;  // n x (2b+1) band rows
  const double* M;
  int n;
  int b;
  double2 c;        // L = ... - c My(x)Mx   (2D)  or  S - c M  (1D)
  double2 corner;   // 1D only: added to L(n-1, n-1)
  const void* gen;  // host-side GenLevel (layered field, layered.cuh) or null; unused on the device
};

struct RedOut {
  double2* partials;
  unsigned* counter;
  double* dst;       // final scalar written by the last block
  double scale;      // dst = sqrt(sum |.|^2) / scale   (monitor: ||f|| or 1, src/precond.cpp:261-262)
  int raw;           // 1: dst = sum |.|^2 (a row slab's share; slabs are summed before the sqrt)
};

// OP_APPLYJ0: out = L x and out2 = omega D2^-1 (L x), D2 the diagonal of the
// level with constant c2 (the A apply that feeds the V-cycle also takes the
// first damped-Jacobi sweep of the shifted operator from the zero iterate)
// OP_JACOBIP: the Jacobi sweep of x + Z e, e the coarse correction (linear prolongation applied on the
// fly to the staged rows: the V-cycle's prolongation and its first post-smoothing sweep in one pass)
enum OpMode { OP_APPLY = 0, OP_RESID = 1, OP_JACOBI = 2, OP_RESNORM = 3, OP_APPLYJ0 = 4, OP_JACOBIP = 5 };

constexpr int kTX = 128;  // threads (columns) per stencil CTA
constexpr int kNS = 8;    // cp.async ring depth (rows in flight per CTA)

// ---------------------------------------------------------------------------
// 1D banded operator L = S - c M (+ corner), one thread per row.
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void k_op1d(LevelDev L, const double2* __restrict__ x, const double2* __restrict__ bv,
                       double2* __restrict__ out, double omega, RedOut red, const int* xidx, size_t xstride) {
  __shared__ double2 scratch[32];
  if (xidx) x += (size_t)(*xidx) * xstride;
  const int n = L.n, b = L.b, NB = 2 * b + 1;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double2 sxv = cmk(0.0, 0.0), mxv = cmk(0.0, 0.0);
    for (int d = -b; d <= b; ++d) {
      const int j = i + d;
      if (j < 0 || j >= n) continue;
      const double2 xv = x[j];
      sxv = cfma_r(L.S[(size_t)i * NB + d + b], xv, sxv);
      mxv = cfma_r(L.M[(size_t)i * NB + d + b], xv, mxv);
    }
    double2 y = csub(sxv, cmul(L.c, mxv));
    if (i == n - 1) y = cfma(L.corner, x[i], y);
    if (MODE == OP_APPLY) {
      out[i] = y;
    } else if (MODE == OP_RESID) {
      out[i] = csub(bv[i], y);
    } else if (MODE == OP_RESNORM) {
      acc += cnorm2(csub(bv[i], y));
    } else {
      double2 D = csub(cmk(L.S[(size_t)i * NB + b], 0.0), cscale(L.M[(size_t)i * NB + b], L.c));
      if (i == n - 1) D = cadd(D, L.corner);
      out[i] = cadd(x[i], cscale(omega, cmul(cinv(D), csub(bv[i], y))));
    }
  }
  if (MODE == OP_RESNORM) {
    double2 total;
    if (grid_sum2(cmk(acc, 0.0), red.partials, red.counter, scratch, &total)) *red.dst = sqrt(total.x) / red.scale;
  }
}

__global__ void k_jacobi0_1d(LevelDev L, const double2* __restrict__ b, double2* __restrict__ out, double omega) {
  const int n = L.n, NB = 2 * L.b + 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double2 D = csub(cmk(L.S[(size_t)i * NB + L.b], 0.0), cscale(L.M[(size_t)i * NB + L.b], L.c));
    if (i == n - 1) D = cadd(D, L.corner);
    out[i] = cscale(omega, cmul(cinv(D), b[i]));
  }
}

// ---------------------------------------------------------------------------
// Transfers.  kind 0: linear MG stencil, kind 1: Bezier deflation stencil.
// Restriction (Z^T r)[q] = sum_o w_o r[2q+o] over in-range fine rows:
//   linear  o = 0..2   w = (1/2, 1, 1/2)
//   Bezier  o = -1..3  w = (1/8, 1/2, (6-drop)/8, 1/2, 1/8)
// Prolongation (Z e)[i]: odd i (0-based) -> linear: e[(i-1)/2];
//   Bezier: 1/8 e[(i-3)/2] + (6-drop)/8 e[(i-1)/2] + 1/8 e[(i+1)/2];
//   even i -> 1/2 (e[i/2-1] + e[i/2]); out-of-range coarse entries dropped.
// ---------------------------------------------------------------------------
struct Stencil {
  int kind;
  double drop;
};

__device__ __forceinline__ int rweights(const Stencil& z, double* w) {  // returns o_lo
  if (z.kind == 0) {
    w[0] = 0.5; w[1] = 1.0; w[2] = 0.5; w[3] = 0.0; w[4] = 0.0;
    return 0;
  }
  w[0] = 0.125; w[1] = 0.5; w[2] = (6.0 - z.drop) / 8.0; w[3] = 0.5; w[4] = 0.125;
  return -1;
}

// fine index i -> up to 3 (coarse index, weight) pairs
__device__ __forceinline__ int pweights(const Stencil& z, int i, int nc, int* q, double* w) {
  int m = 0;
  auto push = [&](int qq, double ww) {
    if (qq >= 0 && qq < nc) { q[m] = qq; w[m] = ww; ++m; }
  };
  if (i & 1) {
    if (z.kind == 0) {
      push((i - 1) / 2, 1.0);
    } else {
      push((i - 3) / 2, 0.125);
      push((i - 1) / 2, (6.0 - z.drop) / 8.0);
      push((i + 1) / 2, 0.125);
    }
  } else {
    push(i / 2 - 1, 0.5);
    push(i / 2, 0.5);
  }
  return m;
}

// out: interleaved (planar == 0) or planar re/im planes of nc^dim (planar == 1)
template <int DIM>
__global__ void k_restrict(Stencil z, const double2* __restrict__ r, int nf, int nc, double2* __restrict__ outc,
                           double* __restrict__ outp) {
  double w[5];
  const int olo = rweights(z, w);
  const int nw = z.kind == 0 ? 3 : 5;
  const size_t NC = DIM == 2 ? (size_t)nc * nc : (size_t)nc;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < NC; g += (size_t)gridDim.x * blockDim.x) {
    double2 acc = cmk(0.0, 0.0);
    if (DIM == 1) {
      const int q = (int)g;
      for (int o = 0; o < nw; ++o) {
        const int i = 2 * q + olo + o;
        if (i >= 0 && i < nf) acc = cfma_r(w[o], r[i], acc);
      }
    } else {
      const int qy = (int)(g / nc), qx = (int)(g % nc);
      for (int oy = 0; oy < nw; ++oy) {
        const int iy = 2 * qy + olo + oy;
        if (iy < 0 || iy >= nf) continue;
        for (int ox = 0; ox < nw; ++ox) {
          const int ixx = 2 * qx + olo + ox;
          if (ixx < 0 || ixx >= nf) continue;
          acc = cfma_r(w[oy] * w[ox], r[(size_t)iy * nf + ixx], acc);
        }
      }
    }
    if (outp) {
      outp[g] = acc.x;
      outp[g + NC] = acc.y;
    } else {
      outc[g] = acc;
    }
  }
}

// mode 0: x += Z e (interleaved e);  mode 1: out = s - Z e (planar e);
// mode 2: out = Z e (planar e)
template <int DIM, int PMODE>
__global__ void k_prolong(Stencil z, const double2* __restrict__ ec, const double* __restrict__ ep, int nf, int nc,
                          const double2* __restrict__ s, double2* __restrict__ out) {
  const size_t NF = DIM == 2 ? (size_t)nf * nf : (size_t)nf;
  const size_t NC = DIM == 2 ? (size_t)nc * nc : (size_t)nc;
  auto ce = [&](size_t qi) -> double2 { return PMODE == 0 ? ec[qi] : cmk(ep[qi], ep[qi + NC]); };
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < NF; g += (size_t)gridDim.x * blockDim.x) {
    double2 acc = cmk(0.0, 0.0);
    if (DIM == 1) {
      int q[3]; double w[3];
      const int m = pweights(z, (int)g, nc, q, w);
      for (int a = 0; a < m; ++a) acc = cfma_r(w[a], ce(q[a]), acc);
    } else {
      const int iy = (int)(g / nf), ixx = (int)(g % nf);
      int qy[3], qx[3]; double wy[3], wx[3];
      const int my = pweights(z, iy, nc, qy, wy);
      const int mx = pweights(z, ixx, nc, qx, wx);
      for (int a = 0; a < my; ++a)
        for (int bb = 0; bb < mx; ++bb) acc = cfma_r(wy[a] * wx[bb], ce((size_t)qy[a] * nc + qx[bb]), acc);
    }
    if (PMODE == 0) out[g] = cadd(out[g], acc);
    else if (PMODE == 1) out[g] = csub(s[g], acc);
    else out[g] = acc;
  }
}

// ---------------------------------------------------------------------------
// Krylov vector kernels (MGS Arnoldi, src/linalg.cpp:41-47, 78-80, 89)
// ---------------------------------------------------------------------------
// dst = conj(a) . b
__global__ void k_dot(const double2* __restrict__ a, const double2* __restrict__ b, size_t N, RedOut red,
                      double2* dst) {
  __shared__ double2 scratch[32];
  double2 acc = cmk(0.0, 0.0);
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < N; g += (size_t)gridDim.x * blockDim.x)
    acc = cadd(acc, cconjmul(a[g], b[g]));
  double2 total;
  if (grid_sum2(acc, red.partials, red.counter, scratch, &total)) *dst = total;
}

// w -= h * vi ; dst = conj(vn) . w      (one fused MGS step)
__global__ void k_axpy_dot(double2* __restrict__ w, const double2* __restrict__ vi, const double2* __restrict__ h,
                           const double2* __restrict__ vn, size_t N, RedOut red, double2* dst) {
  __shared__ double2 scratch[32];
  const double2 hh = *h;
  double2 acc = cmk(0.0, 0.0);
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < N; g += (size_t)gridDim.x * blockDim.x) {
    const double2 nw = csub(w[g], cmul(hh, vi[g]));
    w[g] = nw;
    acc = cadd(acc, cconjmul(vn[g], nw));
  }
  double2 total;
  if (grid_sum2(acc, red.partials, red.counter, scratch, &total)) *dst = total;
}

// w -= h * vi ; hnew = ||w||  -> dst (as complex (hnew, 0)) and *dnorm
__global__ void k_axpy_norm(double2* __restrict__ w, const double2* __restrict__ vi, const double2* __restrict__ h,
                            size_t N, RedOut red, double2* dst) {
  __shared__ double2 scratch[32];
  const double2 hh = h ? *h : cmk(0.0, 0.0);
  double acc = 0.0;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < N; g += (size_t)gridDim.x * blockDim.x) {
    double2 nw = w[g];
    if (vi) {
      nw = csub(nw, cmul(hh, vi[g]));
      w[g] = nw;
    }
    acc += cnorm2(nw);
  }
  double2 total;
  if (grid_sum2(cmk(acc, 0.0), red.partials, red.counter, scratch, &total)) {
    const double nrm = sqrt(total.x);
    *dst = cmk(nrm, 0.0);
    if (red.dst) *red.dst = nrm;
  }
}

// out = a - b
__global__ void k_sub(const double2* __restrict__ a, const double2* __restrict__ b, double2* __restrict__ out,
                      size_t N) {
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < N; g += (size_t)gridDim.x * blockDim.x)
    out[g] = csub(a[g], b[g]);
}

// dst = src / h (h real, read from device; the reference's `w / hnew`)
__global__ void k_scale_inv(double2* __restrict__ dst, const double2* __restrict__ src, const double* __restrict__ h,
                            size_t N) {
  const double s = *h;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < N; g += (size_t)gridDim.x * blockDim.x) {
    const double2 v = src[g];
    dst[g] = cmk(v.x / s, v.y / s);
  }
}

// x = x0 + sum_{i<m} y_i V_i   (basis vectors contiguous, stride N)
__global__ void k_iterate(double2* __restrict__ x, const double2* __restrict__ x0, const double2* __restrict__ V,
                          const double2* __restrict__ y, int m, size_t N) {
  __shared__ double2 ys[128];
  for (int i = threadIdx.x; i < m && i < 128; i += blockDim.x) ys[i] = y[i];
  __syncthreads();
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < N; g += (size_t)gridDim.x * blockDim.x) {
    double2 acc = x0[g];
    for (int i = 0; i < m; ++i) acc = cfma(ys[i], V[(size_t)i * N + g], acc);
    x[g] = acc;
  }
}

// Givens update of column j + back substitution (src/linalg.cpp:49-77).
// H column-major with leading dimension ldh = maxit+1.
__device__ __forceinline__ double2 cdiv(double2 a, double2 b) { return cmul(a, cinv(b)); }
__device__ __forceinline__ double2 cconj(double2 a) { return cmk(a.x, -a.y); }

__global__ void k_givens(double2* H, int ldh, double2* g, double2* cs, double2* sn, double2* y, int j) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double2* col = H + (size_t)j * ldh;
  for (int i = 0; i < j; ++i) {
    const double2 a = col[i], b = col[i + 1];
    const double2 t = cadd(cmul(cs[i], a), cmul(sn[i], b));
    col[i + 1] = cadd(cmul(cmk(-sn[i].x, sn[i].y), a), cmul(cconj(cs[i]), b));
    col[i] = t;
  }
  const double2 hjj = col[j], hj1 = col[j + 1];
  const double denom = sqrt(cnorm2(hjj) + cnorm2(hj1));
  if (denom == 0.0) {
    cs[j] = cmk(1.0, 0.0);
    sn[j] = cmk(0.0, 0.0);
  } else {
    cs[j] = cmk(hjj.x / denom, -hjj.y / denom);
    sn[j] = cmk(hj1.x / denom, -hj1.y / denom);
  }
  col[j] = cadd(cmul(cs[j], hjj), cmul(sn[j], hj1));
  col[j + 1] = cmk(0.0, 0.0);
  const double2 gj = g[j];
  g[j + 1] = cmul(cmk(-sn[j].x, sn[j].y), gj);
  g[j] = cmul(cs[j], gj);
  const int m = j + 1;
  for (int i = m - 1; i >= 0; --i) {
    double2 s = g[i];
    for (int l = i + 1; l < m; ++l) s = csub(s, cmul(H[(size_t)l * ldh + i], y[l]));
    y[i] = cdiv(s, H[(size_t)i * ldh + i]);
  }
}

// ---------------------------------------------------------------------------
// Exact solvers
// ---------------------------------------------------------------------------
// Fast diagonalisation for a small Kronecker-sum operator (n <= 32), one CTA:
// X (n x n, interleaved, [qy][qx]) -> (V (x) V) diag(Dinv) (V (x) V)^T X.
// V column-major (V[i + k n] = v_k(i)), Dinv[ky*n + kx].
__global__ void k_fd_small(const double* __restrict__ V, const double2* __restrict__ Dinv, int n,
                           const double2* __restrict__ X, double2* __restrict__ Y) {
  __shared__ double2 A[32 * 32], Bm[32 * 32];
  __shared__ double Vs[32 * 32];
  const int nn = n * n;
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {
    A[e] = X[e];
    Vs[e] = V[e];
  }
  __syncthreads();
  // B[ky][qx] = sum_qy V(qy,ky) A[qy][qx]
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {
    const int ky = e / n, qx = e % n;
    double2 s = cmk(0.0, 0.0);
    for (int qy = 0; qy < n; ++qy) s = cfma_r(Vs[qy + ky * n], A[qy * n + qx], s);
    Bm[e] = s;
  }
  __syncthreads();
  // A[ky][kx] = Dinv * sum_qx V(qx,kx) B[ky][qx]
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {
    const int ky = e / n, kx = e % n;
    double2 s = cmk(0.0, 0.0);
    for (int qx = 0; qx < n; ++qx) s = cfma_r(Vs[qx + kx * n], Bm[ky * n + qx], s);
    A[e] = cmul(Dinv[e], s);
  }
  __syncthreads();
  // B[ky][qx] = sum_kx V(qx,kx) A[ky][kx]
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {
    const int ky = e / n, qx = e % n;
    double2 s = cmk(0.0, 0.0);
    for (int kx = 0; kx < n; ++kx) s = cfma_r(Vs[qx + kx * n], A[ky * n + kx], s);
    Bm[e] = s;
  }
  __syncthreads();
  // Y[qy][qx] = sum_ky V(qy,ky) B[ky][qx]
  for (int e = threadIdx.x; e < nn; e += blockDim.x) {
    const int qy = e / n, qx = e % n;
    double2 s = cmk(0.0, 0.0);
    for (int ky = 0; ky < n; ++ky) s = cfma_r(Vs[qy + ky * n], Bm[ky * n + qx], s);
    Y[e] = s;
  }
}

// planar complex T (re plane, im plane; n*n each) *= Dinv (complex, n*n)
__global__ void k_fd_scale(double* __restrict__ T, const double2* __restrict__ Dinv, size_t NN) {
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < NN; g += (size_t)gridDim.x * blockDim.x) {
    const double2 v = cmul(cmk(T[g], T[g + NN]), Dinv[g]);
    T[g] = v.x;
    T[g + NN] = v.y;
  }
}

// ---- reflection-folded fast diagonalisation (solver.cu make_fd_folded) ----
// Hh[yb] is col-major (4 n2) x n2, ld 4 n2: row q n2 + kx (q = 2 xb + p), column j,
// so each y transform is one (4 n2) x n2 x n2 GEMM per y parity.
__device__ __forceinline__ size_t fold_idx(int yb, int xb, int p, int kx, int j, int n2) {
  const size_t nn = (size_t)n2 * n2;
  return (size_t)yb * 4 * nn + (size_t)j * 4 * n2 + (size_t)(2 * xb + p) * n2 + kx;
}

// The three kernels below index with a 3D grid (x: the contiguous index, y: the row / column, z: the block), so
// no thread does 64-bit divisions (the grid-stride forms spent most of their instructions on them: 7-10 us each
// for 10-30 MB at C5).
//
// R[yb](q n2 + kx, ky), q = 2 xb + p: (R_p0 + i R_p1) *= D[yb][xb][ky][kx]     grid (ceil(n2 / 256), n2, 4)
__global__ void __launch_bounds__(256) k_scale_folded(double* __restrict__ R, const double2* __restrict__ D, int n2) {
  const int kx = blockIdx.x * 256 + threadIdx.x, ky = blockIdx.y;
  const int xb = blockIdx.z & 1, yb = blockIdx.z >> 1;
  if (kx >= n2) return;
  double* r0 = R + fold_idx(yb, xb, 0, kx, ky, n2);
  double* r1 = R + fold_idx(yb, xb, 1, kx, ky, n2);
  const double2 v = cmul(cmk(*r0, *r1), D[(((size_t)yb * 2 + xb) * n2 + ky) * n2 + kx]);
  *r0 = v.x;
  *r1 = v.y;
}

// Both reflections at once (x rows and y columns of the planar n x n input X):
// Q[xb][yb][p](i, j), i, j < n2: x rows folded first (a +- b), then y columns.
// Q blocks n2 x n2 column-major, block (2 xb + yb) 2 + p.                     grid (ceil(n2 / 256), n2, 2)
__global__ void __launch_bounds__(256) k_fold_both(const double* __restrict__ X, double* __restrict__ Q, int n, int n2) {
  const size_t nn = (size_t)n2 * n2, N2 = (size_t)n * n;
  const int i = blockIdx.x * 256 + threadIdx.x, j = blockIdx.y, p = blockIdx.z;
  if (i >= n2) return;
  const double* Xp = X + p * N2;
  const double a = Xp[(size_t)j * n + i], b = Xp[(size_t)j * n + (n - 1 - i)];
  const double c = Xp[(size_t)(n - 1 - j) * n + i], d = Xp[(size_t)(n - 1 - j) * n + (n - 1 - i)];
  const double f0 = a + b, f1 = a - b, g0 = c + d, g1 = c - d;  // x parity 0 / 1 at columns j, n-1-j
  const size_t o = (size_t)j * n2 + i;
  Q[(size_t)((0 * 2 + 0) * 2 + p) * nn + o] = f0 + g0;
  Q[(size_t)((0 * 2 + 1) * 2 + p) * nn + o] = f0 - g0;
  Q[(size_t)((1 * 2 + 0) * 2 + p) * nn + o] = f1 + g1;
  Q[(size_t)((1 * 2 + 1) * 2 + p) * nn + o] = f1 - g1;
}

// Inverse of k_fold_both: P[xb][yb][p] blocks -> planar n x n Y (y columns
// unfolded first, then x rows).                                                grid (ceil(n2 / 256), n2, 2)
__global__ void __launch_bounds__(256) k_unfold_both(const double* __restrict__ Pb, double* __restrict__ Y, int n, int n2) {
  const size_t nn = (size_t)n2 * n2, N2 = (size_t)n * n;
  const int i = blockIdx.x * 256 + threadIdx.x, j = blockIdx.y, p = blockIdx.z;
  if (i >= n2) return;
  const size_t o = (size_t)j * n2 + i;
  const double p00 = Pb[(size_t)((0 * 2 + 0) * 2 + p) * nn + o], p01 = Pb[(size_t)((0 * 2 + 1) * 2 + p) * nn + o];
  const double p10 = Pb[(size_t)((1 * 2 + 0) * 2 + p) * nn + o], p11 = Pb[(size_t)((1 * 2 + 1) * 2 + p) * nn + o];
  const double z0j = p00 + p01, z0m = p00 - p01, z1j = p10 + p11, z1m = p10 - p11;
  double* Yp = Y + p * N2;
  Yp[(size_t)j * n + i] = z0j + z1j;
  Yp[(size_t)j * n + (n - 1 - i)] = z0j - z1j;
  Yp[(size_t)(n - 1 - j) * n + i] = z0m + z1m;
  Yp[(size_t)(n - 1 - j) * n + (n - 1 - i)] = z0m - z1m;
}

// Banded LU solve, sequential in one thread, with the factors streamed into
// shared memory by the rest of the CTA one chunk ahead (double-buffered), so
// the dependent elimination chain only ever waits on shared memory.  The
// elimination window lives in registers (KL = lower bandwidth of L, the
// factor's upper bandwidth is 2 KL).  in/out interleaved or planar.
template <int KL>
__global__ void __launch_bounds__(256) k_bandlu_staged(const double2* __restrict__ Lf, const double2* __restrict__ Uf,
                                                       const double2* __restrict__ Uinv, const int* __restrict__ piv,
                                                       int n, const double2* __restrict__ b,
                                                       const double* __restrict__ bp, double2* __restrict__ work,
                                                       double2* __restrict__ x, double* __restrict__ xp) {
  constexpr int KU = 2 * KL;
  constexpr int CH = 256;
  extern __shared__ __align__(16) double2 sm[];
  // forward buffers: [2][CH*KL] L, [2][CH+KL] b (rows r0 .. r0+CH+KL-1: the
  // window refill never reads the next chunk), [2][CH] pivot offsets;
  // backward: [2][CH*KU] U, [2][CH] Uinv, [2][CH] y
  constexpr int CB = CH + KL;
  double2* fL = sm;
  double2* fB = fL + 2 * CH * KL;
  int* fP = reinterpret_cast<int*>(fB + 2 * CB);
  const int nch = (n + CH - 1) / CH;
  auto stage_fwd = [&](int c, int buf, int t0, int nt) {
    const int r0 = c * CH, rn = min(CH, n - r0), rb = min(CB, n - r0);
    for (int e = t0; e < rn * KL; e += nt) fL[buf * CH * KL + e] = Lf[(size_t)r0 * KL + e];
    for (int e = t0; e < rb; e += nt) fB[buf * CB + e] = bp ? cmk(bp[r0 + e], bp[r0 + e + n]) : b[r0 + e];
    for (int e = t0; e < rn; e += nt) fP[buf * CH + e] = piv[r0 + e] - (r0 + e);
  };
  stage_fwd(0, 0, threadIdx.x, blockDim.x);
  __syncthreads();
  // window w[0..KL] = rows k..k+KL of the (permuted, partially eliminated) rhs
  double2 w[KL + 1];
#pragma unroll
  for (int r = 0; r <= KL; ++r) w[r] = cmk(0.0, 0.0);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int r = 0; r < KL; ++r) w[r + 1] = r < n ? fB[r] : cmk(0.0, 0.0);
  }
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (threadIdx.x >= 32) {  // warps 1.. stage; warp 0 holds only the sequential lane
      if (c + 1 < nch) stage_fwd(c + 1, buf ^ 1, threadIdx.x - 32, blockDim.x - 32);
    } else if (threadIdx.x == 0) {
      const int r0 = c * CH, rn = min(CH, n - r0);
      const double2* bb = fB + buf * CB;
      const double2* lb = fL + buf * CH * KL;
      const int* pb = fP + buf * CH;
      // operands of step i are loaded during step i-1 (software pipeline)
      double2 ln[KL];
      int dpn = pb[0];
      double2 bn = (r0 + KL < n) ? bb[KL] : cmk(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < KL; ++r) ln[r] = lb[r];
      for (int i = 0; i < rn; ++i) {
        const int k = r0 + i;
        const int dp = dpn;
        double2 l[KL];
#pragma unroll
        for (int r = 0; r < KL; ++r) l[r] = ln[r];
        const double2 bin = bn;
        if (i + 1 < rn) {
          dpn = pb[i + 1];
#pragma unroll
          for (int r = 0; r < KL; ++r) ln[r] = lb[(i + 1) * KL + r];
          bn = (k + 1 + KL < n) ? bb[i + 1 + KL] : cmk(0.0, 0.0);
        }
        // window <- rows k .. k+KL: shift, and bring in row k+KL untouched so far
#pragma unroll
        for (int r = 0; r < KL; ++r) w[r] = w[r + 1];
        w[KL] = bin;
#pragma unroll
        for (int r = 1; r <= KL; ++r)
          if (dp == r) {
            const double2 t = w[0];
            w[0] = w[r];
            w[r] = t;
          }
#pragma unroll
        for (int r = 1; r <= KL; ++r) w[r] = csub(w[r], cmul(l[r - 1], w[0]));
        work[k] = w[0];
      }
    }
    __syncthreads();
  }
  // ---- backward: x_k = (y_k - sum_d U(k,k+d) x_{k+d}) / U(k,k), chunks in reverse
  double2* bU = sm;
  double2* bI = bU + 2 * CH * KU;
  double2* bY = bI + 2 * CH;
  auto stage_bwd = [&](int c, int buf, int t0, int nt) {
    const int r0 = c * CH, rn = min(CH, n - r0);
    for (int e = t0; e < rn * (KU + 1); e += nt) {
      const int i = e / (KU + 1), d = e % (KU + 1);
      if (d > 0) bU[buf * CH * KU + i * KU + (d - 1)] = Uf[(size_t)(r0 + i) * (KU + 1) + d];
    }
    for (int e = t0; e < rn; e += nt) {
      bI[buf * CH + e] = Uinv[r0 + e];
      bY[buf * CH + e] = __ldcg(&work[r0 + e]);
    }
  };
  __threadfence_block();
  stage_bwd(nch - 1, (nch - 1) & 1, threadIdx.x, blockDim.x);
  __syncthreads();
  double2 xv[KU];  // x_{k+1} .. x_{k+KU}
  if (threadIdx.x == 0) {
#pragma unroll
    for (int d = 0; d < KU; ++d) xv[d] = cmk(0.0, 0.0);
  }
  for (int c = nch - 1; c >= 0; --c) {
    const int buf = c & 1;
    if (threadIdx.x >= 32) {
      if (c > 0) stage_bwd(c - 1, buf ^ 1, threadIdx.x - 32, blockDim.x - 32);
    } else if (threadIdx.x == 0) {
      const int r0 = c * CH, rn = min(CH, n - r0);
      const double2* ub = bU + buf * CH * KU;
      double2 un[KU];
      double2 yn = bY[buf * CH + rn - 1], in_ = bI[buf * CH + rn - 1];
#pragma unroll
      for (int d = 0; d < KU; ++d) un[d] = ub[(rn - 1) * KU + d];
      for (int i = rn - 1; i >= 0; --i) {
        const int k = r0 + i;
        double2 u[KU];
#pragma unroll
        for (int d = 0; d < KU; ++d) u[d] = un[d];
        const double2 yk = yn, ik = in_;
        if (i > 0) {
#pragma unroll
          for (int d = 0; d < KU; ++d) un[d] = ub[(i - 1) * KU + d];
          yn = bY[buf * CH + i - 1];
          in_ = bI[buf * CH + i - 1];
        }
        // only the d = 1 term depends on the previous step: sum the rest first
        double2 s0 = yk, s1 = cmk(0.0, 0.0);
#pragma unroll
        for (int d = KU; d >= 2; --d) {
          if (d & 1) s0 = csub(s0, cmul(u[d - 1], xv[d - 1]));
          else s1 = csub(s1, cmul(u[d - 1], xv[d - 1]));
        }
        const double2 xk = cmul(csub(cadd(s0, s1), cmul(u[0], xv[0])), ik);
#pragma unroll
        for (int d = KU - 1; d > 0; --d) xv[d] = xv[d - 1];
        xv[0] = xk;
        if (xp) {
          xp[k] = xk.x;
          xp[k + n] = xk.y;
        } else {
          x[k] = xk;
        }
      }
    }
    __syncthreads();
  }
}

template <int KL>
constexpr size_t bandlu_smem() {
  constexpr int CH = 256;
  const size_t f = sizeof(double2) * (2 * CH * KL + 2 * (CH + KL)) + sizeof(int) * 2 * CH;
  const size_t b = sizeof(double2) * (2 * CH * 2 * KL + 4 * CH);
  return f > b ? f : b;
}

}  // namespace hd
