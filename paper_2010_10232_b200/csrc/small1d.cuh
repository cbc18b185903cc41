// Whole solve of a small 1D system in ONE single-CTA kernel (N <= kSmallMax):
// the transformed right-hand side, the start vector, and the reference's GMRES
// (src/linalg.cpp:10-92, modified Gram-Schmidt in the reference's order,
// conjugated Givens, back substitution and the iterate every iteration, the
// true-residual monitor) with the composed left-preconditioned operator
// (src/precond.cpp:236-245): A, c V-cycles of the shifted operator or its
// banded LU (C_ex), and the Bezier deflation with the banded LU of E.  All
// vectors live in shared memory; the basis and H in global memory (L2).
//
// On the 1D configs the per-kernel path is launch-latency bound (C1: 80
// unknowns, ~20 kernels per iteration at ~5 us each); here one iteration is a
// few dozen __syncthreads-separated phases.  Formulas and summation order per
// element follow k_op1d, k_jacobi0_1d, k_restrict<1>, k_prolong<1, *>,
// k_bandlu_solve and k_givens; the dot products are block reductions in a
// fixed order.
#pragma once

#include "tail1d.cuh"

namespace hd {

constexpr int kSmallMax = 512;      // unknowns
constexpr int kSmallThreads = 512;

struct SmallArgs {
  TailArgs mg;                      // the shifted hierarchy (level 0 = fine), as the tail V-cycle
  int shift, cycles;                // shift: 0 none, 1 V-cycles, 2 exact (C_ex, banded LU below)
  const double2 *sLf, *sUf;         // C_ex: banded LU of the fine shifted operator
  const int* spiv;
  int skl, sku;
  const double *AS, *AM;            // A = S - cA M (+ corner), band b = Ab
  int Ab;
  double2 cA, corner;
  int deflate, nc;
  double drop;
  const double2 *eLf, *eUf;         // E banded LU
  const int* epiv;
  int ekl, eku;
  int N, maxit;
  double tol;
  const double2* f;                 // rhs (global)
  double2* x;                       // solution (global)
  double2* V;                       // basis (global, (maxit+1) x N)
  double2* H;                       // (maxit+1) x maxit, column-major (global)
  double* res;                      // residual history (global, maxit + 1)
  int* state;                       // [0] iterations, [1] converged, [2] case: 0 loop, 1 r0 <= tol, 2 beta == 0
  int mg_off;                       // shared-memory layout (double2 units): the hierarchy at 0 ..
  int vec_off;                      //   then f, w, t1, t2, x0, xk, rhsp, ec (nc), scalars
};

// banded LU factors staged in shared memory (a single thread walks them)
__host__ __device__ inline size_t small_lu_words(int n, int kl, int ku) {
  return static_cast<size_t>(n) * kl + static_cast<size_t>(n) * (ku + 1) + (n + 1) / 2;  // L, U, piv (2 ints / double2)
}

__host__ inline size_t small_smem(const SmallArgs& a) {
  // vectors, ec, g/cs/sn/y/hcol, packed R of the Hessenberg QR
  size_t w = static_cast<size_t>(a.vec_off) + 7 * static_cast<size_t>(a.N) + a.nc + 5 * (a.maxit + 2) +
             static_cast<size_t>(a.maxit + 1) * (a.maxit + 2) / 2 + 64;
  if (a.shift == 1) w += small_lu_words(a.mg.n[a.mg.nl - 1], a.mg.kl, a.mg.ku);
  if (a.deflate) w += small_lu_words(a.nc, a.ekl, a.eku);
  return sizeof(double2) * w;
}

__device__ __forceinline__ double2* small_stage_lu(double2* dst, int n, int kl, int ku, const double2*& Lf,
                                                   const double2*& Uf, const int*& piv) {
  double2* L = dst;
  double2* U = L + (size_t)n * kl;
  int* P = reinterpret_cast<int*>(U + (size_t)n * (ku + 1));
  for (int e = threadIdx.x; e < n * kl; e += blockDim.x) L[e] = Lf[e];
  for (int e = threadIdx.x; e < n * (ku + 1); e += blockDim.x) U[e] = Uf[e];
  for (int e = threadIdx.x; e < n; e += blockDim.x) P[e] = piv[e];
  Lf = L;
  Uf = U;
  piv = P;
  return dst + small_lu_words(n, kl, ku);
}

// ---- block helpers -------------------------------------------------------
__device__ __forceinline__ double small_bsum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < nw; ++w) s += red[w];
  return s;
}

// sum_i conj(a_i) b_i
__device__ __forceinline__ double2 small_dot(const double2* a, const double2* b, int n, double* red) {
  double re = 0.0, im = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 t = cconjmul(a[i], b[i]);
    re += t.x;
    im += t.y;
  }
  const double sr = small_bsum(re, red);
  const double si = small_bsum(im, red);
  return cmk(sr, si);
}

__device__ __forceinline__ double small_norm(const double2* a, int n, double* red) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += cnorm2(a[i]);
  return sqrt(small_bsum(s, red));
}

// out = L x for a level of the hierarchy (l) or A (l < 0)
__device__ __forceinline__ void small_apply(const SmallArgs& a, const double2* x, double2* out) {
  const int n = a.N, b = a.Ab, NB = 2 * b + 1;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double2 sxv = cmk(0.0, 0.0), mxv = cmk(0.0, 0.0);
    for (int d = -b; d <= b; ++d) {
      const int j = i + d;
      if (j < 0 || j >= n) continue;
      const double2 xv = x[j];
      sxv = cfma_r(__ldg(a.AS + (size_t)i * NB + d + b), xv, sxv);
      mxv = cfma_r(__ldg(a.AM + (size_t)i * NB + d + b), xv, mxv);
    }
    double2 y = csub(sxv, cmul(a.cA, mxv));
    if (i == n - 1) y = cfma(a.corner, x[i], y);
    out[i] = y;
  }
  __syncthreads();
}

// Bezier restriction of the fine vector r into ec, E^-1 in place, then
// mode 1: out = s - Z ec;  mode 2: out = Z ec
__device__ void small_deflate(const SmallArgs& a, const double2* r, double2* ec, const double2* s, double2* out,
                              int mode) {
  const int n = a.N, nc = a.nc;
  const double w5[5] = {0.125, 0.5, (6.0 - a.drop) / 8.0, 0.5, 0.125};
  for (int q = threadIdx.x; q < nc; q += blockDim.x) {
    double2 acc = cmk(0.0, 0.0);
    for (int o = 0; o < 5; ++o) {
      const int i = 2 * q - 1 + o;
      if (i >= 0 && i < n) acc = cfma_r(w5[o], r[i], acc);
    }
    ec[q] = acc;
  }
  __syncthreads();
  tail_lu(ec, nc, a.eLf, a.eUf, a.epiv, a.ekl, a.eku);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double2 acc = cmk(0.0, 0.0);
    auto add = [&](int q, double w) {
      if (q >= 0 && q < nc) acc = cfma_r(w, ec[q], acc);
    };
    if (i & 1) {
      add((i - 3) / 2, 0.125);
      add((i - 1) / 2, (6.0 - a.drop) / 8.0);
      add((i + 1) / 2, 0.125);
    } else {
      add(i / 2 - 1, 0.5);
      add(i / 2, 0.5);
    }
    out[i] = mode == 1 ? csub(s[i], acc) : acc;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSmallThreads) k_solve1d_small(SmallArgs a) {
  extern __shared__ __align__(16) double2 ssm[];
  __shared__ double red[32];
  const int tid = threadIdx.x, nt = blockDim.x, N = a.N;
  double2* tsm = ssm + a.mg_off;
  double2* f = ssm + a.vec_off;
  double2* w = f + N;
  double2* t1 = w + N;
  double2* t2 = t1 + N;
  double2* x0 = t2 + N;
  double2* xk = x0 + N;
  double2* rhsp = xk + N;
  double2* ec = rhsp + N;
  double2* g = ec + a.nc;
  double2* cs = g + (a.maxit + 2);
  double2* sn = cs + (a.maxit + 2);
  double2* y = sn + (a.maxit + 2);
  double2* hcol = y + (a.maxit + 2);       // column j of H
  double2* R = hcol + (a.maxit + 2);       // packed upper triangle: column l at l (l + 1) / 2
  const int ldh = a.maxit + 1;
  (void)ldh;
  double2* mg_b0 = tsm + a.mg.off[0] + 2 * a.mg.n[0];
  // the coarsest level's and E's banded LU factors into shared memory
  TailArgs mg = a.mg;
  SmallArgs ax = a;
  double2* lu = R + (size_t)(a.maxit + 1) * (a.maxit + 2) / 2;
  if (a.shift == 1) lu = small_stage_lu(lu, mg.n[mg.nl - 1], mg.kl, mg.ku, mg.Lf, mg.Uf, mg.piv);
  if (a.deflate) lu = small_stage_lu(lu, a.nc, a.ekl, a.eku, ax.eLf, ax.eUf, ax.epiv);
  for (int i = tid; i < N; i += nt) f[i] = a.f[i];
  __syncthreads();
  const double fnorm = small_norm(f, N, red);
  const double scale = fnorm > 0.0 ? fnorm : 1.0;
  // shift inverse of v (into out): V-cycles or the exact banded LU
  auto shift_inv = [&](const double2* v, double2* out) {
    if (a.shift == 2) {
      for (int i = tid; i < N; i += nt) out[i] = v[i];
      __syncthreads();
      tail_lu(out, N, a.sLf, a.sUf, a.spiv, a.skl, a.sku);
      return;
    }
    for (int i = tid; i < N; i += nt) mg_b0[i] = v[i];
    __syncthreads();
    int cur0 = 0;
    for (int cy = 0; cy < a.cycles; ++cy) tail_vcycle(mg, tsm, cy == 0, &cur0);
    const double2* xs = tsm + a.mg.off[0] + cur0 * a.mg.n[0];
    for (int i = tid; i < N; i += nt) out[i] = xs[i];
    __syncthreads();
  };
  // out = op(v) (v, out distinct from t1, t2)
  auto op = [&](const double2* v, double2* out) {
    small_apply(a, v, t1);
    const double2* cur = t1;
    if (a.shift) {
      shift_inv(t1, t2);
      cur = t2;
    }
    if (a.deflate) {
      small_apply(a, cur, t1 == cur ? t2 : t1);
      small_deflate(ax, t1 == cur ? t2 : t1, ec, cur, out, 1);
    } else {
      for (int i = tid; i < N; i += nt) out[i] = cur[i];
      __syncthreads();
    }
  };
  auto monitor = [&](const double2* xv) {
    small_apply(a, xv, t1);
    double s = 0.0;
    for (int i = tid; i < N; i += nt) s += cnorm2(csub(f[i], t1[i]));
    return sqrt(small_bsum(s, red)) / scale;
  };
  // rhs' = P MG^-1 f ; x0 = Q f  (src/precond.cpp:247-256)
  const double2* b = f;
  if (a.shift) {
    shift_inv(f, w);
    b = w;
  }
  if (a.deflate) {
    small_apply(a, b, t1);
    small_deflate(ax, t1, ec, b, rhsp, 1);
    small_deflate(ax, f, ec, nullptr, x0, 2);
  } else {
    for (int i = tid; i < N; i += nt) {
      rhsp[i] = b[i];
      x0[i] = cmk(0.0, 0.0);
    }
    __syncthreads();
  }
  const double r0 = monitor(x0);
  if (r0 <= a.tol) {  // src/linalg.cpp:17-22
    for (int i = tid; i < N; i += nt) a.x[i] = x0[i];
    if (tid == 0) {
      a.res[0] = r0;
      a.state[0] = 0;
      a.state[1] = 1;
      a.state[2] = 1;
    }
    return;
  }
  // r = rhs' - op(x0); beta; V0 = r / beta  (src/linalg.cpp:24-33)
  op(x0, w);
  for (int i = tid; i < N; i += nt) w[i] = csub(rhsp[i], w[i]);
  __syncthreads();
  const double beta = small_norm(w, N, red);
  if (beta == 0.0) {
    const double rr = monitor(x0);
    for (int i = tid; i < N; i += nt) a.x[i] = x0[i];
    if (tid == 0) {
      a.state[0] = 0;
      a.state[1] = rr <= a.tol;
      a.state[2] = 2;
    }
    return;
  }
  for (int i = tid; i < N; i += nt) a.V[i] = cmk(w[i].x / beta, w[i].y / beta);
  for (int i = tid; i <= a.maxit; i += nt) g[i] = cmk(i == 0 ? beta : 0.0, 0.0);
  __syncthreads();
  int it = 0, conv = 0;
  for (int j = 0; j < a.maxit; ++j) {
    // w = op(v_j), v_j staged from the basis
    for (int i = tid; i < N; i += nt) xk[i] = a.V[(size_t)j * N + i];
    __syncthreads();
    op(xk, w);
    // modified Gram-Schmidt (src/linalg.cpp:42-45)
    for (int i = 0; i <= j; ++i) {
      const double2* vi = a.V + (size_t)i * N;
      double re = 0.0, im = 0.0;
      for (int q = tid; q < N; q += nt) {
        const double2 t = cconjmul(vi[q], w[q]);
        re += t.x;
        im += t.y;
      }
      const double2 h = cmk(small_bsum(re, red), small_bsum(im, red));
      for (int q = tid; q < N; q += nt) w[q] = csub(w[q], cmul(h, vi[q]));
      if (tid == 0) hcol[i] = h;
      __syncthreads();
    }
    const double hnew = small_norm(w, N, red);  // :46-47
    if (tid == 0) {
      double2* col = hcol;
      col[j + 1] = cmk(hnew, 0.0);
      // Givens (src/linalg.cpp:49-66) and back substitution (:70-77), as k_givens
      for (int i = 0; i < j; ++i) {
        const double2 p = col[i], q = col[i + 1];
        const double2 t = cadd(cmul(cs[i], p), cmul(sn[i], q));
        col[i + 1] = cadd(cmul(cmk(-sn[i].x, sn[i].y), p), cmul(cconj(cs[i]), q));
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
      double2* Rj = R + (size_t)j * (j + 1) / 2;
      for (int i = 0; i <= j; ++i) Rj[i] = col[i];
      const double2 gj = g[j];
      g[j + 1] = cmul(cmk(-sn[j].x, sn[j].y), gj);
      g[j] = cmul(cs[j], gj);
      const int m = j + 1;
      for (int i = m - 1; i >= 0; --i) {
        double2 s = g[i];
        for (int l = i + 1; l < m; ++l) s = csub(s, cmul(R[(size_t)l * (l + 1) / 2 + i], y[l]));
        y[i] = cdiv(s, R[(size_t)i * (i + 1) / 2 + i]);
      }
    }
    __syncthreads();
    // x_j = x0 + sum y_i v_i (:78-80), monitor (:82-88)
    for (int q = tid; q < N; q += nt) {
      double2 acc = x0[q];
      for (int i = 0; i <= j; ++i) acc = cfma(y[i], a.V[(size_t)i * N + q], acc);
      xk[q] = acc;
    }
    __syncthreads();
    const double rr = monitor(xk);
    if (tid == 0) a.res[j] = rr;
    it = j + 1;
    if (rr <= a.tol) {
      conv = 1;
      break;
    }
    if (hnew < 1e-300) break;  // breakdown
    if (j + 1 < a.maxit)
      for (int q = tid; q < N; q += nt) a.V[(size_t)(j + 1) * N + q] = cmk(w[q].x / hnew, w[q].y / hnew);
    __syncthreads();
  }
  for (int i = tid; i < N; i += nt) a.x[i] = xk[i];
  if (tid == 0) {
    a.state[0] = it;
    a.state[1] = conv;
    a.state[2] = 0;
  }
}

}  // namespace hd
