// Shared-memory tiled 2D transfers (separable Kronecker-square stencils).
//
// Restriction rc = (z (x) z)^T r: a CTA stages the fine region that feeds an
// 8 x 32 tile of coarse points (coalesced, zero-filled outside), contracts x
// then y in shared memory, and writes the tile (interleaved or planar).
// Prolongation out = base +- (z (x) z) e: a CTA stages the coarse region of a
// 16 x 64 fine tile and produces 4 fine points per thread.
// linear z  (src/precond.cpp:57-76):  even j inject, odd j average;
// Bezier z  (src/precond.cpp:34-55):  even j 1/8 (1, 6-drop, 1), odd j 1/2 (1, 1).
#pragma once

#include "kernels.cuh"

namespace hd {

constexpr int kRQY = 8, kRQX = 32;   // coarse tile of the restriction
constexpr int kPFY = 16, kPFX = 64;  // fine tile of the prolongation

template <int KIND>
struct ZW {
  static constexpr int lo = KIND == 0 ? 0 : -1;
  static constexpr int nw = KIND == 0 ? 3 : 5;
  __device__ static double w(int o, double drop) {  // restriction weight at offset lo + o
    if (KIND == 0) return o == 1 ? 1.0 : 0.5;
    return o == 0 || o == 4 ? 0.125 : (o == 2 ? (6.0 - drop) / 8.0 : 0.5);
  }
};

// PLANAR: 0 interleaved output (outc), 1 planar (outp: re plane then im plane).
// J0 (interleaved only): also x0 = omega D^-1 rc, the first damped-Jacobi sweep
// of the coarse level Lc from the zero iterate (k_jacobi0_2d_t's arithmetic).
template <int KIND, int PLANAR, bool J0 = false>
__global__ void __launch_bounds__(256) k_restrict2d(double drop, const double2* __restrict__ r, int nf, int nc,
                                                    double2* __restrict__ outc, double* __restrict__ outp, int qb,
                                                    int qe, LevelDev Lc = LevelDev{}, double omega = 0.0,
                                                    double2* __restrict__ x0 = nullptr) {
  constexpr int lo = ZW<KIND>::lo, nw = ZW<KIND>::nw;
  constexpr int RR = 2 * kRQY + nw - 1;  // fine rows of the region
  constexpr int RC = 2 * kRQX + nw - 1;  // fine cols
  __shared__ double2 f[RR][RC + 1];
  __shared__ double2 tx[RR][kRQX];
  // coarse rows [qb, qe) (a row slab; whole grid: 0, nc), global row addressing
  const int qx0 = blockIdx.x * kRQX, qy0 = qb + blockIdx.y * kRQY;
  const int fx0 = 2 * qx0 + lo, fy0 = 2 * qy0 + lo;
  const int fymax = 2 * (min(qy0 + kRQY, qe) - 1) + lo + nw - 1;
  // all loads of the region issued before any is consumed (blockDim == 256)
  constexpr int NLD = (RR * RC + 255) / 256;
  double2 v[NLD];
#pragma unroll
  for (int k = 0; k < NLD; ++k) {
    const int e = threadIdx.x + k * 256;
    const int rr = e / RC, cc = e % RC;
    const int fy = fy0 + rr, fx = fx0 + cc;
    // only the fine rows the tile's coarse rows [qy0, min(qy0 + kRQY, qe)) use: a row slab's
    // buffer ends a halo below its last row, so a partial tile must not read past it
    v[k] = (e < RR * RC && fy >= 0 && fy < nf && fy <= fymax && fx >= 0 && fx < nf) ? __ldg(r + (size_t)fy * nf + fx)
                                                                                     : cmk(0.0, 0.0);
  }
#pragma unroll
  for (int k = 0; k < NLD; ++k) {
    const int e = threadIdx.x + k * 256;
    if (e < RR * RC) f[e / RC][e % RC] = v[k];
  }
  __syncthreads();
  double w[nw];
#pragma unroll
  for (int o = 0; o < nw; ++o) w[o] = ZW<KIND>::w(o, drop);
  for (int e = threadIdx.x; e < RR * kRQX; e += blockDim.x) {
    const int rr = e / kRQX, qx = e % kRQX;
    double2 s = cmk(0.0, 0.0);
#pragma unroll
    for (int o = 0; o < nw; ++o) s = cfma_r(w[o], f[rr][2 * qx + o], s);
    tx[rr][qx] = s;
  }
  __syncthreads();
  const size_t NC = (size_t)nc * nc;
  for (int e = threadIdx.x; e < kRQY * kRQX; e += blockDim.x) {
    const int qy = e / kRQX, qx = e % kRQX;
    const int gy = qy0 + qy, gx = qx0 + qx;
    if (gy >= qe || gx >= nc) continue;
    double2 s = cmk(0.0, 0.0);
#pragma unroll
    for (int o = 0; o < nw; ++o) s = cfma_r(w[o], tx[2 * qy + o][qx], s);
    const size_t gi = (size_t)gy * nc + gx;
    if (PLANAR) {
      outp[gi] = s.x;
      outp[gi + NC] = s.y;
    } else {
      outc[gi] = s;
      if (J0) {
        const int NB = 2 * Lc.b + 1;
        const double my = Lc.M[(size_t)gy * NB + Lc.b], sy = Lc.S[(size_t)gy * NB + Lc.b];
        const double mxx = Lc.M[(size_t)gx * NB + Lc.b], sxx = Lc.S[(size_t)gx * NB + Lc.b];
        const double2 D = csub(cmk(my * sxx + sy * mxx, 0.0), cscale(my * mxx, Lc.c));
        x0[gi] = cscale(omega, cmul(cinv(D), s));
      }
    }
  }
}

// Linear restriction rc = (z (x) z)^T r as a warp-streaming kernel (fine levels; k_restrict2d<0,0,J0>'s
// arithmetic in the same order, so the same bits): a warp owns 32 coarse columns of a strip of QR coarse
// rows and walks the 2 QR + 1 fine rows that feed them.  Per fine row a lane loads its two fine columns
// 2q, 2q+1 (32 contiguous bytes; the third tap 2q+2 is the next lane's first value, lane 31 loads its own),
// restricts in x in registers and adds the row into the (at most two) coarse rows it feeds; a coarse row is
// written when its third fine row has passed.  No shared memory, no block barrier, ~10 instructions per fine
// point (the tiled kernel: ~200, a quarter of them index arithmetic); kRSU fine rows are loaded ahead.
// C5 fine level: 19.1 -> 14.1 us per launch.  (The same treatment of the linear prolongation x += Z e gave
// 18.2 -> 17.3 us: that kernel already moves its 92 MB at 5.1 TB/s, so the tiled form stays.)
constexpr int kRSU = 4;      // fine rows in flight per warp
constexpr int kRSWarps = 4;  // warps per CTA (independent)

template <bool J0>
__global__ void __launch_bounds__(32 * kRSWarps) k_restrict_lin_stream(const double2* __restrict__ r, int nf, int nc,
                                                                        int QR, int strips_x, int ntasks,
                                                                        double2* __restrict__ outc, LevelDev Lc,
                                                                        double omega, double2* __restrict__ x0) {
  const int lane = threadIdx.x & 31;
  const int task = blockIdx.x * kRSWarps + (threadIdx.x >> 5);
  if (task >= ntasks) return;
  const int q0 = (task % strips_x) * 32, qy0 = (task / strips_x) * QR;
  const int qy1 = min(qy0 + QR, nc);
  const int qx = q0 + lane;             // this lane's coarse column
  const int c0 = 2 * qx;                // its first fine column
  const bool v0 = c0 < nf, v1 = c0 + 1 < nf, v2 = lane == 31 && c0 + 2 < nf;
  const int fy0 = 2 * qy0, nrows = 2 * (qy1 - qy0) + 1;  // fine rows fy0 .. fy0 + nrows - 1
  auto load_row = [&](int k, double2& a, double2& b, double2& e) {  // fine row fy0 + k (zero past the grid)
    const int fy = fy0 + k;
    const bool rv = k < nrows && fy < nf;
    const double2* p = r + (size_t)(rv ? fy : 0) * nf + c0;
    a = rv && v0 ? __ldg(p) : cmk(0.0, 0.0);
    b = rv && v1 ? __ldg(p + 1) : cmk(0.0, 0.0);
    e = rv && v2 ? __ldg(p + 2) : cmk(0.0, 0.0);
  };
  double2 fa[kRSU], fb[kRSU], fe[kRSU];
#pragma unroll
  for (int u = 0; u < kRSU; ++u) load_row(u, fa[u], fb[u], fe[u]);
  double2 acur = cmk(0.0, 0.0), aprev = cmk(0.0, 0.0);  // coarse rows q (started) and q - 1 (finishing)
  int q = qy0;
  const int NBc = J0 ? 2 * Lc.b + 1 : 1;
  for (int kb = 0; kb < nrows; kb += kRSU) {
#pragma unroll
    for (int u = 0; u < kRSU; ++u) {
      const int k = kb + u;
      if (k < nrows) {  // warp-uniform
        const double2 a = fa[u], b = fb[u];
        // third tap: the next lane's first value (lane 31: its own extra load)
        double2 cN = cmk(__shfl_down_sync(0xffffffffu, a.x, 1), __shfl_down_sync(0xffffffffu, a.y, 1));
        if (lane == 31) cN = fe[u];
        load_row(k + kRSU, fa[u], fb[u], fe[u]);  // refill the slot kRSU rows ahead
        // x restriction (weights 1/2, 1, 1/2 in tap order, k_restrict2d's chain from zero)
        const double2 tx = cfma_r(0.5, cN, cfma_r(1.0, b, cfma_r(0.5, a, cmk(0.0, 0.0))));
        if ((k & 1) == 0) {
          // even fine row 2 q: third tap of coarse row q - 1 (complete -> store), first tap of coarse row q
          if (k > 0) {
            const double2 sres = cfma_r(0.5, tx, aprev);
            const int gy = q - 1;
            if (qx < nc) {
              const size_t gi = (size_t)gy * nc + qx;
              outc[gi] = sres;
              if (J0) {
                const double my = Lc.M[(size_t)gy * NBc + Lc.b], sy = Lc.S[(size_t)gy * NBc + Lc.b];
                const double mxx = Lc.M[(size_t)qx * NBc + Lc.b], sxx = Lc.S[(size_t)qx * NBc + Lc.b];
                const double2 D = csub(cmk(my * sxx + sy * mxx, 0.0), cscale(my * mxx, Lc.c));
                x0[gi] = cscale(omega, cmul(cinv(D), sres));
              }
            }
          }
          acur = cfma_r(0.5, tx, cmk(0.0, 0.0));
        } else {
          // odd fine row 2 q + 1: middle tap of coarse row q, which then waits for its third tap
          aprev = cfma_r(1.0, tx, acur);
          ++q;
        }
      }
    }
  }
}

// fine index i -> coarse neighbours as offsets into a staged region starting at
// coarse index qbase; returns count.  Same stencil as pweights() in kernels.cuh.
template <int KIND>
__device__ __forceinline__ int pw2(int i, int nc, double drop, int* q, double* w) {
  int m = 0;
  auto push = [&](int qq, double ww) {
    if (qq >= 0 && qq < nc) {
      q[m] = qq;
      w[m] = ww;
      ++m;
    }
  };
  if (i & 1) {
    if (KIND == 0) {
      push((i - 1) / 2, 1.0);
    } else {
      push((i - 3) / 2, 0.125);
      push((i - 1) / 2, (6.0 - drop) / 8.0);
      push((i + 1) / 2, 0.125);
    }
  } else {
    push(i / 2 - 1, 0.5);
    push(i / 2, 0.5);
  }
  return m;
}

// Separable prolongation weights of fine index i into the zero-padded coarse
// region (local index l = q - q0, q0 = f0/2 - 1 for an even tile origin f0):
// the three taps cover local indices li-1, li, li+1 with li = i/2 - q0 for odd
// i (linear: 0, 1, 0; Bezier: 1/8, (6-drop)/8, 1/8 on (i-3)/2, (i-1)/2, (i+1)/2)
// and li-1, li for even i (1/2, 1/2 on i/2 - 1, i/2).  Coarse indices outside
// [0, nc) are zero in the region, which drops those entries exactly as the
// reference's stencil does (no renormalisation).
template <int KIND>
__device__ __forceinline__ void ptaps(int i, double drop, double& w0, double& w1, double& w2) {
  if (i & 1) {
    if (KIND == 0) { w0 = 0.0; w1 = 1.0; w2 = 0.0; }
    else { w0 = 0.125; w1 = (6.0 - drop) / 8.0; w2 = 0.125; }
  } else {
    w0 = 0.5; w1 = 0.5; w2 = 0.0;
  }
}

// PMODE 0: out += Z e (interleaved e);  1: out = s - Z e (planar e);  2: out = Z e (planar e)
template <int KIND, int PMODE>
__global__ void __launch_bounds__(256) k_prolong2d(double drop, const double2* __restrict__ ec,
                                                   const double* __restrict__ ep, int nf, int nc,
                                                   const double2* __restrict__ s, double2* __restrict__ out, int fb,
                                                   int fe) {
  constexpr int CR = kPFY / 2 + 3, CC = kPFX / 2 + 3;
  __shared__ double2 cs[CR][CC];
  __shared__ double2 ty[kPFY][CC];  // y-interpolated coarse columns for every fine row of the tile
  // fine rows [fb, fe) (a row slab, fb even; whole grid: 0, nf), global row addressing
  const int fx0 = blockIdx.x * kPFX, fy0 = fb + blockIdx.y * kPFY;
  const int qx0 = fx0 / 2 - 1, qy0 = fy0 / 2 - 1;  // region origin (may be -1)
  const int qymax = min(fy0 + kPFY, fe) / 2;        // largest coarse row a fine row < fe uses
  const size_t NC = (size_t)nc * nc;
  for (int e = threadIdx.x; e < CR * CC; e += blockDim.x) {
    const int rr = e / CC, cc = e % CC;
    const int qy = qy0 + rr, qx = qx0 + cc;
    double2 v = cmk(0.0, 0.0);
    // coarse rows past qymax feed no fine row of the tile below fe (and a row
    // slab's coarse buffer may end right after its halo)
    if (qy >= 0 && qy < nc && qy <= qymax && qx >= 0 && qx < nc) {
      const size_t qi = (size_t)qy * nc + qx;
      v = PMODE == 0 ? ec[qi] : cmk(ep[qi], ep[qi + NC]);
    }
    cs[rr][cc] = v;
  }
  __syncthreads();
  // y pass: fine row fy (local r) from coarse rows li-1..li+1, li = fy/2 - qy0
  for (int e = threadIdx.x; e < kPFY * CC; e += blockDim.x) {
    const int r = e / CC, cc = e % CC;
    const int fy = fy0 + r;
    const int li = fy / 2 - qy0;  // >= 1
    double w0, w1, w2;
    ptaps<KIND>(fy, drop, w0, w1, w2);
    double2 t;
    if (fy & 1) t = cfma_r(w0, cs[li - 1][cc], cfma_r(w1, cs[li][cc], cscale(w2, cs[li + 1][cc])));
    else t = cfma_r(w0, cs[li - 1][cc], cscale(w1, cs[li][cc]));
    ty[r][cc] = t;
  }
  __syncthreads();
  // x pass + combine with the fine vector, 4 points per thread (coalesced rows);
  // the fine-vector loads of all 4 points are issued first (blockDim == 256)
  constexpr int NPT = kPFY * kPFX / 256;
  double2 base[NPT];
#pragma unroll
  for (int k = 0; k < NPT; ++k) {
    const int e = threadIdx.x + k * 256;
    const int fy = fy0 + e / kPFX, fx = fx0 + e % kPFX;
    const size_t gi = (size_t)fy * nf + fx;
    base[k] = cmk(0.0, 0.0);
    if (PMODE != 2 && fy < fe && fx < nf) base[k] = PMODE == 0 ? out[gi] : __ldcs(s + gi);
  }
#pragma unroll
  for (int k = 0; k < NPT; ++k) {
    const int e = threadIdx.x + k * 256;
    const int r = e / kPFX, cx = e % kPFX;
    const int fy = fy0 + r, fx = fx0 + cx;
    if (fy >= fe || fx >= nf) continue;
    const int li = fx / 2 - qx0;
    double w0, w1, w2;
    ptaps<KIND>(fx, drop, w0, w1, w2);
    double2 acc;
    if (fx & 1) acc = cfma_r(w0, ty[r][li - 1], cfma_r(w1, ty[r][li], cscale(w2, ty[r][li + 1])));
    else acc = cfma_r(w0, ty[r][li - 1], cscale(w1, ty[r][li]));
    const size_t gi = (size_t)fy * nf + fx;
    if (PMODE == 0) out[gi] = cadd(base[k], acc);
    else if (PMODE == 1) out[gi] = csub(base[k], acc);
    else out[gi] = acc;
  }
}

// x = omega D^-1 b on a 2D level, 2D grid (no 64-bit div/mod per element)
__global__ void __launch_bounds__(256) k_jacobi0_2d_t(LevelDev L, const double2* __restrict__ b,
                                                      double2* __restrict__ out, double omega, int rb, int re) {
  const int n = L.n, NB = 2 * L.b + 1;
  const int ix = blockIdx.x * 64 + (threadIdx.x & 63);
  const int iy0 = rb + blockIdx.y * 16 + (threadIdx.x >> 6) * 4;
  if (ix >= n) return;
  double2 bv[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {  // all loads in flight before the divisions
    const int iy = iy0 + r;
    bv[r] = iy < re ? ld_stream(b + (size_t)iy * n + ix) : cmk(0.0, 0.0);
  }
  const double mxx = L.M[(size_t)ix * NB + L.b], sxx = L.S[(size_t)ix * NB + L.b];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int iy = iy0 + r;
    if (iy >= re) break;
    const double my = L.M[(size_t)iy * NB + L.b], sy = L.S[(size_t)iy * NB + L.b];
    const double2 D = csub(cmk(my * sxx + sy * mxx, 0.0), cscale(my * mxx, L.c));
    out[(size_t)iy * n + ix] = cscale(omega, cmul(cinv(D), bv[r]));
  }
}

}  // namespace hd
