// Level operator and restriction in one pass:
//
//   rc = (z (x) z)^T r,   r = L x  (APPLY: the projection's A w, src/precond.cpp:106-107)
//                         r = b - L x  (RESID: the V-cycle residual, src/precond.cpp:147-149)
//
// r is never stored.  The kernel is the streaming stencil of stencil.cuh
// (each warp streams the rows of a strip through a cp.async ring, x pass from
// shared memory, y pass into rotating register accumulators), with the warp's
// 32 fine columns aligned to the restriction instead of to 32: warp w owns the
// coarse columns [q0, q0 + QW), q0 = w QW, and computes the fine columns
// 2 q0 + lo .. 2 q0 + lo + 31 that feed them (QW = 14 for the Bezier stencil,
// 15 for the linear one; neighbouring warps recompute the few shared fine
// columns).  Each completed fine row is restricted in x by warp shuffles
// (coarse column t of the warp sums lanes 2t .. 2t + nw - 1) and accumulated
// into the (at most 3) coarse rows it feeds; a coarse row is written when its
// last fine row has passed.  Fine rows and columns outside the grid are zero,
// which drops those stencil entries exactly as the reference does.
// A strip covers the fine rows of its coarse rows [qy0, qy1), so strips
// overlap by nw - 2 fine rows (recomputed).
//
// Output: interleaved (the next multigrid level's right-hand side, with J0 its
// first damped-Jacobi sweep from zero as in k_restrict2d) or planar (the
// deflation coarse vector fed to the E solve).
#pragma once

#include "stencil.cuh"
#include "transfer.cuh"

namespace hd {

template <int KIND>
__host__ __device__ constexpr int sr_qw() {
  return KIND == 0 ? 15 : 14;  // coarse columns per warp: 2 (QW - 1) + nw <= 32
}

template <int B, int MODE, int KIND, int PLANAR, bool J0>
__global__ void __launch_bounds__(kSW * kSWarps) k_stencil_restrict2d(LevelDev L, const double2* __restrict__ x,
                                                                      const double2* __restrict__ bv, double drop,
                                                                      int nc, int QR, double2* __restrict__ outc,
                                                                      double* __restrict__ outp, LevelDev Lc,
                                                                      double omega, double2* __restrict__ x0c) {
  constexpr int NB = 2 * B + 1;
  constexpr int W = kSW + 2 * B;
  constexpr int kSRing = stencil_ring<B>();
  constexpr bool NEED_B = MODE == OP_RESID;
  constexpr int lo = ZW<KIND>::lo, nw = ZW<KIND>::nw;
  constexpr int QW = sr_qw<KIND>();
  extern __shared__ __align__(16) double2 dsm[];
  double2(*ring)[kSRing][W] = reinterpret_cast<double2(*)[kSRing][W]>(dsm);
  double2(*bring)[kSRing][kSW] = reinterpret_cast<double2(*)[kSRing][kSW]>(dsm + kSWarps * kSRing * W);
  double2* cy = dsm + kSWarps * kSRing * (W + (NEED_B ? kSW : 0));

  const int n = L.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q0 = (blockIdx.x * kSWarps + warp) * QW;  // first coarse column of the warp
  const int x0 = 2 * q0 + lo;                          // its first fine column
  const int qy0 = blockIdx.y * QR, qy1 = min(qy0 + QR, nc);
  const int y0 = 2 * qy0 + lo;                         // first fine output row of the strip
  const int yend = 2 * (qy1 - 1) + lo + nw;            // one past the last
  const int nout = max(0, yend - y0);
  const int nin = nout + 2 * B;
  const int ix = x0 + lane;
  const bool colv = ix >= 0 && ix < n;

  // (My, Sy) of the strip's output rows, zero outside the grid and the strip
  for (int e = threadIdx.x; e < (nout + 4 * B) * NB; e += blockDim.x) {
    const int r = e / NB - 2 * B, d = e % NB;
    const int gy = y0 + r;
    cy[e] = (r >= 0 && r < nout && gy >= 0 && gy < n) ? cmk(L.M[(size_t)gy * NB + d], L.S[(size_t)gy * NB + d])
                                                       : cmk(0.0, 0.0);
  }
  double sx[NB], mx[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    sx[j] = colv ? L.S[(size_t)ix * NB + j] : 0.0;
    mx[j] = colv ? L.M[(size_t)ix * NB + j] : 0.0;
  }
  __syncthreads();
  if (q0 >= nc || nout == 0) return;
  double wz[nw];
#pragma unroll
  for (int o = 0; o < nw; ++o) wz[o] = ZW<KIND>::w(o, drop);
  double2(*rg)[W] = ring[warp];
  const int colA = x0 - B + lane;
  const int colB = x0 - B + kSW + lane;
  const bool okA = colA >= 0 && colA < n;
  const bool hasB = lane < 2 * B;
  const bool okB = hasB && colB >= 0 && colB < n;
  const double2* pA = x + (ptrdiff_t)(y0 - B) * n + (okA ? colA : 0);
  const double2* pB = x + (ptrdiff_t)(y0 - B) * n + (okB ? colB : 0);
  const double2* pb = bv + (ptrdiff_t)(y0 - 2 * B) * n + (colv ? ix : 0);
  int rl = y0 - B;  // global row of the next load
  auto load = [&](int sl) {
    const bool rv = (rl >= 0) && (rl < n);
    cp_async16(&rg[sl][lane], rv && okA ? pA : x, rv && okA);
    if (hasB) cp_async16(&rg[sl][kSW + lane], rv && okB ? pB : x, rv && okB);
    if (NEED_B) {
      const int rbw = rl - B;
      const bool v = (rbw >= y0) && (rbw < yend) && rbw >= 0 && rbw < n && colv;
      cp_async16(&bring[warp][sl][lane], v ? pb : bv, v);
      pb += n;
    }
    pA += n;
    pB += n;
    ++rl;
  };
#pragma unroll
  for (int k = 0; k < kSRing - 1; ++k) {
    if (k < nin) load(k);
    cp_async_commit();
  }
  double2 Y[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) Y[j] = cmk(0.0, 0.0);
  const double2 c = L.c;
  const double2* cyk = cy;
  // coarse-row accumulators of the rows qa, qa + 1, qa + 2 (lanes t < QW: coarse column q0 + t)
  double2 A0 = cmk(0.0, 0.0), A1 = cmk(0.0, 0.0), A2 = cmk(0.0, 0.0);
  int qa = qy0;
  const int t = lane;
  const bool cv = t < QW && q0 + t < nc;
  const size_t NC = (size_t)nc * nc;
  for (int kb = 0; kb < nin; kb += kSRing) {
#pragma unroll
    for (int tt = 0; tt < kSRing; ++tt) {
      const int k = kb + tt;
      const int s = tt;
      if (k < nin) {
        cp_async_wait<kSRing - 2>();
        __syncwarp();
        if (k + kSRing - 1 < nin) load((tt + kSRing - 1) % kSRing);
        cp_async_commit();
        double2 u0 = cmk(0.0, 0.0), u1 = cmk(0.0, 0.0), v0 = cmk(0.0, 0.0), v1 = cmk(0.0, 0.0);
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          const double2 xv = rg[s][lane + j];
          if (j & 1) {
            u1 = cfma_r(sx[j], xv, u1);
            v1 = cfma_r(mx[j], xv, v1);
          } else {
            u0 = cfma_r(sx[j], xv, u0);
            v0 = cfma_r(mx[j], xv, v0);
          }
        }
        const double2 v = cadd(v0, v1);
        const double2 Pk = csub(cadd(u0, u1), cmul(c, v));
#pragma unroll
        for (int d = 0; d < NB; ++d) {
          const double2 cyd = cyk[d * NB + (2 * B - d)];
          double2& yo = Y[(tt + 1 + d) % NB];
          yo = cfma_r(cyd.x, Pk, cfma_r(cyd.y, v, yo));
        }
        if (k >= 2 * B) {  // output row o = k - 2B of the strip is complete
          double2& yo = Y[(tt + 1) % NB];
          const int o = y0 + k - 2 * B;  // global fine row
          double2 r = cmk(0.0, 0.0);
          if (colv && o >= 0 && o < n) r = NEED_B ? csub(bring[warp][s][lane], yo) : yo;
          yo = cmk(0.0, 0.0);
          // x restriction: coarse column t sums fine lanes 2t .. 2t + nw - 1
          double2 cx = cmk(0.0, 0.0);
#pragma unroll
          for (int j = 0; j < nw; ++j) {
            const int src = min(2 * t + j, 31);
            const double2 rv = cmk(__shfl_sync(0xffffffffu, r.x, src), __shfl_sync(0xffffffffu, r.y, src));
            cx = cfma_r(wz[j], rv, cx);
          }
          // y restriction: fine row o feeds coarse rows qa .. qa+2 at offset j = o - (2 qy + lo)
          {
            const int j0 = o - (2 * qa + lo), j1 = j0 - 2, j2 = j0 - 4;
            if (j0 >= 0 && j0 < nw) A0 = cfma_r(ZW<KIND>::w(j0, drop), cx, A0);
            if (j1 >= 0 && j1 < nw) A1 = cfma_r(ZW<KIND>::w(j1, drop), cx, A1);
            if (j2 >= 0 && j2 < nw) A2 = cfma_r(ZW<KIND>::w(j2, drop), cx, A2);
          }
          if (o == 2 * qa + lo + nw - 1) {  // coarse row qa complete
            if (cv && qa < qy1) {
              const size_t gi = (size_t)qa * nc + q0 + t;
              if (PLANAR) {
                outp[gi] = A0.x;
                outp[gi + NC] = A0.y;
              } else {
                outc[gi] = A0;
                if (J0) {
                  const int NBc = 2 * Lc.b + 1, gx = q0 + t;
                  const double my = Lc.M[(size_t)qa * NBc + Lc.b], sy = Lc.S[(size_t)qa * NBc + Lc.b];
                  const double mxx = Lc.M[(size_t)gx * NBc + Lc.b], sxx = Lc.S[(size_t)gx * NBc + Lc.b];
                  const double2 D = csub(cmk(my * sxx + sy * mxx, 0.0), cscale(my * mxx, Lc.c));
                  x0c[gi] = cscale(omega, cmul(cinv(D), A0));
                }
              }
            }
            A0 = A1;
            A1 = A2;
            A2 = cmk(0.0, 0.0);
            ++qa;
          }
        }
        cyk += NB;
      }
    }
  }
  cp_async_wait<0>();
}

}  // namespace hd
