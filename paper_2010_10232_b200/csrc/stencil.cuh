// Sum-factorised Kronecker-sum stencil, warp-synchronous streaming version.
//
//   L = My (x) Sx + Sy (x) Mx - c My (x) Mx      (2D, x fastest)
//   y = My (Sx x - c Mx x) + Sy (Mx x)  =  sum_d My(iy,d) P(iy+d) + Sy(iy,d) Q(iy+d)
//
// Each warp owns 32 consecutive columns of a strip of rows and streams the
// rows through its own cp.async ring in shared memory (32 + 2B halo columns
// per row, zero-filled outside the domain); there is no block-level barrier
// in the row loop.  The x pass forms P = Sx x - c Mx x and Q = Mx x for the
// newest row; the y pass reads the last 2B+1 (P, Q) from register queues that
// are rotated statically (the row loop is unrolled by 2B+1), so no register
// moves are executed.  x-direction coefficients live in registers, the y
// coefficients of the strip in shared memory as (My, Sy) pairs.
//
// Modes: APPLY y; RESID b - y; JACOBI x + omega D^-1 (b - y); RESNORM
// ||b - y||^2 (deterministic grid reduction, no write).
#pragma once

#include "kernels.cuh"

namespace hd {

constexpr int kSW = 32;      // columns per warp
constexpr int kSWarps = 4;   // warps per CTA
constexpr int kSRing = 8;    // ring depth (rows in flight per warp)
constexpr int kSRows = 32;   // rows per strip (max)

template <int B, int MODE>
__global__ void __launch_bounds__(kSW * kSWarps) k_stencil2d(LevelDev L, const double2* __restrict__ x,
                                                            const double2* __restrict__ bv,
                                                            double2* __restrict__ out, double omega, int RY,
                                                            RedOut red, const int* xidx, size_t xstride) {
  if (xidx) x += (size_t)(*xidx) * xstride;  // graph mode: x = V + j N
  constexpr int NB = 2 * B + 1;
  constexpr int W = kSW + 2 * B;
  constexpr bool NEED_B = MODE != OP_APPLY;
  __shared__ __align__(16) double2 ring[kSWarps][kSRing][W];
  __shared__ __align__(16) double2 bring[NEED_B ? kSWarps : 1][NEED_B ? kSRing : 1][kSW];
  __shared__ __align__(16) double2 cy[kSRows + 1][NB];  // (My, Sy) per strip row
  __shared__ double2 scratch[32];

  const int n = L.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x0 = (blockIdx.x * kSWarps + warp) * kSW;
  const int y0 = blockIdx.y * RY;
  const int yend = min(y0 + RY, n);
  const int nout = max(0, yend - y0);
  const int nin = nout + 2 * B;
  const int ix = x0 + lane;
  const bool colv = ix < n;

  for (int e = threadIdx.x; e < nout * NB; e += blockDim.x) {
    const int r = e / NB, d = e % NB;
    cy[r][d] = cmk(L.M[(size_t)(y0 + r) * NB + d], L.S[(size_t)(y0 + r) * NB + d]);
  }
  double sx[NB], mx[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    sx[j] = colv ? L.S[(size_t)ix * NB + j] : 0.0;
    mx[j] = colv ? L.M[(size_t)ix * NB + j] : 0.0;
  }
  __syncthreads();  // cy staged (the only block barrier in the row loop's scope)
  if (x0 >= n && MODE != OP_RESNORM) return;
  double acc = 0.0;
  if (x0 < n) {
    double2(*rg)[W] = ring[warp];
    // per-lane load descriptors: main column and (lanes < 2B) one halo column
    const int colA = x0 - B + lane;
    const int colB = x0 - B + kSW + lane;
    const bool hasB = lane < 2 * B;
    auto load = [&](int k) {
      const int r = y0 - B + k;
      const int s = k % kSRing;
      const bool rv = (r >= 0) && (r < n);
      const double2* rowp = x + (size_t)(rv ? r : 0) * n;
      bool v = rv && colA >= 0 && colA < n;
      cp_async16(&rg[s][lane], rowp + (v ? colA : 0), v);
      if (hasB) {
        v = rv && colB < n;
        cp_async16(&rg[s][kSW + lane], rowp + (v ? colB : 0), v);
      }
      if (NEED_B) {
        const int rb = r - B;
        v = (rb >= y0) && (rb < yend) && colv;
        cp_async16(&bring[warp][s][lane], bv + (v ? (size_t)rb * n + ix : 0), v);
      }
    };
#pragma unroll
    for (int k = 0; k < kSRing - 1; ++k) {
      if (k < nin) load(k);
      cp_async_commit();
    }
    double2 P[NB], Q[NB], XC[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) P[j] = Q[j] = XC[j] = cmk(0.0, 0.0);
    const double2 c = L.c;
    // rows k = kb + t, t = 0..NB-1; slot of row k in the queues is k % NB == t
    for (int kb = 0; kb < nin; kb += NB) {
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        const int k = kb + t;
        if (k < nin) {
          cp_async_wait<kSRing - 2>();
          __syncwarp();
          if (k + kSRing - 1 < nin) load(k + kSRing - 1);
          cp_async_commit();
          const int s = k % kSRing;
          double2 u = cmk(0.0, 0.0), v = cmk(0.0, 0.0);
#pragma unroll
          for (int j = 0; j < NB; ++j) {
            const double2 xv = rg[s][lane + j];
            u = cfma_r(sx[j], xv, u);
            v = cfma_r(mx[j], xv, v);
          }
          P[t] = csub(u, cmul(c, v));
          Q[t] = v;
          if (MODE == OP_JACOBI) XC[t] = rg[s][lane + B];
          if (k >= 2 * B) {
            const int ro = k - 2 * B;  // output row offset; row iy+d sits in slot (t + 1 + d) % NB
            double2 y = cmk(0.0, 0.0);
#pragma unroll
            for (int d = 0; d < NB; ++d) {
              const int q = (t + 1 + d) % NB;
              const double2 cyd = cy[ro][d];
              y = cfma_r(cyd.x, P[q], y);
              y = cfma_r(cyd.y, Q[q], y);
            }
            if (colv) {
              const size_t gi = (size_t)(y0 + ro) * n + ix;
              if (MODE == OP_APPLY) {
                out[gi] = y;
              } else if (MODE == OP_RESID) {
                out[gi] = csub(bring[warp][s][lane], y);
              } else if (MODE == OP_RESNORM) {
                acc += cnorm2(csub(bring[warp][s][lane], y));
              } else {
                const double2 cyc = cy[ro][B];
                const double2 D = csub(cmk(cyc.x * sx[B] + cyc.y * mx[B], 0.0), cscale(cyc.x * mx[B], c));
                const double2 r = csub(bring[warp][s][lane], y);
                out[gi] = cadd(XC[(t + 1 + B) % NB], cscale(omega, cmul(cinv(D), r)));
              }
            }
          }
        }
      }
    }
    cp_async_wait<0>();
  }
  if (MODE == OP_RESNORM) {  // every thread of the CTA reaches this reduction
    double2 total;
    if (grid_sum2(cmk(acc, 0.0), red.partials, red.counter, scratch, &total)) *red.dst = sqrt(total.x) / red.scale;
  }
}

}  // namespace hd
