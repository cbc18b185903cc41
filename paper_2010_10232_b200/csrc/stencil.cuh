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
// moves are executed.  Every sum is split into two independent FMA chains
// (even / odd taps) to keep the FP64 pipe fed at low occupancy.
// x-direction coefficients live in registers, the y coefficients of the strip
// in shared memory as (My, Sy) pairs.  The strip height RY is chosen by the
// host so that the tile count fills whole waves of resident CTAs.
//
// Modes: APPLY y; APPLYJ0 y and omega D2^-1 y; RESID b - y; JACOBI x + omega D^-1 (b - y); RESNORM
// ||b - y||^2 (deterministic grid reduction, no write); JACOBIP: JACOBI of x + Z e (src/precond.cpp:151-152
// in one pass): the warp also stages the rows of the coarse correction e that its fine rows interpolate
// from and adds the linear prolongation (k_prolong2d's arithmetic: y then x, weights 1/2, 1/2 | 1) to
// every staged row before its x pass, so x + Z e is never stored.
#pragma once

#include "kernels.cuh"

namespace hd {

constexpr int kSW = 32;      // columns per warp
constexpr int kSWarps = 4;   // warps per CTA
constexpr int kSRowsMax = 128;
constexpr int kSCR = 16;     // JACOBIP: coarse rows in a warp's ring (>= (ring depth)/2 + 2)
constexpr int kSCW = 24;     // JACOBIP: coarse columns a warp's 32 + 2B fine columns interpolate from (B <= 6)

// ring depth (rows in flight per warp): the band height 2B+1 if that is >= 7,
// else its smallest multiple >= 8, so that the row loop unrolled over one ring period addresses
// both the ring slots and the rotating accumulators statically
// HD_SRING_MULT scales the depth by a whole number of band periods (A/B builds).
#ifndef HD_SRING_MULT
#define HD_SRING_MULT 1
#endif
template <int B>
__host__ __device__ constexpr int stencil_ring() {
  return HD_SRING_MULT * (2 * B + 1 >= 7 ? 2 * B + 1 : (2 * B + 1) * ((8 + 2 * B) / (2 * B + 1)));
}

template <int B, int MODE>
__host__ __device__ constexpr size_t stencil_smem(int ry) {
  return sizeof(double2) * ((size_t)kSWarps * stencil_ring<B>() * ((kSW + 2 * B) + (MODE != OP_APPLY && MODE != OP_APPLYJ0 ? kSW : 0)) +
                            (size_t)(ry + 4 * B + 1) * (2 * B + 1) +
                            (MODE == OP_JACOBIP ? (size_t)kSWarps * (kSCR + 1) * kSCW : 0));
}

#ifndef HD_STENCIL_MINB
#define HD_STENCIL_MINB 1
#endif

template <int B, int MODE>
__global__ void __launch_bounds__(kSW * kSWarps, HD_STENCIL_MINB) k_stencil2d(LevelDev L, const double2* __restrict__ x,
                                                            const double2* __restrict__ bv,
                                                            double2* __restrict__ out, double omega, int RY,
                                                            RedOut red, const int* xidx, size_t xstride, int rb,
                                                            int re, double2* __restrict__ out2, double2 c2,
                                                            const double2* __restrict__ ec = nullptr, int nc = 0) {
  constexpr int NB = 2 * B + 1;
  constexpr int W = kSW + 2 * B;
  constexpr int kSRing = stencil_ring<B>();
  constexpr bool NEED_B = MODE != OP_APPLY && MODE != OP_APPLYJ0;
  constexpr bool JAC = MODE == OP_JACOBI || MODE == OP_JACOBIP;
  if (xidx) x += (size_t)(*xidx) * xstride;  // graph mode: x = V + j N
  extern __shared__ __align__(16) double2 dsm[];
  double2(*ring)[kSRing][W] = reinterpret_cast<double2(*)[kSRing][W]>(dsm);
  double2(*bring)[kSRing][kSW] = reinterpret_cast<double2(*)[kSRing][kSW]>(dsm + kSWarps * kSRing * W);
  double2* cy = dsm + kSWarps * kSRing * (W + (NEED_B ? kSW : 0));  // (My, Sy) per strip row, NB each
  __shared__ double2 scratch[32];

  const int n = L.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int x0 = (blockIdx.x * kSWarps + warp) * kSW;
  // output rows [rb, re) (a row slab; the whole grid: 0, n).  Pointers are
  // addressed with global rows: rows of a slab's halo are read through them,
  // rows outside [0, n) are zero.
  const int y0 = rb + blockIdx.y * RY;
  const int yend = min(y0 + RY, re);
  const int nout = max(0, yend - y0);
  const int nin = nout + 2 * B;
  const int ix = x0 + lane;
  const bool colv = ix < n;
  // JACOBIP: this warp's ring of coarse rows (slot q & (kSCR-1), columns cq0 .. cq0 + kSCW - 1) and one
  // row of y-interpolated coarse values; they sit behind the (My, Sy) table of the tallest strip
  double2(*cr)[kSCW] = nullptr;
  double2* tyr = nullptr;
  const int cq0 = (x0 >> 1) + ((-B - 1) >> 1);  // floor((x0 - B - 1) / 2): x0 is a multiple of 32
  if (MODE == OP_JACOBIP) {
    double2* cbase = cy + (size_t)(RY + 4 * B + 1) * NB + (size_t)warp * (kSCR + 1) * kSCW;
    cr = reinterpret_cast<double2(*)[kSCW]>(cbase);
    tyr = cbase + kSCR * kSCW;
  }

  // (My, Sy) band rows of output rows o = -2B .. nout+2B-1 of the strip,
  // zero outside [0, nout): accumulation into out-of-strip rows is a no-op
  for (int e = threadIdx.x; e < (nout + 4 * B) * NB; e += blockDim.x) {
    const int r = e / NB - 2 * B, d = e % NB;
    cy[e] = (r >= 0 && r < nout) ? cmk(L.M[(size_t)(y0 + r) * NB + d], L.S[(size_t)(y0 + r) * NB + d])
                                 : cmk(0.0, 0.0);
  }
  double sx[NB], mx[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    sx[j] = colv ? L.S[(size_t)ix * NB + j] : 0.0;
    mx[j] = colv ? L.M[(size_t)ix * NB + j] : 0.0;
  }
  __syncthreads();  // cy staged (the only block barrier before the final reduction)
  if (x0 >= n && MODE != OP_RESNORM) return;
  double acc = 0.0;
  if (x0 < n) {
    double2(*rg)[W] = ring[warp];
    // per-lane load descriptors, advanced by one row per step
    const int colA = x0 - B + lane;
    const int colB = x0 - B + kSW + lane;
    const bool okA = colA >= 0 && colA < n;
    const bool hasB = lane < 2 * B;
    const bool okB = hasB && colB < n;
    const double2* pA = x + (ptrdiff_t)(y0 - B) * n + (okA ? colA : 0);
    const double2* pB = x + (ptrdiff_t)(y0 - B) * n + (okB ? colB : 0);
    const double2* pb = bv + (ptrdiff_t)(y0 - 2 * B) * n + (colv ? ix : 0);
    int rl = y0 - B;  // global row of the next load
    auto load = [&](int sl) {  // sl: its ring slot (static at every call site)
      const bool rv = (rl >= 0) && (rl < n);
      cp_async16(&rg[sl][lane], rv && okA ? pA : x, rv && okA);
      if (hasB) cp_async16(&rg[sl][kSW + lane], rv && okB ? pB : x, rv && okB);
      if (NEED_B) {
        const int rb = rl - B;
        const bool v = (rb >= y0) && (rb < yend) && colv;
        cp_async16(&bring[warp][sl][lane], v ? pb : bv, v);
        pb += n;
      }
      if (MODE == OP_JACOBIP && lane < kSCW) {
        // fine row rl interpolates from the coarse rows (rl-1)>>1 and rl>>1: a new one appears at even rl
        // (the strip's first row brings both); rows and columns outside the coarse grid are zero
        const int qc = cq0 + lane;
        const bool cv = qc >= 0 && qc < nc;
        auto cload = [&](int q) {
          const bool v = cv && q >= 0 && q < nc;
          cp_async16(&cr[q & (kSCR - 1)][lane], v ? ec + (size_t)q * nc + qc : ec, v);
        };
        if (rl == y0 - B && (rl & 1) == 0) cload((rl - 1) >> 1);
        if (rl == y0 - B || (rl & 1) == 0) cload(rl >> 1);
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
    // scatter form: row k contributes to the 2B+1 pending output rows
    // o = k-2B .. k; output o lives in accumulator slot o % NB == (t+1+d) % NB
    // for d = o - (k-2B), and is complete (stored) after row k = o + 2B.
    double2 Y[NB], XC[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) Y[j] = XC[j] = cmk(0.0, 0.0);
    const double2 c = L.c;
    double2* outp = out + (size_t)y0 * n + ix;
    const double2* cyk = cy;  // band row of output o = k - 2B (padded index o + 2B == k)
    for (int kb = 0; kb < nin; kb += kSRing) {
#pragma unroll
      for (int t = 0; t < kSRing; ++t) {
        const int k = kb + t;
        const int s = t;  // ring slot of row k (kb is a multiple of the ring depth)
        if (k < nin) {
          cp_async_wait<kSRing - 2>();
          __syncwarp();
          if (k + kSRing - 1 < nin) load((t + kSRing - 1) % kSRing);
          cp_async_commit();
          if (MODE == OP_JACOBIP) {  // rg[s] += (Z e)(row, .): y interpolation into tyr, then x
            const int rk = y0 - B + k;
            if (rk >= 0 && rk < n) {  // warp-uniform
              if (lane < kSCW) {
                const double2 cb = cr[(rk >> 1) & (kSCR - 1)][lane];
                tyr[lane] = (rk & 1) ? cb : cfma_r(0.5, cr[((rk - 1) >> 1) & (kSCR - 1)][lane], cscale(0.5, cb));
              }
              __syncwarp();
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int e = h * kSW + lane;
                const int fx = x0 - B + e;
                if ((h == 0 || lane < 2 * B) && fx >= 0 && fx < n) {
                  const int li = (fx >> 1) - cq0;
                  const double2 pz = (fx & 1) ? tyr[li] : cfma_r(0.5, tyr[li - 1], cscale(0.5, tyr[li]));
                  rg[s][e] = cadd(rg[s][e], pz);
                }
              }
            }
            __syncwarp();
          }
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
          if (JAC) XC[(t + 1 + B) % NB] = rg[s][lane + B];  // centre of output k - B
#pragma unroll
          for (int d = 0; d < NB; ++d) {
            // output o = k - 2B + d takes row k with its band offset 2B - d
            const double2 cyd = cyk[d * NB + (2 * B - d)];
            double2& yo = Y[(t + 1 + d) % NB];
            yo = cfma_r(cyd.x, Pk, cfma_r(cyd.y, v, yo));
          }
          if (k >= 2 * B) {  // output o = k - 2B is complete
            double2& yo = Y[(t + 1) % NB];
            if (colv) {
              if (MODE == OP_APPLY) {
                *outp = yo;
              } else if (MODE == OP_APPLYJ0) {
                *outp = yo;
                const double2 cyc = cyk[B];
                const double2 D = csub(cmk(cyc.x * sx[B] + cyc.y * mx[B], 0.0), cscale(cyc.x * mx[B], c2));
                out2[outp - out] = cscale(omega, cmul(cinv(D), yo));
              } else if (MODE == OP_RESID) {
                *outp = csub(bring[warp][s][lane], yo);
              } else if (MODE == OP_RESNORM) {
                acc += cnorm2(csub(bring[warp][s][lane], yo));
              } else {
                const double2 cyc = cyk[B];
                const double2 D = csub(cmk(cyc.x * sx[B] + cyc.y * mx[B], 0.0), cscale(cyc.x * mx[B], c));
                const double2 r = csub(bring[warp][s][lane], yo);
                *outp = cadd(XC[(t + 1) % NB], cscale(omega, cmul(cinv(D), r)));
              }
            }
            yo = cmk(0.0, 0.0);
            outp += n;
          }
          cyk += NB;
        }
      }
    }
    cp_async_wait<0>();
  }
  if (MODE == OP_RESNORM) {  // every thread of the CTA reaches this reduction
    double2 total;
    if (grid_sum2(cmk(acc, 0.0), red.partials, red.counter, scratch, &total))
      *red.dst = red.raw ? total.x : sqrt(total.x) / red.scale;
  }
}

}  // namespace hd
