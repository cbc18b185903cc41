// Sum-factorised Kronecker-sum stencil on the Blackwell tensor-copy engine.
//
//   L = My (x) Sx + Sy (x) Mx - c My (x) Mx      (2D, x fastest; see stencil.cuh)
//
// Same arithmetic, in the same order, as k_stencil2d (stencil.cuh): the x pass
// forms P = Sx x - c Mx x and Q = Mx x of the newest input row, the y pass
// scatters them into the 2B+1 pending output rows held in statically rotated
// register accumulators.  Outputs are bit-identical to k_stencil2d.
//
// What differs is how the data moves and how much each lane does:
//   * every warp is its own pipeline: lane 0 issues cp.async.bulk.tensor box
//     loads (UTMALDG) of kTSR input rows per stage into the warp's ring and the
//     warp waits on the stage's mbarrier.  Rows and columns outside the grid
//     are zero-filled by the copy engine, so the row loop has no edge
//     predicates and no per-lane address arithmetic for loads;
//   * a lane owns TWO adjacent columns: 2B+2 shared-memory loads feed two
//     x passes (instead of 2B+1 each), and the broadcast loads of the y
//     coefficients are shared by both columns;
//   * a warp's 64 columns are two 32-column regions A and B; the lanes
//     i = lane mod 8 < 4 of every quarter-warp work in A, the others in B, and
//     B's box starts one column early.  The 16-byte chunks a quarter-warp
//     reads in one LDS.128 are then 8 distinct chunks mod 8 (even ones from A,
//     odd ones from B): no bank conflicts although a lane's stride is 32 bytes;
//   * the y coefficients come per INPUT row r from a table CT built at setup:
//     CT[r][d] = (My, Sy)(o, r) for the outputs o = r - B + d (zero outside the
//     grid), and CT[r][2B+1] = the diagonal pair of output r - B (Jacobi).  A
//     row is 8 (B = 3) 16-byte pairs, copied per stage by one cp.async.bulk.
//
// A warp's task is a strip of 64 columns x RY output rows; tasks are numbered
// x fastest and dealt to the warps of the grid, one each (the host sizes RY so
// that the tasks fill the resident warps in one wave).
//
// Modes as stencil.cuh: APPLY, APPLYJ0, RESID, JACOBI, RESNORM.
#pragma once

#include <cuda.h>  // CUtensorMap (type only: cuTensorMapEncodeTiled is resolved through the runtime)

#include "stencil.cuh"

namespace hd {

constexpr int kTW = 64;     // columns per warp task
constexpr int kTWarps = 4;  // warps per CTA
constexpr int kTSR = 2;     // input rows per stage
constexpr int kTNS = 5;     // stages in a warp's ring
constexpr int kTBC = 64;    // columns of the right-hand-side box (one box per stage; its two loads per row pair
                            // take a 2-way bank conflict, 16 of ~50 wavefronts)

template <int B>
__host__ __device__ constexpr int tma_xc() {
  return 2 * B + 34;  // columns of an x box: 32 + 2B halo + the one-column shift, even
}
template <int B>
__host__ __device__ constexpr int tma_ctw() {
  return 2 * B + 2;  // pairs per CT row: 2B+1 band entries + the diagonal of output r - B
}
__host__ __device__ constexpr size_t tma_up128(size_t v) { return (v + 127) / 128 * 128; }

template <int B, int MODE>
struct TmaLayout {
  static constexpr bool NEED_B = MODE != OP_APPLY && MODE != OP_APPLYJ0;
  static constexpr size_t xbox = tma_up128((size_t)kTSR * tma_xc<B>() * 16);
  static constexpr size_t bbox = tma_up128((size_t)kTSR * kTBC * 16);
  static constexpr size_t ctb = tma_up128((size_t)kTSR * tma_ctw<B>() * 16);
  static constexpr size_t stage = 2 * xbox + (NEED_B ? bbox : 0) + ctb;
  static constexpr size_t warp = (size_t)kTNS * stage + 128;  // + the stage barriers
  static constexpr size_t total = (size_t)kTWarps * warp + 128;  // + alignment slack
  static constexpr unsigned tx = 2 * kTSR * tma_xc<B>() * 16 + (NEED_B ? kTSR * kTBC * 16 : 0) +
                                 kTSR * tma_ctw<B>() * 16;
};

__device__ __forceinline__ unsigned tq_sa(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void tq_mbar_init(unsigned b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(count));
}
__device__ __forceinline__ void tq_expect(unsigned b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tq_wait(unsigned b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @p bra D;\n bra W;\n"
      "D:\n}\n" ::"r"(b),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tq_box(unsigned dst, const CUtensorMap* tm, int c0, int c1, int c2, unsigned bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"(tm), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
// 16-byte shared-memory load at a 32-bit shared address + a compile-time offset (LDS.128)
template <int OFF>
__device__ __forceinline__ double2 tq_lds(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+%3];" : "=d"(v.x), "=d"(v.y) : "r"(a), "n"(OFF) : "memory");
  return v;
}
__device__ __forceinline__ void tq_bulk(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// CT of one level (see the header comment); rows r = -B .. n + B + pad - 1 at index r + B
__global__ void k_build_ct(LevelDev L, double2* __restrict__ ct, int rows) {
  const int NB = 2 * L.b + 1, CW = NB + 1, B = L.b;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * CW; e += gridDim.x * blockDim.x) {
    const int r = e / CW - B, d = e % CW;
    double2 v = cmk(0.0, 0.0);
    if (d < NB) {
      const int o = r - B + d;
      if (o >= 0 && o < L.n) v = cmk(L.M[(size_t)o * NB + (2 * B - d)], L.S[(size_t)o * NB + (2 * B - d)]);
    } else {
      const int o = r - B;
      if (o >= 0 && o < L.n) v = cmk(L.M[(size_t)o * NB + B], L.S[(size_t)o * NB + B]);
    }
    ct[e] = v;
  }
}

template <int B, int MODE>
__global__ void __launch_bounds__(32 * kTWarps, 2)
    k_stencil2d_tma(const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmb, LevelDev L,
                    const double2* __restrict__ ct, double2* __restrict__ out, double omega, int RY, int strips_x,
                    int ntasks, RedOut red, const int* xidx, double2* __restrict__ out2, double2 c2) {
  constexpr int NB = 2 * B + 1;
  constexpr int XC = tma_xc<B>();
  constexpr int CW = tma_ctw<B>();
  using Lay = TmaLayout<B, MODE>;
  constexpr bool NEED_B = Lay::NEED_B;
  constexpr unsigned kStage = (unsigned)Lay::stage;
  constexpr unsigned kCOff = 2 * (unsigned)Lay::xbox + (NEED_B ? (unsigned)Lay::bbox : 0u);  // CT rows of a stage
  extern __shared__ __align__(128) unsigned char tsm_raw[];
  __shared__ double2 scratch[32];

  const int n = L.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int task = blockIdx.x * kTWarps + warp;
  double acc = 0.0;
  if (task < ntasks) {
    const unsigned sbase = ((tq_sa(tsm_raw) + 127u) & ~127u) + (unsigned)warp * (unsigned)Lay::warp;
    const unsigned sbar = sbase + kTNS * kStage;
    const int tx_ = task % strips_x, ty_ = task / strips_x;
    const int X0 = tx_ * kTW;
    const int y0 = ty_ * RY;
    const int yend = min(y0 + RY, n);
    const int nout = yend - y0;
    const int nin = nout + 2 * B;
    const int nstages = (nin + kTSR - 1) / kTSR;
    const int jv = xidx ? *xidx : 0;

    // lane -> its two columns (region A: i < 4, region B: i >= 4 of every quarter-warp)
    const int q = lane >> 3, i8 = lane & 7, sel = i8 >> 2, pp = 4 * q + (i8 & 3);
    const int c0 = X0 + 32 * sel + 2 * pp;
    const bool v0 = c0 < n, v1 = c0 + 1 < n;

    if (lane == 0) {
#pragma unroll
      for (int s = 0; s < kTNS; ++s) tq_mbar_init(sbar + 8 * s, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncwarp();
    auto issue = [&](int g, int s) {  // lane 0: stage g (input rows y0 - B + g kTSR ...) into slot s = g % kTNS
      const int rl = y0 - B + g * kTSR;
      const unsigned sb = sbase + s * kStage, bar = sbar + 8 * s;
      tq_expect(bar, Lay::tx);
      tq_box(sb, &tmx, 2 * (X0 - B), rl, jv, bar);
      tq_box(sb + (unsigned)Lay::xbox, &tmx, 2 * (X0 + 32 - B - 1), rl, jv, bar);
      if (NEED_B) tq_box(sb + 2 * (unsigned)Lay::xbox, &tmb, 2 * X0, rl - B, 0, bar);
      tq_bulk(sb + kCOff, ct + (size_t)(rl + B) * CW, kTSR * CW * 16, bar);
    };
    if (lane == 0) {
      for (int g = 0; g < kTNS && g < nstages; ++g) issue(g, g);
    }

    double sx0[NB], mx0[NB], sx1[NB], mx1[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      sx0[j] = v0 ? L.S[(size_t)c0 * NB + j] : 0.0;
      mx0[j] = v0 ? L.M[(size_t)c0 * NB + j] : 0.0;
      sx1[j] = v1 ? L.S[(size_t)(c0 + 1) * NB + j] : 0.0;
      mx1[j] = v1 ? L.M[(size_t)(c0 + 1) * NB + j] : 0.0;
    }
    // per-lane byte offsets inside a stage
    const unsigned xoff = (sel ? (unsigned)Lay::xbox : 0u) + (unsigned)(2 * pp + sel) * 16u;
    const unsigned boff = 2 * (unsigned)Lay::xbox + (unsigned)(32 * sel + 2 * pp) * 16u;

    double2 Y0[NB], Y1[NB], XC0[NB], XC1[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) Y0[j] = Y1[j] = XC0[j] = XC1[j] = cmk(0.0, 0.0);
    const double2 c = L.c;
    double2* outp = out + (size_t)y0 * n + c0;
    // ring position of the row being computed (cur) and of the row whose x values are prefetched (nxt)
    int g = 0, s = 0, rs = 0;      // cur: global stage, slot, row in stage
    int ns = 0, nrs = 0;           // nxt: slot, row in stage
    unsigned nph = 0;              // parity of nxt's slot
    unsigned st = sbase;           // shared address of cur's stage
    unsigned nst = sbase;          // ... of nxt's stage
    double2 xv[NB + 1];
    tq_wait(sbar, 0);
    {
      const unsigned a = nst + xoff;
#pragma unroll
      for (int j = 0; j < NB + 1; ++j) xv[j] = cmk(0.0, 0.0);
      xv[0] = tq_lds<0>(a);
      if (NB + 1 > 1) xv[1] = tq_lds<16>(a);
      if (NB + 1 > 2) xv[2] = tq_lds<32>(a);
      if (NB + 1 > 3) xv[3] = tq_lds<48>(a);
      if (NB + 1 > 4) xv[4] = tq_lds<64>(a);
      if (NB + 1 > 5) xv[5] = tq_lds<80>(a);
      if (NB + 1 > 6) xv[6] = tq_lds<96>(a);
      if (NB + 1 > 7) xv[7] = tq_lds<112>(a);
      if (NB + 1 > 8) xv[8] = tq_lds<128>(a);
      if (NB + 1 > 9) xv[9] = tq_lds<144>(a);
      if (NB + 1 > 10) xv[10] = tq_lds<160>(a);
      if (NB + 1 > 11) xv[11] = tq_lds<176>(a);
      if (NB + 1 > 12) xv[12] = tq_lds<192>(a);
      if (NB + 1 > 13) xv[13] = tq_lds<208>(a);
    }
    for (int kb = 0; kb < nin; kb += NB) {
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        const int k = kb + t;
        if (k < nin) {
          // y coefficients of this input row (consumed after the x pass)
          const unsigned ca = st + kCOff + (unsigned)rs * (CW * 16);
          double2 cyv[NB + 1];
#pragma unroll
          for (int d = 0; d < NB + 1; ++d) cyv[d] = cmk(0.0, 0.0);
          cyv[0] = tq_lds<0>(ca);
          if (NB + 1 > 1) cyv[1] = tq_lds<16>(ca);
          if (NB + 1 > 2) cyv[2] = tq_lds<32>(ca);
          if (NB + 1 > 3) cyv[3] = tq_lds<48>(ca);
          if (NB + 1 > 4) cyv[4] = tq_lds<64>(ca);
          if (NB + 1 > 5) cyv[5] = tq_lds<80>(ca);
          if (NB + 1 > 6) cyv[6] = tq_lds<96>(ca);
          if (NB + 1 > 7) cyv[7] = tq_lds<112>(ca);
          if (NB + 1 > 8) cyv[8] = tq_lds<128>(ca);
          if (NB + 1 > 9) cyv[9] = tq_lds<144>(ca);
          if (NB + 1 > 10) cyv[10] = tq_lds<160>(ca);
          if (NB + 1 > 11) cyv[11] = tq_lds<176>(ca);
          if (NB + 1 > 12) cyv[12] = tq_lds<192>(ca);
          if (NB + 1 > 13) cyv[13] = tq_lds<208>(ca);
          double2 b0 = cmk(0.0, 0.0), b1 = cmk(0.0, 0.0);
          if (NEED_B) {
            const unsigned ba = st + boff + (unsigned)rs * (kTBC * 16);
            b0 = tq_lds<0>(ba);
            b1 = tq_lds<16>(ba);
          }
          // x pass
          double2 u0 = cmk(0.0, 0.0), u1 = cmk(0.0, 0.0), w0 = cmk(0.0, 0.0), w1 = cmk(0.0, 0.0);
          double2 p0 = cmk(0.0, 0.0), p1 = cmk(0.0, 0.0), r0 = cmk(0.0, 0.0), r1 = cmk(0.0, 0.0);
#pragma unroll
          for (int j = 0; j < NB; ++j) {
            if (j & 1) {
              u1 = cfma_r(sx0[j], xv[j], u1);
              w1 = cfma_r(mx0[j], xv[j], w1);
              p1 = cfma_r(sx1[j], xv[j + 1], p1);
              r1 = cfma_r(mx1[j], xv[j + 1], r1);
            } else {
              u0 = cfma_r(sx0[j], xv[j], u0);
              w0 = cfma_r(mx0[j], xv[j], w0);
              p0 = cfma_r(sx1[j], xv[j + 1], p0);
              r0 = cfma_r(mx1[j], xv[j + 1], r0);
            }
          }
          if (MODE == OP_JACOBI) {
            XC0[(t + 1 + B) % NB] = xv[B];
            XC1[(t + 1 + B) % NB] = xv[B + 1];
          }
          // the next row's x values: loaded now, behind the y pass of this row
          // (unconditional loads: past the last row they read a valid ring address and are unused)
          {
            if (++nrs == kTSR) {
              nrs = 0;
              nst += kStage;
              if (++ns == kTNS) {
                ns = 0;
                nph ^= 1u;
                nst = sbase;
              }
              if (k + 1 < nin) tq_wait(sbar + 8 * ns, nph);
            }
            const unsigned a = nst + xoff + (unsigned)nrs * (XC * 16);
            xv[0] = tq_lds<0>(a);
            if (NB + 1 > 1) xv[1] = tq_lds<16>(a);
            if (NB + 1 > 2) xv[2] = tq_lds<32>(a);
            if (NB + 1 > 3) xv[3] = tq_lds<48>(a);
            if (NB + 1 > 4) xv[4] = tq_lds<64>(a);
            if (NB + 1 > 5) xv[5] = tq_lds<80>(a);
            if (NB + 1 > 6) xv[6] = tq_lds<96>(a);
            if (NB + 1 > 7) xv[7] = tq_lds<112>(a);
            if (NB + 1 > 8) xv[8] = tq_lds<128>(a);
            if (NB + 1 > 9) xv[9] = tq_lds<144>(a);
            if (NB + 1 > 10) xv[10] = tq_lds<160>(a);
            if (NB + 1 > 11) xv[11] = tq_lds<176>(a);
            if (NB + 1 > 12) xv[12] = tq_lds<192>(a);
            if (NB + 1 > 13) xv[13] = tq_lds<208>(a);
          }
          const double2 va = cadd(w0, w1), vb = cadd(r0, r1);
          const double2 Pa = csub(cadd(u0, u1), cmul(c, va));
          const double2 Pb = csub(cadd(p0, p1), cmul(c, vb));
#pragma unroll
          for (int d = 0; d < NB; ++d) {
            const double2 cyd = cyv[d];
            double2& ya = Y0[(t + 1 + d) % NB];
            double2& yb = Y1[(t + 1 + d) % NB];
            ya = cfma_r(cyd.x, Pa, cfma_r(cyd.y, va, ya));
            yb = cfma_r(cyd.x, Pb, cfma_r(cyd.y, vb, yb));
          }
          {
            double2& ya = Y0[(t + 1) % NB];
            double2& yb = Y1[(t + 1) % NB];
            if (k >= 2 * B) {  // output row y0 + k - 2B is complete
              const double2 cyc = cyv[NB];
              if (MODE == OP_APPLY) {
                if (v0) outp[0] = ya;
                if (v1) outp[1] = yb;
              } else if (MODE == OP_APPLYJ0) {
                if (v0) {
                  outp[0] = ya;
                  const double2 D = csub(cmk(cyc.x * sx0[B] + cyc.y * mx0[B], 0.0), cscale(cyc.x * mx0[B], c2));
                  out2[outp - out] = cscale(omega, cmul(cinv(D), ya));
                }
                if (v1) {
                  outp[1] = yb;
                  const double2 D = csub(cmk(cyc.x * sx1[B] + cyc.y * mx1[B], 0.0), cscale(cyc.x * mx1[B], c2));
                  out2[outp - out + 1] = cscale(omega, cmul(cinv(D), yb));
                }
              } else if (MODE == OP_RESID) {
                if (v0) outp[0] = csub(b0, ya);
                if (v1) outp[1] = csub(b1, yb);
              } else if (MODE == OP_RESNORM) {
                if (v0) acc += cnorm2(csub(b0, ya));
                if (v1) acc += cnorm2(csub(b1, yb));
              } else {
                if (v0) {
                  const double2 D = csub(cmk(cyc.x * sx0[B] + cyc.y * mx0[B], 0.0), cscale(cyc.x * mx0[B], c));
                  outp[0] = cadd(XC0[(t + 1) % NB], cscale(omega, cmul(cinv(D), csub(b0, ya))));
                }
                if (v1) {
                  const double2 D = csub(cmk(cyc.x * sx1[B] + cyc.y * mx1[B], 0.0), cscale(cyc.x * mx1[B], c));
                  outp[1] = cadd(XC1[(t + 1) % NB], cscale(omega, cmul(cinv(D), csub(b1, yb))));
                }
              }
              outp += n;
            }
            ya = cmk(0.0, 0.0);
            yb = cmk(0.0, 0.0);
          }
          if (++rs == kTSR || k + 1 == nin) {  // stage consumed: refill its slot
            rs = 0;
            __syncwarp();
            if (lane == 0 && g + kTNS < nstages) issue(g + kTNS, s);
            ++g;
            st += kStage;
            if (++s == kTNS) {
              s = 0;
              st = sbase;
            }
          }
        }
      }
    }
  }
  if (MODE == OP_RESNORM) {  // every thread of the CTA reaches this reduction
    double2 total;
    if (grid_sum2(cmk(acc, 0.0), red.partials, red.counter, scratch, &total))
      *red.dst = red.raw ? total.x : sqrt(total.x) / red.scale;
  }
}

}  // namespace hd
