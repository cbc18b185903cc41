// Partially diagonalised exact solve of the 2D deflation matrix
//   E = E_M (x) E_S + E_S (x) E_M - k^2 E_M (x) E_M            (src/precond.cpp:95-104)
// E_S V = E_M V diag(lam), V^T E_M V = I (x direction, cuSOLVER sygvd at setup).
// With X the coarse vector as an n x n matrix (rows x, columns y), E vec(X) =
// vec(B) becomes, for every x mode m, the real banded system along y
//   (E_S + (lam_m - k^2) E_M) y_m = (V^T B)_m ,     X = V Y,
// so one application is: T = V^T B (GEMM), n independent banded solves along y
// with the LU factors (partial pivoting, host, at setup) of the n mode
// matrices, X = V T (GEMM).  Two GEMMs instead of the four of the full fast
// diagonalisation, and an exact direct method like the reference's SparseLU
// (its rounding is held to the exact-solver envelope, tests/golden/
// make_e_envelope.py).
//
// k_pfd_ysolve: one warp per group of kPG = 8 modes, one lane per mode running
// the re and im planes as two interleaved real recurrences.  Each lane runs the
// forward sweep (row interchanges + unit-L elimination, window of KL+1
// partially eliminated right-hand-side rows in registers), writing y in place,
// then the backward sweep (U with 2KL superdiagonals, window of the last 2KL
// x values in registers), writing x in place.  The mode tables and the
// right-hand-side rows stream through a kPD-deep ring of cp.async stages of kPR
// rows each: the recurrences are latency-bound chains (a few dependent FMAs
// per row), so the loads must run far ahead of them.
#pragma once

#include "device_common.cuh"

namespace hd {

constexpr int kPG = 8;   // modes per warp
constexpr int kPR = 8;   // rows per ring stage
constexpr int kPD = 16;  // ring stages

struct PfdArgs {
  double* T;         // np x 2n column-major: T[m + (iy + plane n) np]; in: V^T B, out: Y
  const double* F;   // forward tables [g][k][KL+1][kPG]: l_1..l_KL, pivot offset (as a double)
  const double* Bt;  // backward tables [g][k][2KL+1][kPG]: 1/u_kk, u_k,k+1 .. u_k,k+2KL
  int n;             // rows (y) and modes (x)
  int np;            // modes padded to a multiple of kPG (identity rows beyond n)
};

template <int KL>
__host__ __device__ constexpr size_t pfd_smem() {
  // the larger of the forward and backward stages, times the ring depth
  constexpr size_t fwd = static_cast<size_t>(kPR) * ((KL + 1) * kPG + 2 * kPG) * sizeof(double);
  constexpr size_t bwd = static_cast<size_t>(kPR) * ((2 * KL + 1) * kPG + 2 * kPG) * sizeof(double);
  return kPD * (fwd > bwd ? fwd : bwd);
}

__device__ __forceinline__ void pfd_cp16(void* s, const void* g) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(s));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g) : "memory");
}
__device__ __forceinline__ void pfd_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void pfd_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int KL>
__global__ void __launch_bounds__(32) k_pfd_ysolve(PfdArgs a) {
  constexpr int KU = 2 * KL;
  constexpr int FW = (KL + 1) * kPG;        // forward table doubles per row
  constexpr int BW = (KU + 1) * kPG;        // backward table doubles per row
  constexpr int SF = kPR * (FW + 2 * kPG);  // doubles per forward stage
  constexpr int SB = kPR * (BW + 2 * kPG);  // doubles per backward stage
  constexpr int SS = SF > SB ? SF : SB;     // slot stride
  extern __shared__ double pfd_sm[];
  const int lane = threadIdx.x;
  const int g = blockIdx.x;
  const int n = a.n, np = a.np;
  const int mm = lane & (kPG - 1);  // this lane's mode; it runs both planes (two independent chains)
  const bool active = lane < kPG;
  double* const Tg = a.T + static_cast<size_t>(g) * kPG;  // + (iy + plane n) np
  const size_t pstride = static_cast<size_t>(n) * np;     // plane offset in T
  const int nst = (n + kPR - 1) / kPR;

  // ---------------- forward: rows 0 .. n-1 ----------------
  const double* Fg = a.F + static_cast<size_t>(g) * n * FW;
  auto issue_f = [&](int s) {
    if (s < nst) {
      double* slot = pfd_sm + static_cast<size_t>(s % kPD) * SS;
      const int r0 = s * kPR, rows = min(kPR, n - r0);
      const int fch = rows * FW / 2;  // 16-byte chunks of the table rows
      for (int c = lane; c < fch; c += 32) pfd_cp16(slot + 2 * c, Fg + static_cast<size_t>(r0) * FW + 2 * c);
      const int tch = rows * 2 * (kPG / 2);  // per row: 2 planes x kPG doubles
      for (int c = lane; c < tch; c += 32) {
        const int r = c / kPG, rem = c % kPG, p = rem / (kPG / 2), q = rem % (kPG / 2);
        pfd_cp16(slot + kPR * FW + (r * 2 + p) * kPG + 2 * q,
                 Tg + static_cast<size_t>(r0 + r + p * n) * np + 2 * q);
      }
    }
    pfd_commit();
  };
  auto t_at = [&](int q, int p) -> double {  // right-hand side row q, plane p (0 past the end)
    if (q >= n) return 0.0;
    const double* slot = pfd_sm + static_cast<size_t>((q / kPR) % kPD) * SS;
    return slot[kPR * FW + ((q % kPR) * 2 + p) * kPG + mm];
  };
#pragma unroll 1
  for (int s = 0; s < kPD; ++s) issue_f(s);
  pfd_wait<kPD - 2>();
  __syncwarp();
  double w0[KL + 1], w1[KL + 1];  // window rows k .. k+KL of both planes
#pragma unroll
  for (int r = 0; r <= KL; ++r) {
    w0[r] = active ? t_at(r, 0) : 0.0;
    w1[r] = active ? t_at(r, 1) : 0.0;
  }
#pragma unroll 1
  for (int s = 0; s < nst; ++s) {
    const double* slot = pfd_sm + static_cast<size_t>(s % kPD) * SS;
    const int r0 = s * kPR;
    // the stage's coefficients and the refill rows into registers first, so the
    // recurrence below is a chain of register selects and FMAs only
    double lf[kPR][KL];
    int pv[kPR];
    double tn0[kPR], tn1[kPR];
#pragma unroll
    for (int rr = 0; rr < kPR; ++rr) {
      const double* fr = slot + rr * FW;
#pragma unroll
      for (int q = 0; q < KL; ++q) lf[rr][q] = fr[q * kPG + mm];
      pv[rr] = static_cast<int>(fr[KL * kPG + mm]);
      tn0[rr] = t_at(r0 + rr + KL + 1, 0);
      tn1[rr] = t_at(r0 + rr + KL + 1, 1);
    }
#pragma unroll
    for (int rr = 0; rr < kPR; ++rr) {
      const int k = r0 + rr;
      if (k < n && active) {
        const int p = pv[rr];
        // row interchange k <-> k + p inside the window
        double y0 = w0[0], y1 = w1[0];
#pragma unroll
        for (int r = 1; r <= KL; ++r)
          if (p == r) {
            y0 = w0[r];
            w0[r] = w0[0];
            y1 = w1[r];
            w1[r] = w1[0];
          }
#pragma unroll
        for (int r = 1; r <= KL; ++r) {
          w0[r] = fma(-lf[rr][r - 1], y0, w0[r]);
          w1[r] = fma(-lf[rr][r - 1], y1, w1[r]);
        }
        Tg[static_cast<size_t>(k) * np + mm] = y0;
        Tg[pstride + static_cast<size_t>(k) * np + mm] = y1;
#pragma unroll
        for (int r = 0; r < KL; ++r) {
          w0[r] = w0[r + 1];
          w1[r] = w1[r + 1];
        }
        w0[KL] = tn0[rr];
        w1[KL] = tn1[rr];
      }
    }
    __syncwarp();
    issue_f(s + kPD);
    pfd_wait<kPD - 2>();
    __syncwarp();
  }
  pfd_wait<0>();
  __threadfence();  // y visible to the backward sweep's cp.async (L2) reads
  __syncwarp();

  // ---------------- backward: rows n-1 .. 0 ----------------
  const double* Bg = a.Bt + static_cast<size_t>(g) * n * BW;
  auto lo_of = [&](int s) { return max(0, n - (s + 1) * kPR); };
  auto issue_b = [&](int s) {
    if (s < nst) {
      double* slot = pfd_sm + static_cast<size_t>(s % kPD) * SS;
      const int klo = lo_of(s), rows = n - s * kPR - klo;
      const int bch = rows * BW / 2;
      for (int c = lane; c < bch; c += 32) pfd_cp16(slot + 2 * c, Bg + static_cast<size_t>(klo) * BW + 2 * c);
      const int tch = rows * 2 * (kPG / 2);
      for (int c = lane; c < tch; c += 32) {
        const int r = c / kPG, rem = c % kPG, p = rem / (kPG / 2), q = rem % (kPG / 2);
        pfd_cp16(slot + kPR * BW + (r * 2 + p) * kPG + 2 * q,
                 Tg + static_cast<size_t>(klo + r + p * n) * np + 2 * q);
      }
    }
    pfd_commit();
  };
#pragma unroll 1
  for (int s = 0; s < kPD; ++s) issue_b(s);
  double xa[KU], xb[KU];  // x_{k+1} .. x_{k+KU} of both planes
#pragma unroll
  for (int d = 0; d < KU; ++d) xa[d] = xb[d] = 0.0;
#pragma unroll 1
  for (int s = 0; s < nst; ++s) {
    pfd_wait<kPD - 1>();
    __syncwarp();
    const double* slot = pfd_sm + static_cast<size_t>(s % kPD) * SS;
    const int klo = lo_of(s), khi = n - 1 - s * kPR;
#pragma unroll
    for (int rr = 0; rr < kPR; ++rr) {
      const int k = khi - rr;
      if (k >= klo && active) {
        const int r = k - klo;
        const double* br = slot + r * BW;
        double u[KU + 1];
#pragma unroll
        for (int d = 0; d <= KU; ++d) u[d] = br[d * kPG + mm];
        double acc0 = slot[kPR * BW + (r * 2) * kPG + mm];
        double acc1 = slot[kPR * BW + (r * 2 + 1) * kPG + mm];
        // the far taps first: only the last FMA waits for x_{k+1}
#pragma unroll
        for (int d = KU; d >= 1; --d) {
          acc0 = fma(-u[d], xa[d - 1], acc0);
          acc1 = fma(-u[d], xb[d - 1], acc1);
        }
        const double x0 = acc0 * u[0], x1 = acc1 * u[0];
        Tg[static_cast<size_t>(k) * np + mm] = x0;
        Tg[pstride + static_cast<size_t>(k) * np + mm] = x1;
#pragma unroll
        for (int d = KU - 1; d >= 1; --d) {
          xa[d] = xa[d - 1];
          xb[d] = xb[d - 1];
        }
        xa[0] = x0;
        xb[0] = x1;
      }
    }
    __syncwarp();
    issue_b(s + kPD);
  }
  pfd_wait<0>();
}

}  // namespace hd
