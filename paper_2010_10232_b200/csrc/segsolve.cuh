// Segmented (SPIKE-style) solve with a banded LU factorisation P A = L U
// (partial pivoting, L: KL sub-diagonals, U: KU = 2 KL super-diagonals) --
// the 1D exact solves (deflation E, C_ex, coarsest level) without the
// n-step sequential chain of the single-lane kernel.
//
// Both sweeps are linear recurrences with fixed coefficients:
//   forward  (LAPACK gbtrs order) on the window w = rows k..k+KL:
//            swap w_0 <-> w_p(k); y_k = w_0; w_q -= l(k+q, k) y_k; shift in b_{k+KL+1}
//   backward x_k = (y_k - sum_{d=1..KU} u(k, k+d) x_{k+d}) / u(k, k)
// The rows are cut into P segments of kSegL rows.  Every segment runs both
// sweeps locally from a zero boundary (the forward window starts from the raw
// rhs rows), in parallel; by linearity the true values differ from the local
// ones by h_k . Delta_i (forward: Delta_i = true window - raw rhs at the
// segment start) and h'_k . X_{i+1} (backward: X_{i+1} = the true x of the next
// KU rows).  h, h' and the window transfer matrices F_i are fixed and computed
// at setup; the boundary values follow from two short sequential scans over
// the segments:  Delta_{i+1} = D_i + F_i Delta_i,  X_i = X0_i + H'_i X_{i+1}.
// Arithmetic is that of the same factorisation; only the association of the
// sums changes (rounding-level differences).
//
// Layout: every per-row table is stored [row-in-segment r][field][segment i]
// (rows past n padded with the identity), so a warp of 32 segments reads one
// coalesced line per field and row; the scans stage their per-segment maps
// through shared memory in chunks.
#pragma once

#include "device_common.cuh"

namespace hd {

constexpr int kSegL = 64;   // rows per segment
// segments per staged scan chunk: <= 16, double buffer within 48 KB of static shared memory
__host__ __device__ constexpr int seg_chunk(int per) { return 49152 / (2 * per * 16) < 16 ? 49152 / (2 * per * 16) : 16; }

struct SegArgs {
  int n, P;
  const double2* L;      // [r][KL][P]  multipliers l(k+q, k)
  const int* pv;         // [r][P]      pivot offset p(k) - k
  const double2* hf;     // [r][KL+1][P] forward influence rows
  const double2* U;      // [r][KU][P]  u(k, k+d), d = 1..KU
  const double2* Ui;     // [r][P]      1 / u(k, k)
  const double2* hb;     // [r][KU][P]  backward influence rows
  const double2* Ff;     // [P][KL+1][KL+1] forward window transfer (row-major)
  const double2* Hb;     // [P][KU][KU]     backward boundary map H'_i (rows: first KU rows of segment i)
  double2* y;            // [r][P]
  double2* x0;           // [r][P]
  double2* D;            // [P][KL+1] window increments
  double2* Dl;           // [P][KL+1] Delta_i
  double2* X0;           // [P][KU]   local x of the first KU rows
  double2* Xb;           // [P+1][KU] true x of the first KU rows
  double2* AgF;          // [kScanWarps][(KL+1)^2] matrix parts of the forward scan's group maps (setup)
  double2* AgB;          // [kScanWarps][KU^2]     ... of the backward scan's
};

__device__ __forceinline__ double2 seg_rhs(const double2* b, const double* bp, int n, int k) {
  if (k >= n) return cmk(0.0, 0.0);
  return bp ? cmk(bp[k], bp[k + n]) : b[k];
}

// Rows of per-row tables in flight per segment thread (cp.async ring in shared
// memory; each lane copies and later reads only its own segment's entries).
constexpr int kSegDepth = 16;
template <int KL>
__host__ __device__ constexpr size_t seg_fwd_smem() {
  return (size_t)kSegDepth * 32 * ((KL + 1) * sizeof(double2) + sizeof(int));
}
template <int KL>
__host__ __device__ constexpr size_t seg_bwd_smem() {
  return (size_t)kSegDepth * 32 * (3 * KL + 3) * sizeof(double2);
}

// local forward sweep of every segment (thread per segment, warp = 32
// segments).  The per-row tables (pivot, multipliers, the rhs row shifted in)
// stream through a kSegDepth-row cp.async ring, so the dependent elimination
// chain never waits on a global load.
template <int KL>
__global__ void __launch_bounds__(32) k_seg_fwd(SegArgs a, const double2* __restrict__ b,
                                                const double* __restrict__ bp) {
  extern __shared__ __align__(16) double2 sring[];
  double2(*rl)[KL + 1][32] = reinterpret_cast<double2(*)[KL + 1][32]>(sring);  // [slot][L_0..L_{KL-1}, b][lane]
  int(*rp)[32] = reinterpret_cast<int(*)[32]>(sring + (size_t)kSegDepth * (KL + 1) * 32);
  const int lane = threadIdx.x;
  const int i = blockIdx.x * 32 + lane;
  const bool valid = i < a.P;
  const int P = a.P, s = i * kSegL, n = a.n;
  // row r's tables: pv, L[r][0..KL-1], rhs row s + r + KL + 1
  auto issue = [&](int r) {
    if (r < kSegL) {
      const int sl = r % kSegDepth;
      cp_async4(&rp[sl][lane], a.pv + (size_t)r * P + (valid ? i : 0), valid);
#pragma unroll
      for (int q = 0; q < KL; ++q) cp_async16(&rl[sl][q][lane], a.L + ((size_t)r * KL + q) * P + (valid ? i : 0), valid);
      const int k = s + r + KL + 1;
      const bool kv = valid && k < n;
      if (bp) {
        cp_async8(&rl[sl][KL][lane].x, bp + (kv ? k : 0), kv);
        cp_async8(&rl[sl][KL][lane].y, bp + (kv ? k + n : 0), kv);
      } else {
        cp_async16(&rl[sl][KL][lane], b + (kv ? k : 0), kv);
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int t = 0; t < kSegDepth - 1; ++t) issue(t);
  double2 w[KL + 1];
#pragma unroll
  for (int q = 0; q <= KL; ++q) w[q] = valid ? seg_rhs(b, bp, n, s + q) : cmk(0.0, 0.0);
  for (int r = 0; r < kSegL; ++r) {
    cp_async_wait<kSegDepth - 2>();
    issue(r + kSegDepth - 1);
    const int sl = r % kSegDepth;
    const int pc = rp[sl][lane];
    double2 yk = w[0];
#pragma unroll
    for (int q = 1; q <= KL; ++q) yk = pc == q ? w[q] : yk;
#pragma unroll
    for (int q = 1; q <= KL; ++q) {
      const double2 wq = pc == q ? w[0] : w[q];
      w[q] = csub(wq, cmul(rl[sl][q - 1][lane], yk));
    }
    if (valid) a.y[(size_t)r * P + i] = yk;
#pragma unroll
    for (int q = 0; q < KL; ++q) w[q] = w[q + 1];
    w[KL] = rl[sl][KL][lane];
  }
  cp_async_wait<0>();
  if (!valid) return;
  // D_i = end window - raw rhs rows e..e+KL
#pragma unroll
  for (int q = 0; q <= KL; ++q) a.D[(size_t)i * (KL + 1) + q] = csub(w[q], seg_rhs(b, bp, n, s + kSegL + q));
}

// Delta_0 = 0, Delta_{i+1} = D_i + F_i Delta_i  (one warp; lane q owns component q;
// the maps are staged kSegC segments at a time, double-buffered)
template <int KL>
__global__ void __launch_bounds__(32) k_seg_scan_fwd(SegArgs a) {
  constexpr int W = KL + 1, PER = W * W + W;  // F_i then D_i
  constexpr int kSegC = seg_chunk(PER);
  __shared__ __align__(16) double2 buf[2][kSegC * PER];
  const int lane = threadIdx.x;
  const int nch = (a.P + kSegC - 1) / kSegC;
  auto stage = [&](int c) {
    if (c < nch) {
      const int i0 = c * kSegC, ni = min(kSegC, a.P - i0);
      double2* d = buf[c & 1];
      for (int e = lane; e < ni * W * W; e += 32) cp_async16(d + e, a.Ff + (size_t)i0 * W * W + e, true);
      for (int e = lane; e < ni * W; e += 32) cp_async16(d + kSegC * W * W + e, a.D + (size_t)i0 * W + e, true);
    }
    cp_async_commit();
  };
  stage(0);
  double2 dl = cmk(0.0, 0.0);
  for (int c = 0; c < nch; ++c) {
    stage(c + 1);
    cp_async_wait<1>();
    __syncwarp();
    const double2* F = buf[c & 1];
    const double2* Dd = F + kSegC * W * W;
    const int ni = min(kSegC, a.P - c * kSegC);
    for (int t = 0; t < ni; ++t) {
      const int i = c * kSegC + t;
      if (lane < W) a.Dl[(size_t)i * W + lane] = dl;
      double2 nx = lane < W ? Dd[t * W + lane] : cmk(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < W; ++r) {
        const double2 dr = cmk(__shfl_sync(0xffffffffu, dl.x, r), __shfl_sync(0xffffffffu, dl.y, r));
        if (lane < W) nx = cfma(F[(t * W + lane) * W + r], dr, nx);
      }
      dl = nx;
    }
    __syncwarp();
  }
  cp_async_wait<0>();
}

// forward correction y_k += h_k . Delta_i, then the local backward sweep; the
// per-row tables (y, h, U, 1/u) stream through a kSegDepth-row cp.async ring
// as in k_seg_fwd
template <int KL>
__global__ void __launch_bounds__(32) k_seg_bwd(SegArgs a) {
  constexpr int KU = 2 * KL, NF = KL + KU + 3;  // y, hf[KL+1], U[KU], 1/u
  extern __shared__ __align__(16) double2 sring[];
  double2(*rg)[NF][32] = reinterpret_cast<double2(*)[NF][32]>(sring);
  const int lane = threadIdx.x;
  const int i = blockIdx.x * 32 + lane;
  const bool valid = i < a.P;
  const int P = a.P, ii = valid ? i : 0;
  auto issue = [&](int t) {  // t-th row from the end: r = kSegL - 1 - t
    if (t < kSegL) {
      const int r = kSegL - 1 - t, sl = t % kSegDepth;
      cp_async16(&rg[sl][0][lane], a.y + (size_t)r * P + ii, valid);
#pragma unroll
      for (int q = 0; q <= KL; ++q) cp_async16(&rg[sl][1 + q][lane], a.hf + ((size_t)r * (KL + 1) + q) * P + ii, valid);
#pragma unroll
      for (int d = 0; d < KU; ++d) cp_async16(&rg[sl][KL + 2 + d][lane], a.U + ((size_t)r * KU + d) * P + ii, valid);
      cp_async16(&rg[sl][KL + KU + 2][lane], a.Ui + (size_t)r * P + ii, valid);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int t = 0; t < kSegDepth - 1; ++t) issue(t);
  double2 dl[KL + 1];
#pragma unroll
  for (int q = 0; q <= KL; ++q) dl[q] = valid ? a.Dl[(size_t)i * (KL + 1) + q] : cmk(0.0, 0.0);
  double2 xw[KU];  // x_{k+1} .. x_{k+KU}
#pragma unroll
  for (int d = 0; d < KU; ++d) xw[d] = cmk(0.0, 0.0);
  for (int t = 0; t < kSegL; ++t) {
    const int r = kSegL - 1 - t, sl = t % kSegDepth;
    cp_async_wait<kSegDepth - 2>();
    issue(t + kSegDepth - 1);
    double2 sacc = rg[sl][0][lane];
#pragma unroll
    for (int q = 0; q <= KL; ++q) sacc = cfma(rg[sl][1 + q][lane], dl[q], sacc);
#pragma unroll
    for (int d = KU; d >= 1; --d) sacc = csub(sacc, cmul(rg[sl][KL + 1 + d][lane], xw[d - 1]));
    const double2 xk = cmul(sacc, rg[sl][KL + KU + 2][lane]);
#pragma unroll
    for (int d = KU - 1; d >= 1; --d) xw[d] = xw[d - 1];
    xw[0] = xk;
    if (valid) a.x0[(size_t)r * P + i] = xk;
  }
  cp_async_wait<0>();
  if (!valid) return;
#pragma unroll
  for (int d = 0; d < KU; ++d) a.X0[(size_t)i * KU + d] = xw[d];  // xw[d] = x_{s+d}
}

// X_P = 0, X_i = X0_i + H'_i X_{i+1}  (one warp, lane d owns component d)
template <int KL>
__global__ void __launch_bounds__(32) k_seg_scan_bwd(SegArgs a) {
  constexpr int KU = 2 * KL, PER = KU * KU + KU;  // H'_i then X0_i
  constexpr int kSegC = seg_chunk(PER);
  __shared__ __align__(16) double2 buf[2][kSegC * PER];
  const int lane = threadIdx.x;
  const int nch = (a.P + kSegC - 1) / kSegC;
  // chunks are staged from the last segment backwards: chunk c covers segments
  // [P - (c+1) kSegC, P - c kSegC)
  auto stage = [&](int c) {
    if (c < nch) {
      const int i1 = a.P - c * kSegC, i0 = max(0, i1 - kSegC), ni = i1 - i0;
      double2* d = buf[c & 1];
      for (int e = lane; e < ni * KU * KU; e += 32) cp_async16(d + e, a.Hb + (size_t)i0 * KU * KU + e, true);
      for (int e = lane; e < ni * KU; e += 32) cp_async16(d + kSegC * KU * KU + e, a.X0 + (size_t)i0 * KU + e, true);
    }
    cp_async_commit();
  };
  stage(0);
  double2 xn = cmk(0.0, 0.0);
  if (lane < KU) a.Xb[(size_t)a.P * KU + lane] = xn;
  for (int c = 0; c < nch; ++c) {
    stage(c + 1);
    cp_async_wait<1>();
    __syncwarp();
    const double2* H = buf[c & 1];
    const double2* X0 = H + kSegC * KU * KU;
    const int i1 = a.P - c * kSegC, i0 = max(0, i1 - kSegC);
    for (int i = i1 - 1; i >= i0; --i) {
      const int t = i - i0;
      double2 v = lane < KU ? X0[t * KU + lane] : cmk(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < KU; ++r) {
        const double2 xr = cmk(__shfl_sync(0xffffffffu, xn.x, r), __shfl_sync(0xffffffffu, xn.y, r));
        if (lane < KU) v = cfma(H[(t * KU + lane) * KU + r], xr, v);
      }
      xn = v;
      if (lane < KU) a.Xb[(size_t)i * KU + lane] = xn;
    }
    __syncwarp();
  }
  cp_async_wait<0>();
}

// ---- two-level scan over the segments (replaces the P-step sequential scans) ----
// The boundary recurrences are affine maps applied in step order t = 0..P-1:
//   forward  (BWD = 0): map i = t,       s <- D_i + F_i s,  out[i] = s before the map (Delta_i)
//   backward (BWD = 1): map i = P-1-t,   s <- X0_i + H'_i s, out[i] = s after the map (X_i), out[P] = 0
// Phase 1: warp g composes the maps of its group of m consecutive steps into one
// affine map (A_g, b_g).  Phase 2: one warp runs the G group maps in order and
// records every group's incoming state.  Phase 3: warp g replays its group's m
// maps from that state, in the sequential kernels' arithmetic, writing the
// outputs.  3 x m + G dependent steps instead of P; the incoming states differ
// from the sequential scan's only by the rounding of the compositions.
constexpr int kScanWarps = 16, kScanRing = 4;

template <int DM>
__host__ __device__ constexpr size_t seg_scan2_smem() {
  return sizeof(double2) * ((size_t)kScanWarps * kScanRing * (DM * DM + DM) +  // map ring per warp
                            (size_t)kScanWarps * 2 * (DM * DM + DM) +           // A, b double-buffered per warp
                            (size_t)kScanWarps * (DM * DM + DM) +               // group maps (A_g, b_g)
                            (size_t)kScanWarps * DM);                           // group incoming states
}

// AG, PRE: the matrix part A_g of every group map depends only on the factorisation, not on the right-hand
// side.  PRE = 1 (once at setup, ct = zeros): phase 1 composes (A, b) as matrix products and stores A_g to AG.
// PRE = 0 (every solve): phase 1 runs only the vector recurrence b <- M b + c (the same arithmetic as the b part
// of the composition, so the same bits) and reads A_g from AG: DM-fold less work in the kernel's longest phase.
template <int DM, int BWD, int PRE = 0>
__global__ void __launch_bounds__(kScanWarps * 32) k_seg_scan2(const double2* __restrict__ Mt,
                                                               const double2* __restrict__ ct, double2* __restrict__ out,
                                                               int P, double2* __restrict__ AG) {
  constexpr int DD = DM * DM, PER = DD + DM;
  extern __shared__ __align__(16) double2 ssm[];
  const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
  double2* ring = ssm + (size_t)g * kScanRing * PER;
  double2* ab = ssm + (size_t)kScanWarps * kScanRing * PER + (size_t)g * 2 * PER;  // [2][A | b]
  double2* agg = ssm + (size_t)kScanWarps * (kScanRing + 2) * PER;                // [G][A_g | b_g]
  double2* sin = agg + (size_t)kScanWarps * PER;                                   // [G][DM]
  const int m = (P + kScanWarps - 1) / kScanWarps;
  const int t0 = min(P, g * m), t1 = min(P, t0 + m);
  auto mapidx = [&](int t) { return BWD ? P - 1 - t : t; };
  auto issue = [&](int t) {
    if (t < t1) {
      const int i = mapidx(t);
      double2* d = ring + (size_t)((t - t0) % kScanRing) * PER;
      for (int e = lane; e < DD; e += 32) cp_async16(d + e, Mt + (size_t)i * DD + e, true);
      for (int e = lane; e < DM; e += 32) cp_async16(d + DD + e, ct + (size_t)i * DM + e, true);
    }
    cp_async_commit();
  };
  // phase 1: (A, b) <- (M A, M b + c) over the group's steps
  for (int t = t0; t < t0 + kScanRing - 1; ++t) issue(t);
  if (PRE) {
    for (int e = lane; e < PER; e += 32) ab[e] = cmk(e < DD && e / DM == e % DM ? 1.0 : 0.0, 0.0);
    __syncwarp();
    int cur = 0;
    for (int t = t0; t < t1; ++t) {
      cp_async_wait<kScanRing - 2>();
      __syncwarp();
      issue(t + kScanRing - 1);
      const double2* M = ring + (size_t)((t - t0) % kScanRing) * PER;
      const double2* A = ab + cur * PER;
      double2* An = ab + (cur ^ 1) * PER;
      for (int e = lane; e < PER; e += 32) {
        double2 v;
        if (e < DD) {  // (M A)(r, c)
          const int r = e / DM, c = e % DM;
          v = cmk(0.0, 0.0);
#pragma unroll
          for (int k = 0; k < DM; ++k) v = cfma(M[r * DM + k], A[k * DM + c], v);
        } else {  // (M b + c)(r)
          const int r = e - DD;
          v = M[DD + r];
#pragma unroll
          for (int k = 0; k < DM; ++k) v = cfma(M[r * DM + k], A[DD + k], v);
        }
        An[e] = v;
      }
      cur ^= 1;
      __syncwarp();
    }
    cp_async_wait<0>();
    for (int e = lane; e < PER; e += 32) agg[(size_t)g * PER + e] = ab[cur * PER + e];
    for (int e = lane; e < DD; e += 32) AG[(size_t)g * DD + e] = ab[cur * PER + e];
  } else {
    // b <- M b + c, lane r owns component r (M's vector part is c); A_g comes from the setup pass
    double2 bv = cmk(0.0, 0.0);
    for (int t = t0; t < t1; ++t) {
      cp_async_wait<kScanRing - 2>();
      __syncwarp();
      issue(t + kScanRing - 1);
      const double2* M = ring + (size_t)((t - t0) % kScanRing) * PER;
      double2 nx = lane < DM ? M[DD + lane] : cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < DM; ++k) {
        const double2 bk = cmk(__shfl_sync(0xffffffffu, bv.x, k), __shfl_sync(0xffffffffu, bv.y, k));
        if (lane < DM) nx = cfma(M[lane * DM + k], bk, nx);
      }
      bv = nx;
      __syncwarp();
    }
    cp_async_wait<0>();
    for (int e = lane; e < DD; e += 32) agg[(size_t)g * PER + e] = __ldg(AG + (size_t)g * DD + e);
    if (lane < DM) agg[(size_t)g * PER + DD + lane] = bv;
  }
  __syncthreads();
  if (PRE) return;  // the setup pass only wanted the A_g
  // phase 2: group maps in order, lane q owns component q
  if (g == 0) {
    double2 sv = cmk(0.0, 0.0);
    for (int gg = 0; gg < kScanWarps; ++gg) {
      if (lane < DM) sin[gg * DM + lane] = sv;
      const double2* Ag = agg + (size_t)gg * PER;
      double2 nx = lane < DM ? Ag[DD + lane] : cmk(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < DM; ++r) {
        const double2 sr = cmk(__shfl_sync(0xffffffffu, sv.x, r), __shfl_sync(0xffffffffu, sv.y, r));
        if (lane < DM) nx = cfma(Ag[lane * DM + r], sr, nx);
      }
      sv = nx;
    }
    if (BWD && lane < DM) out[(size_t)P * DM + lane] = cmk(0.0, 0.0);
  }
  __syncthreads();
  // phase 3: replay the group's steps from its incoming state
  for (int t = t0; t < t0 + kScanRing - 1; ++t) issue(t);
  double2 sv = lane < DM ? sin[g * DM + lane] : cmk(0.0, 0.0);
  for (int t = t0; t < t1; ++t) {
    cp_async_wait<kScanRing - 2>();
    __syncwarp();
    issue(t + kScanRing - 1);
    const int i = mapidx(t);
    if (!BWD && lane < DM) out[(size_t)i * DM + lane] = sv;
    const double2* M = ring + (size_t)((t - t0) % kScanRing) * PER;
    double2 nx = lane < DM ? M[DD + lane] : cmk(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < DM; ++r) {
      const double2 sr = cmk(__shfl_sync(0xffffffffu, sv.x, r), __shfl_sync(0xffffffffu, sv.y, r));
      if (lane < DM) nx = cfma(M[lane * DM + r], sr, nx);
    }
    sv = nx;
    if (BWD && lane < DM) out[(size_t)i * DM + lane] = sv;
    __syncwarp();
  }
  cp_async_wait<0>();
}

// x_k = x0_k + h'_k . X_{i+1}  (thread per row), output interleaved or planar
template <int KL>
__global__ void k_seg_out(SegArgs a, double2* __restrict__ x, double* __restrict__ xp) {
  constexpr int KU = 2 * KL;
  const int P = a.P;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.n; k += gridDim.x * blockDim.x) {
    const int i = k / kSegL, r = k % kSegL;
    double2 v = a.x0[(size_t)r * P + i];
#pragma unroll
    for (int d = 0; d < KU; ++d) v = cfma(a.hb[((size_t)r * KU + d) * P + i], a.Xb[(size_t)(i + 1) * KU + d], v);
    if (xp) {
      xp[k] = v.x;
      xp[k + a.n] = v.y;
    } else {
      x[k] = v;
    }
  }
}

}  // namespace hd
