// One-reduction Arnoldi for GMRES: modified Gram-Schmidt in its inverse
// compact-WY form (h = (I + L)^-1 V^H w, L = strictly lower part of V^H V),
// which is algebraically the reference's MGS (src/linalg.cpp:42-45):
//   h_i = v_i^H (w - sum_{l<i} h_l v_l) = s_i - sum_{l<i} (v_i^H v_l) h_l .
// Two streaming passes per iteration replace the j+2 sequential reductions:
//
//   pass 1 (k_lsa_dots):   s_i = u_i^H w (i <= j), G_jl = u_j^H u_l (l < j),
//                          and, lagged by one iteration, the iterate
//                          x_{j-1} = x0 + sum_{i<j} y_i v_i (src/linalg.cpp:78-80)
//                          -> last CTA: (I+L) h = s, H(:, j) = h
//   pass 2 (k_lsa_update): u_{j+1} = w - sum_i h_i v_i, ||u_{j+1}||
//                          -> last CTA: hnew, Givens + back substitution (:46-77)
//
// The basis is stored unnormalised (u_i) with scales sigma_i = 1/||u_i||
// (v_i = sigma_i u_i), so no separate normalisation pass exists; the composed
// operator is linear, so op(v_j) = sigma_j op(u_j).  Reductions are
// deterministic: per-warp shuffle trees, per-CTA fixed-order sums, and the
// last CTA to finish sums the per-CTA partials in index order.
#pragma once

#include "device_common.cuh"

namespace hd {

constexpr int kLsaBD = 256;  // threads per CTA
constexpr int kLsaTE = 4;    // elements per thread per tile
constexpr int kLsaMaxJ = 128;

struct LsaArgs {
  const double2* U;   // basis u_0..u_maxit, stride N
  double2* Uw;        // == U (u_{j+1} written)
  const double2* w;   // raw op(u_j)
  const double2* x0;
  double2* x;         // lagged iterate out
  size_t N;
  int j;              // iteration index
  int mode;           // pass 1: 0 = dots + iterate, 1 = iterate only;  pass 2: unused
  double* sig;        // sigma_i
  double2* L;         // lower Gram, row-major ldl (L[i*ldl + l], l < i)
  int ldl;
  double2* H;         // column-major ldh
  int ldh;
  double2* g;
  double2* cs;
  double2* sn;
  double2* ch;        // c_i = h_i sigma_i (pass 2 coefficients)
  double2* cx;        // c'_i = y_i sigma_i (iterate coefficients, from the previous pass 2)
  double* hnew_out;
  double2* partials;  // gridDim.x * (2 kLsaMaxJ + 2)
  unsigned* counter;  // last-block ticket, zero between launches
  const int* done;    // early exit (speculative graph iterations); may be null
  const int* dj;      // device-side iteration index (graph mode); overrides j when set
};

__device__ __forceinline__ double2 lsa_warp_sum(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, o);
    v.y += __shfl_down_sync(0xffffffffu, v.y, o);
  }
  return v;  // valid in lane 0
}

// last CTA to arrive returns true (after a fence); counter reset by it
__device__ __forceinline__ bool lsa_last_block(unsigned* counter) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// Sum slot q of the per-CTA partials (fixed order) -- one warp per slot.
__device__ __forceinline__ double2 lsa_collect(const double2* partials, int nslot, int q) {
  double2 s = cmk(0.0, 0.0);
  const int lane = threadIdx.x & 31;
  for (unsigned b = lane; b < gridDim.x; b += 32) s = cadd(s, __ldcg(&partials[(size_t)b * nslot + q]));
  s = lsa_warp_sum(s);
  return cmk(__shfl_sync(0xffffffffu, s.x, 0), __shfl_sync(0xffffffffu, s.y, 0));
}

// ---------------------------------------------------------------------------
// pass 1: dots against w and u_j, lagged iterate
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kLsaBD, 2) k_lsa_dots(LsaArgs a) {
  constexpr int NW = kLsaBD / 32;
  __shared__ double2 acc[NW][2 * kLsaMaxJ + 2];  // per-warp partials of s_i and G_jl
  __shared__ double2 sh_cx[kLsaMaxJ];
  __shared__ double2 sh_s[kLsaMaxJ + 1];
  __shared__ double2 sh_lj[kLsaMaxJ];
  if (a.done && *((volatile const int*)a.done)) return;
  const int j = a.dj ? *a.dj : a.j;
  const bool dots = a.mode == 0;
  const bool iter = j >= 1 || a.mode == 1;     // x_{j-1} (mode 1: x_j, iterate-only)
  const int mi = a.mode == 1 ? j + 1 : j;      // iterate terms
  const int nd = dots ? j + 1 : 0;             // vectors entering the dots
  const int nv = max(nd, iter ? mi : 0);       // vectors streamed
  const int nslot = 2 * kLsaMaxJ + 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = threadIdx.x; q < NW * nslot; q += kLsaBD) (&acc[0][0])[q] = cmk(0.0, 0.0);
  for (int q = threadIdx.x; q < mi; q += kLsaBD) sh_cx[q] = a.cx[q];
  __syncthreads();
  const size_t N = a.N;
  const size_t tile = (size_t)kLsaBD * kLsaTE;
  const double2* uj = a.U + (size_t)j * N;
  for (size_t t0 = (size_t)blockIdx.x * tile; t0 < N; t0 += (size_t)gridDim.x * tile) {
    double2 wv[kLsaTE], ujv[kLsaTE], xv[kLsaTE];
#pragma unroll
    for (int u = 0; u < kLsaTE; ++u) {
      const size_t e = t0 + (size_t)u * kLsaBD + threadIdx.x;
      const bool ok = e < N;
      wv[u] = (dots && ok) ? ld_stream(a.w + e) : cmk(0.0, 0.0);
      ujv[u] = (dots && ok && j > 0) ? uj[e] : cmk(0.0, 0.0);
      xv[u] = (iter && ok) ? ld_stream(a.x0 + e) : cmk(0.0, 0.0);
    }
    // software pipeline: the loads of vector i+1 are in flight while vector i
    // is reduced (8 outstanding 16-B loads per thread)
    double2 vc[kLsaTE], vnx[kLsaTE];
    auto load_vec = [&](int i, double2* dst) {
      const double2* ui = a.U + (size_t)i * N;
#pragma unroll
      for (int u = 0; u < kLsaTE; ++u) {
        const size_t e = t0 + (size_t)u * kLsaBD + threadIdx.x;
        dst[u] = (i < nv && e < N) ? __ldg(ui + e) : cmk(0.0, 0.0);
      }
    };
    load_vec(0, vc);
    for (int i = 0; i < nv; ++i) {
      load_vec(i + 1, vnx);
      if (i < nd) {
        double2 s = cmk(0.0, 0.0), gl = cmk(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < kLsaTE; ++u) {
          s = cadd(s, cconjmul(vc[u], wv[u]));
          gl = cadd(gl, cconjmul(ujv[u], vc[u]));
        }
        s = lsa_warp_sum(s);
        if (i < j) gl = lsa_warp_sum(gl);
        if (lane == 0) {
          acc[warp][i] = cadd(acc[warp][i], s);
          if (i < j) acc[warp][kLsaMaxJ + 1 + i] = cadd(acc[warp][kLsaMaxJ + 1 + i], gl);
        }
      }
      if (iter && i < mi) {
        const double2 c = sh_cx[i];
#pragma unroll
        for (int u = 0; u < kLsaTE; ++u) xv[u] = cfma(c, vc[u], xv[u]);
      }
#pragma unroll
      for (int u = 0; u < kLsaTE; ++u) vc[u] = vnx[u];
    }
    if (iter) {
#pragma unroll
      for (int u = 0; u < kLsaTE; ++u) {
        const size_t e = t0 + (size_t)u * kLsaBD + threadIdx.x;
        if (e < N) a.x[e] = xv[u];
      }
    }
  }
  if (!dots) return;
  __syncthreads();
  // CTA partials: fixed-order sum over warps
  for (int q = threadIdx.x; q < nslot; q += kLsaBD) {
    const bool used = q < nd || (q >= kLsaMaxJ + 1 && q < kLsaMaxJ + 1 + j);
    if (!used) continue;
    double2 s = cmk(0.0, 0.0);
    for (int wv2 = 0; wv2 < NW; ++wv2) s = cadd(s, acc[wv2][q]);
    a.partials[(size_t)blockIdx.x * nslot + q] = s;
  }
  if (!lsa_last_block(a.counter)) return;
  // ---- last CTA: totals, Gram row j, triangular solve (I + L) h = s --------
  const double sj = a.sig[j];
  for (int q = warp; q < nd; q += NW) {
    const double2 s = lsa_collect(a.partials, nslot, q);
    if (lane == 0) sh_s[q] = cscale(a.sig[q] * sj, s);
  }
  for (int q = warp; q < j; q += NW) {
    const double2 gsum = lsa_collect(a.partials, nslot, kLsaMaxJ + 1 + q);
    if (lane == 0) {
      const double2 lq = cscale(sj * a.sig[q], gsum);  // v_j^H v_q
      a.L[(size_t)j * a.ldl + q] = lq;
      sh_lj[q] = lq;
    }
  }
  __syncthreads();
  __threadfence_block();
  // h_i = s_i - sum_{l<i} L_il h_l  (L_il = v_i^H v_l), one warp,
  // sequential in i, parallel over l with a fixed-order reduction
  if (warp == 0) {
    double2* Hj = a.H + (size_t)j * a.ldh;
    double2* hs = &acc[0][0];  // reuse: h_0..h_j
    for (int i = 0; i <= j; ++i) {
      double2 t = cmk(0.0, 0.0);
      for (int l = lane; l < i; l += 32)
        t = cadd(t, cmul(i == j ? sh_lj[l] : __ldcg(&a.L[(size_t)i * a.ldl + l]), hs[l]));
      t = lsa_warp_sum(t);
      if (lane == 0) {
        const double2 h = csub(sh_s[i], t);
        hs[i] = h;
        Hj[i] = h;
        a.ch[i] = cscale(a.sig[i], h);
      }
      __syncwarp();
    }
  }
  if (threadIdx.x == 0) *a.counter = 0u;
}

// ---------------------------------------------------------------------------
// pass 2: u_{j+1} = sigma_j w - sum_i c_i u_i,  hnew = ||u_{j+1}||, Givens
// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 lsa_cdiv(double2 a, double2 b) { return cmul(a, cinv(b)); }

__global__ void __launch_bounds__(kLsaBD) k_lsa_update(LsaArgs a) {
  constexpr int NW = kLsaBD / 32;
  __shared__ double2 sh_c[kLsaMaxJ + 1];
  __shared__ double red[NW];
  if (a.done && *((volatile const int*)a.done)) return;
  const int j = a.dj ? *a.dj : a.j;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = threadIdx.x; q <= j; q += kLsaBD) sh_c[q] = __ldcg(&a.ch[q]);
  __syncthreads();
  const double sj = a.sig[j];
  const size_t N = a.N;
  const size_t tile = (size_t)kLsaBD * kLsaTE;
  double2* un = a.Uw + (size_t)(j + 1) * N;
  double nrm = 0.0;
  for (size_t t0 = (size_t)blockIdx.x * tile; t0 < N; t0 += (size_t)gridDim.x * tile) {
    double2 wv[kLsaTE];
#pragma unroll
    for (int u = 0; u < kLsaTE; ++u) {
      const size_t e = t0 + (size_t)u * kLsaBD + threadIdx.x;
      wv[u] = e < N ? cscale(sj, ld_stream(a.w + e)) : cmk(0.0, 0.0);
    }
    // two vectors per step: 8 outstanding 16-B loads per thread
    for (int i = 0; i <= j; i += 2) {
      const bool two = i + 1 <= j;
      const double2* u0 = a.U + (size_t)i * N;
      const double2* u1 = a.U + (size_t)(i + 1) * N;
      double2 v0[kLsaTE], v1[kLsaTE];
#pragma unroll
      for (int u = 0; u < kLsaTE; ++u) {
        const size_t e = t0 + (size_t)u * kLsaBD + threadIdx.x;
        v0[u] = e < N ? __ldg(u0 + e) : cmk(0.0, 0.0);
        v1[u] = (two && e < N) ? __ldg(u1 + e) : cmk(0.0, 0.0);
      }
      const double2 c0 = sh_c[i], c1 = two ? sh_c[i + 1] : cmk(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < kLsaTE; ++u) {
        wv[u] = csub(wv[u], cmul(c0, v0[u]));
        if (two) wv[u] = csub(wv[u], cmul(c1, v1[u]));
      }
    }
#pragma unroll
    for (int u = 0; u < kLsaTE; ++u) {
      const size_t e = t0 + (size_t)u * kLsaBD + threadIdx.x;
      if (e < N) {
        un[e] = wv[u];
        nrm += cnorm2(wv[u]);
      }
    }
  }
  // CTA partial of ||u_{j+1}||^2
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nrm += __shfl_down_sync(0xffffffffu, nrm, o);
  if (lane == 0) red[warp] = nrm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < NW; ++q) s += red[q];
    a.partials[blockIdx.x] = cmk(s, 0.0);
  }
}

// ---------------------------------------------------------------------------
// pass 2 tail (one CTA): hnew from the per-CTA partials of k_lsa_update,
// sigma_{j+1}, Givens of column j, back substitution, iterate coefficients.
// nparts = gridDim.x of the update pass.  Dynamic smem: packed R + work.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kLsaBD) k_lsa_givens(LsaArgs a, int nparts) {
  extern __shared__ __align__(16) double2 sm[];
  __shared__ double s_hnew;
  if (a.done && *((volatile const int*)a.done)) return;
  const int j = a.dj ? *a.dj : a.j;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    double s = 0.0;
    for (int b = lane; b < nparts; b += 32) s += __ldcg(&a.partials[b]).x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) s_hnew = sqrt(s);
  }
  const int m = j + 1;
  double2* col = a.H + (size_t)j * a.ldh;
  double2* R = sm;                           // packed upper triangle, column c at c(c+1)/2
  double2* s = R + (size_t)m * (m + 1) / 2;  // g
  double2* cl = s + m + 1;
  double2* cc = cl + j + 2;
  double2* ss = cc + j + 1;
  for (int r = threadIdx.x; r <= j; r += blockDim.x) cl[r] = __ldcg(&col[r]);
  for (int r = threadIdx.x; r < j; r += blockDim.x) {
    cc[r] = a.cs[r];
    ss[r] = a.sn[r];
  }
  const int npk = j * (j + 1) / 2;  // rotated columns 0..j-1, one round of loads
  for (int q = threadIdx.x; q < npk; q += blockDim.x) {
    int c = static_cast<int>((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
    while ((c + 1) * (c + 2) / 2 <= q) ++c;
    while (c * (c + 1) / 2 > q) --c;
    const int r = q - c * (c + 1) / 2;
    R[q] = a.H[(size_t)c * a.ldh + r];
  }
  for (int r = threadIdx.x; r <= j; r += blockDim.x) s[r] = a.g[r];
  __syncthreads();
  const double hnew = s_hnew;
  if (threadIdx.x == 0) {
    cl[j + 1] = cmk(hnew, 0.0);
    *a.hnew_out = hnew;
    a.sig[j + 1] = hnew > 0.0 ? 1.0 / hnew : 0.0;
    for (int i = 0; i < j; ++i) {
      const double2 p = cl[i], q = cl[i + 1];
      cl[i] = cadd(cmul(cc[i], p), cmul(ss[i], q));
      cl[i + 1] = cadd(cmul(cmk(-ss[i].x, ss[i].y), p), cmul(cmk(cc[i].x, -cc[i].y), q));
    }
    const double2 hjj = cl[j], hj1 = cl[j + 1];
    const double denom = sqrt(cnorm2(hjj) + cnorm2(hj1));
    double2 c, sn;
    if (denom == 0.0) {
      c = cmk(1.0, 0.0);
      sn = cmk(0.0, 0.0);
    } else {
      c = cmk(hjj.x / denom, -hjj.y / denom);
      sn = cmk(hj1.x / denom, -hj1.y / denom);
    }
    a.cs[j] = c;
    a.sn[j] = sn;
    cl[j] = cadd(cmul(c, hjj), cmul(sn, hj1));
    cl[j + 1] = cmk(0.0, 0.0);
    const double2 gj = s[j];
    a.g[j + 1] = cmul(cmk(-sn.x, sn.y), gj);
    s[j] = cmul(c, gj);
    a.g[j] = s[j];
  }
  __syncthreads();
  for (int r = threadIdx.x; r < j + 2; r += blockDim.x) {
    col[r] = cl[r];
    if (r <= j) R[(size_t)j * (j + 1) / 2 + r] = cl[r];
  }
  __syncthreads();
  if (warp == 0) {  // column-oriented back substitution; c'_i = y_i sigma_i
    for (int i = m - 1; i >= 0; --i) {
      double2 yi = cmk(0.0, 0.0);
      if (lane == 0) {
        yi = lsa_cdiv(s[i], R[(size_t)i * (i + 1) / 2 + i]);
        a.cx[i] = cscale(a.sig[i], yi);
      }
      yi.x = __shfl_sync(0xffffffffu, yi.x, 0);
      yi.y = __shfl_sync(0xffffffffu, yi.y, 0);
      const double2* Ri = R + (size_t)i * (i + 1) / 2;
      for (int l = lane; l < i; l += 32) s[l] = csub(s[l], cmul(Ri[l], yi));
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// Device-side loop control for the graph-resident GMRES loop (WHILE node).
// ---------------------------------------------------------------------------
struct LoopState {
  int j;          // current iteration
  int done;       // loop finished (all remaining body kernels exit early)
  int iters;      // GmresResult::iterations when done
  int conv;       // converged flag
  int need_tail;  // budget exhausted: the host forms x_{maxit-1} and its monitor
};

// After the monitor of x_{j-1} (src/linalg.cpp:82-88): record the residual,
// stop on tolerance or Krylov breakdown of the previous step.
__global__ void k_loop_check(LoopState* s, const double* dres, double* res_hist, double tol,
                             cudaGraphConditionalHandle h) {
  if (s->done) return;
  const int j = s->j;
  if (j < 1) return;
  const double rr = dres[0];
  res_hist[j - 1] = rr;
  if (rr <= tol) {
    s->conv = 1;
    s->done = 1;
    s->iters = j;
    cudaGraphSetConditional(h, 0);
    return;
  }
  if (dres[1] < 1e-300) {  // hnew of iteration j-1
    s->done = 1;
    s->iters = j;
    cudaGraphSetConditional(h, 0);
  }
}

__global__ void k_loop_next(LoopState* s, int maxit, cudaGraphConditionalHandle h) {
  if (s->done) return;
  if (s->j + 1 >= maxit) {
    s->done = 1;
    s->need_tail = 1;
    s->iters = maxit;
    cudaGraphSetConditional(h, 0);
    return;
  }
  s->j += 1;
}

}  // namespace hd
