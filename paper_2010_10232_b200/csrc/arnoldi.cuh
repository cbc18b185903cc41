// Persistent cooperative Arnoldi tail: one launch per GMRES iteration does
//   modified Gram-Schmidt of w against V_0..V_j   (src/linalg.cpp:42-45)
//   hnew = ||w||, V_{j+1} = w / hnew               (:46-47, :89)
//   Givens rotations of column j + back substitution (:49-77)
//   x_j = x0 + sum_i y_i V_i                       (:78-80)
//
// B200 design: w never leaves the chip during the MGS chain.  Each CTA owns a
// contiguous chunk; thread t holds its elements e_k = c0 + k*BD + t, the first
// RW in registers and the rest in shared memory (C5: 17 complex per thread,
// 4 in registers + 13 in 208 KB of shared memory, 148 CTAs x 1024 threads).
// MGS step i streams V_i from HBM once for the dot and re-reads it from L2 for
// the update in step i+1 (fused with the dot against V_{i+1}).  Between the
// two, a split grid barrier: each CTA arrives, issues L2 prefetches of its
// chunk of V_{i+1}, then waits -- the HBM fetch overlaps the barrier latency.
// The exact MGS order of the reference is kept: h_i is formed from w after
// the updates with h_0..h_{i-1}.  Reductions: block tree -> one partial per
// CTA -> every CTA sums the G partials in index order (deterministic and
// identical in every CTA).
#pragma once

#include "device_common.cuh"

namespace hd {

constexpr int kArnBD = 1024;  // threads per CTA
constexpr int kArnRW = 4;     // register-resident complex per thread
constexpr int kArnU = 4;      // shared-memory elements processed per batch (loads first)

struct ArnoldiArgs {
  const double2* V;     // basis, (maxit+1) x N
  double2* Vw;          // == V, written at V_{j+1}
  const double2* w;     // op(V_j)
  const double2* x0;
  double2* x;           // iterate out
  size_t N;
  int* dj;              // device iteration index j (read; incremented at the end)
  const int* done;      // early exit flag (speculative launches); may be null
  double2* H;           // column-major, ldh
  int ldh;
  double2* g;
  double2* cs;
  double2* sn;
  double2* y;
  double* hnew_out;     // scalar
  double2* partials;    // 2 * G
  unsigned* bar;        // grid barrier counter, zero at launch
  int K;                // elements per thread (ceil(chunk / BD))
  size_t chunk;         // elements per CTA
  unsigned long long* trace;  // optional phase timestamps (block 0)
};

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void bar_arrive(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
  }
}

__device__ __forceinline__ void bar_wait(unsigned* bar, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar));
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}

// sum of the G partials of `slot`, identical in every CTA (lane-0 order)
__device__ __forceinline__ double2 arn_collect(const double2* partials, int slot, double2* sred) {
  if (threadIdx.x < 32) {
    double2 s = cmk(0.0, 0.0);
    for (unsigned i = threadIdx.x; i < gridDim.x; i += 32) s = cadd(s, __ldcg(&partials[slot * gridDim.x + i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s.x += __shfl_down_sync(0xffffffffu, s.x, o);
      s.y += __shfl_down_sync(0xffffffffu, s.y, o);
    }
    if (threadIdx.x == 0) sred[32] = s;
  }
  __syncthreads();
  return sred[32];
}

__device__ __forceinline__ double2 cdiv_(double2 a, double2 b) { return cmul(a, cinv(b)); }

// Givens update of column j and back substitution by block 0
// (src/linalg.cpp:49-77).  sm: >= (m(m+1)/2 + 3(j+2)) complex.
__device__ void arn_givens(const ArnoldiArgs& a, int j, double2* sm) {
  const int m = j + 1;
  double2* col = a.H + (size_t)j * a.ldh;
  double2* R = sm;                              // packed upper triangle, column c at c(c+1)/2
  double2* s = R + (size_t)m * (m + 1) / 2;     // g[0..m)
  double2* cl = s + m + 1;                      // column j (j+2 entries)
  double2* cc = cl + j + 2;                     // cs[0..j)
  double2* ss = cc + j + 1;                     // sn[0..j)
  for (int r = threadIdx.x; r < j + 2; r += blockDim.x) cl[r] = col[r];
  for (int r = threadIdx.x; r < j; r += blockDim.x) {
    cc[r] = a.cs[r];
    ss[r] = a.sn[r];
  }
  for (int c = 0; c < j; ++c)
    for (int r = threadIdx.x; r <= c; r += blockDim.x) R[(size_t)c * (c + 1) / 2 + r] = a.H[(size_t)c * a.ldh + r];
  for (int r = threadIdx.x; r <= j; r += blockDim.x) s[r] = a.g[r];
  __syncthreads();
  if (threadIdx.x == 0) {
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
  // column-oriented back substitution, one warp, s in shared memory
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int i = m - 1; i >= 0; --i) {
      double2 yi = cmk(0.0, 0.0);
      if (lane == 0) {
        yi = cdiv_(s[i], R[(size_t)i * (i + 1) / 2 + i]);
        a.y[i] = yi;
      }
      yi.x = __shfl_sync(0xffffffffu, yi.x, 0);
      yi.y = __shfl_sync(0xffffffffu, yi.y, 0);
      const double2* Ri = R + (size_t)i * (i + 1) / 2;
      for (int l = lane; l < i; l += 32) s[l] = csub(s[l], cmul(Ri[l], yi));
      __syncwarp();
    }
  }
}

template <int RW>
__global__ void __launch_bounds__(kArnBD, 1) k_arnoldi(ArnoldiArgs a) {
  HD_PDL_ENTRY();
  extern __shared__ __align__(16) double2 wsm[];
  __shared__ double2 sred[33];
  __shared__ double2 ys[128];
  __shared__ int s_j;
  if (a.done && *((volatile const int*)a.done)) return;  // uniform across the grid
  const int BD = blockDim.x;
  const int t = threadIdx.x;
  const bool tr = a.trace && blockIdx.x == 0 && t == 0;
  if (tr) a.trace[0] = gtime();
  if (t == 0) s_j = *((volatile int*)a.dj);
  __syncthreads();
  const int j = s_j;
  const size_t N = a.N;
  const size_t c0 = (size_t)blockIdx.x * a.chunk;
  const size_t c1 = min(N, c0 + a.chunk);
  const int K = a.K;
  const unsigned G = gridDim.x;
  unsigned phase = 0;
  // resident store: element k at e = c0 + k*BD + t; k < RW in wr[], else wsm
  double2 wr[RW];
#pragma unroll
  for (int k = 0; k < RW; ++k) {
    const size_t e = c0 + (size_t)k * BD + t;
    wr[k] = (k < K && e < c1) ? ld_stream(a.w + e) : cmk(0.0, 0.0);
  }
  for (int k = RW; k < K; ++k) {
    const size_t e = c0 + (size_t)k * BD + t;
    wsm[(size_t)(k - RW) * BD + t] = e < c1 ? ld_stream(a.w + e) : cmk(0.0, 0.0);
  }
  // ---- MGS chain: step i fuses  w -= h_{i-1} V_{i-1}  with  acc = conj(V_i).w
  //      (i <= j)  or  acc = |w|^2  (i = j+1)
  double2* Hj = a.H + (size_t)j * a.ldh;
  double2 h = cmk(0.0, 0.0);
  for (int i = 0; i <= j + 1; ++i) {
    const double2* Vo = i > 0 ? a.V + (size_t)(i - 1) * N : nullptr;
    const double2* Vn = i <= j ? a.V + (size_t)i * N : nullptr;
    double2 acc = cmk(0.0, 0.0);
    {
      double2 vo[RW], vn[RW];
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        const size_t e = c0 + (size_t)k * BD + t;
        const bool ok = k < K && e < c1;
        vo[k] = (Vo && ok) ? ld_stream(Vo + e) : cmk(0.0, 0.0);  // last use: evict first
        vn[k] = (Vn && ok) ? Vn[e] : cmk(0.0, 0.0);                // kept in L2 for step i+1
      }
#pragma unroll
      for (int k = 0; k < RW; ++k) {
        wr[k] = csub(wr[k], cmul(h, vo[k]));
        if (Vn) acc = cadd(acc, cconjmul(vn[k], wr[k]));
        else acc.x += cnorm2(wr[k]);
      }
    }
    for (int k0 = RW; k0 < K; k0 += kArnU) {
      double2 vo[kArnU], vn[kArnU];
#pragma unroll
      for (int u = 0; u < kArnU; ++u) {
        const size_t e = c0 + (size_t)(k0 + u) * BD + t;
        const bool ok = (k0 + u) < K && e < c1;
        vo[u] = (Vo && ok) ? ld_stream(Vo + e) : cmk(0.0, 0.0);
        vn[u] = (Vn && ok) ? Vn[e] : cmk(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kArnU; ++u) {
        if (k0 + u < K) {
          double2* ws = &wsm[(size_t)(k0 + u - RW) * BD + t];
          const double2 wv = csub(*ws, cmul(h, vo[u]));
          *ws = wv;
          if (Vn) acc = cadd(acc, cconjmul(vn[u], wv));
          else acc.x += cnorm2(wv);
        }
      }
    }
    // split grid barrier: publish the partial, prefetch V_{i+1}, then wait
    acc = block_sum2(acc, sred);
    if (t == 0) a.partials[(phase & 1) * G + blockIdx.x] = acc;
    bar_arrive(a.bar);
    ++phase;
    if (i + 1 <= j && (t & 7) == 0) {  // one prefetch per 128-B line
      const double2* Vp = a.V + (size_t)(i + 1) * N;
      for (int k = 0; k < K; ++k) {
        const size_t e = c0 + (size_t)k * BD + t;
        if (e < c1) prefetch_l2(Vp + e);
      }
    }
    bar_wait(a.bar, phase * G);
    h = arn_collect(a.partials, (phase - 1) & 1, sred);
    if (i <= j && blockIdx.x == 0 && t == 0) Hj[i] = h;
  }
  if (tr) a.trace[1] = gtime();
  // h now holds (|w|^2, 0)
  const double hnew = sqrt(h.x);
  if (blockIdx.x == 0 && t == 0) {
    Hj[j + 1] = cmk(hnew, 0.0);
    *a.hnew_out = hnew;
  }
  // V_{j+1} = w / hnew (written unconditionally; unused once GMRES stops)
  double2* Vn1 = a.Vw + (size_t)(j + 1) * N;
  const double inv = hnew > 0.0 ? 1.0 / hnew : 0.0;
#pragma unroll
  for (int k = 0; k < RW; ++k) {
    const size_t e = c0 + (size_t)k * BD + t;
    if (k < K && e < c1) Vn1[e] = cmk(wr[k].x * inv, wr[k].y * inv);
  }
  for (int k = RW; k < K; ++k) {
    const size_t e = c0 + (size_t)k * BD + t;
    if (e < c1) {
      const double2 wv = wsm[(size_t)(k - RW) * BD + t];
      Vn1[e] = cmk(wv.x * inv, wv.y * inv);
    }
  }
  // ---- Givens + back substitution in block 0 -------------------------------
  if (blockIdx.x == 0) {
    __syncthreads();  // wsm is reused as the R stage
    arn_givens(a, j, wsm);
    if (tr) a.trace[2] = gtime();
  }
  bar_arrive(a.bar);
  ++phase;
  bar_wait(a.bar, phase * G);
  if (tr) a.trace[3] = gtime();
  // ---- iterate x = x0 + sum_{i<=j} y_i V_i  (i outer: K independent loads per thread)
  const int m = j + 1;
  for (int q = t; q < m; q += BD) ys[q] = __ldcg(&a.y[q]);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < RW; ++k) {
    const size_t e = c0 + (size_t)k * BD + t;
    wr[k] = (k < K && e < c1) ? a.x0[e] : cmk(0.0, 0.0);
  }
  for (int k = RW; k < K; ++k) {
    const size_t e = c0 + (size_t)k * BD + t;
    wsm[(size_t)(k - RW) * BD + t] = e < c1 ? a.x0[e] : cmk(0.0, 0.0);
  }
  for (int i = 0; i < m; ++i) {
    const double2 yi = ys[i];
    const double2* Vi = a.V + (size_t)i * N;
    double2 v[RW];
#pragma unroll
    for (int k = 0; k < RW; ++k) {
      const size_t e = c0 + (size_t)k * BD + t;
      v[k] = (k < K && e < c1) ? ld_stream(Vi + e) : cmk(0.0, 0.0);
    }
#pragma unroll
    for (int k = 0; k < RW; ++k) wr[k] = cfma(yi, v[k], wr[k]);
    for (int k0 = RW; k0 < K; k0 += kArnU) {
      double2 vv[kArnU];
#pragma unroll
      for (int u = 0; u < kArnU; ++u) {
        const size_t e = c0 + (size_t)(k0 + u) * BD + t;
        vv[u] = ((k0 + u) < K && e < c1) ? ld_stream(Vi + e) : cmk(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < kArnU; ++u)
        if (k0 + u < K) {
          double2* ws = &wsm[(size_t)(k0 + u - RW) * BD + t];
          *ws = cfma(yi, vv[u], *ws);
        }
    }
  }
#pragma unroll
  for (int k = 0; k < RW; ++k) {
    const size_t e = c0 + (size_t)k * BD + t;
    if (k < K && e < c1) a.x[e] = wr[k];
  }
  for (int k = RW; k < K; ++k) {
    const size_t e = c0 + (size_t)k * BD + t;
    if (e < c1) a.x[e] = wsm[(size_t)(k - RW) * BD + t];
  }
  if (tr) a.trace[4] = gtime();
  if (blockIdx.x == 0 && t == 0) *a.dj = j + 1;
}

}  // namespace hd
