// Exact solve of a 2D level operator that is not a Kronecker sum as a block
// tridiagonal system, standing in for the reference's Eigen::SparseLU: the
// deflation matrix E = Z^T A Z of the wedge and layered fields (real;
// src/precond.cpp:95-99, 103) and the whole shifted operator of C_ex on those
// fields (complex; src/precond.cpp:204-211).
//
// Ordering the unknowns lexicographically (x fastest) and grouping q = b grid
// rows (b = the stencil's half-width in y) into one "super-row" of m = q*n
// unknowns makes E block tridiagonal with nb = ceil(n/q) diagonal blocks D_i
// and couplings B_i = E[i, i+1], C_i = E[i, i-1].  The factorisation is
// twisted at the middle block k = nb/2 (cuBLAS / cuSOLVER at setup, partial
// pivoting inside each diagonal block): eliminated from the top for i < k,
//
//   S_0 = D_0,  S_i = D_i - G_i B_{i-1},  G_i = C_i S_{i-1}^-1,  H_i = S_i^-1 B_i,
//
// from the bottom for i > k,
//
//   T_{nb-1} = D_{nb-1},  T_i = D_i - G'_i C_{i+1},  G'_i = B_i T_{i+1}^-1,  H'_i = T_i^-1 C_i,
//
// and M = D_k - G_k B_{k-1} - G'_k C_{k+1} in the middle.  Per solve (real
// operator: the re and im planes are two real right-hand sides; complex
// operator: one complex right-hand side, planar), both halves run at once:
//
//   y_i = r_i - G_i y_{i-1} (i < k),   z_i = r_i - G'_i z_{i+1} (i > k),
//   w_i = S_i^-1 y_i,  w'_i = T_i^-1 z_i                     (alongside),
//   x_k = M^-1 (r_k - G_k y_{k-1} - G'_k z_{k+1}),
//   x_i = w_i - H_i x_{i+1} (i < k),   x_i = w'_i - H'_i x_{i-1} (i > k),
//
// about nb + 2 dependent steps instead of the 2 nb of a one-sided sweep.
//
// k_btri_solve runs this in one persistent kernel (one CTA per SM, a grid
// barrier between dependent steps).  A barrier-free variant that ordered the
// steps by dataflow on self-validating vector slots (sentinel-filled buffers
// polled by the consumers) was correct but 2x slower: 720 warps polling L2
// starve the producers' stores.  Each warp owns matrix rows; the matrices are
// stored row-major (a warp streams one contiguous row) and a warp loads the
// row of its first task of the next step between arriving at and waiting on
// the barrier.  Each step's input vectors are staged once per CTA in shared
// memory.  Padding rows (n not a multiple of q) carry an identity diagonal
// and a zero right-hand side.
#pragma once

#include "layered.cuh"

namespace hd {

// scalar helpers over double (real operator) and double2 (complex operator)
__device__ __forceinline__ double bt_zero(double) { return 0.0; }
__device__ __forceinline__ double2 bt_zero(double2) { return cmk(0.0, 0.0); }
__device__ __forceinline__ void bt_set(double& d, double2 v) { d = v.x; }
__device__ __forceinline__ void bt_set(double2& d, double2 v) { d = v; }
__device__ __forceinline__ double bt_one(double) { return 1.0; }
__device__ __forceinline__ double2 bt_one(double2) { return cmk(1.0, 0.0); }
// acc (re, im) += a * (vr + i vi)
__device__ __forceinline__ void bt_fma(double a, double vr, double vi, double& sr, double& si) {
  sr = fma(a, vr, sr);
  si = fma(a, vi, si);
}
__device__ __forceinline__ void bt_fma(double2 a, double vr, double vi, double& sr, double& si) {
  sr = fma(a.x, vr, fma(-a.y, vi, sr));
  si = fma(a.x, vi, fma(a.y, vr, si));
}

// warps per CTA by the registers a row needs per lane (doubles per lane)
// (round 2, C4, 24 doubles per lane: 256 / 320 / 384 / 512 / 640 / 768 threads give 27.6 / 26.3 / 25.9 / 28.3 /
// 28.5 / 31.8 ms per solve; prefetching the rows of a warp's first TWO tasks across the barrier: 26.3 ms -- the
// step time is the barrier and the dependent vector hand-over, not the rows' DRAM latency; blocks of 2b grid
// rows (m = 1440, 40 blocks, dense factors): 28.2 ms -- half the steps, twice the bytes, 15 us per step)
#ifndef HD_BTRI_T32
#define HD_BTRI_T32 384
#endif
__host__ __device__ constexpr int btri_threads(int regs) { return regs <= 16 ? 512 : (regs <= 32 ? HD_BTRI_T32 : 256); }

struct BtriArgs {
  int n, q, m, nb, k;  // grid side, rows per block, block size m = q*n, blocks, middle block
  size_t NN;           // n^2 (unknowns); padded length nb*m
  const void* GT;      // nb blocks, row-major: G_i (0 < i <= k), G'_i (k < i < nb-1)   [double or double2]
  const void* G2;      // one block: G'_k (k < nb-1)
  const void* SinvT;   // nb blocks, row-major: S_i^-1 (i < k), M^-1 (k), T_i^-1 (i > k)
  const void* HT;      // nb blocks, row-major: H_i (i < k), H'_i (i > k)
  double* y;           // 2 planes x nb*m
  double* w;           // 2 planes x nb*m
  double* x;           // 2 planes x nb*m
  double* io;          // in/out planar (re plane NN, im plane NN)
  unsigned* bar;       // grid barrier counter, zeroed before the launch
  const void* steps;   // the solve's step table (BtStep per step), built on the host at setup
  int nsteps;
};

// Column-major m x m blocks D_i, B_i (= E[i, i+1]), C_i (= E[i, i-1]) of the
// level operator (T = double: its real part; the coefficients must be real).
template <class T>
__global__ void k_btri_blocks(GenLevel L, int q, int m, int nb, T* __restrict__ D, T* __restrict__ Bu,
                              T* __restrict__ Cl) {
  const int n = L.n;
  const size_t mm = (size_t)m * m, tot = (size_t)nb * mm;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(e / mm);
    const size_t rem = e % mm;
    const int a = (int)(rem % m), c = (int)(rem / m);  // column-major (row a, column c)
    const int iy = i * q + a / n, ix = a % n;
    T d = bt_zero(T()), bu = bt_zero(T()), cl = bt_zero(T());
    if (iy < n) {
      // diagonal block: column c is unknown (i*q + c/n, c%n)
      const int jy = i * q + c / n, jx = c % n;
      const int dy = jy - iy, dx = jx - ix;
      if (jy < n && dy >= -L.b && dy <= L.b && dx >= -L.b && dx <= L.b) bt_set(d, gen_entry(L, iy, ix, dy, dx));
      const int jyu = (i + 1) * q + c / n, dyu = jyu - iy;
      if (jyu < n && dyu <= L.b && dx >= -L.b && dx <= L.b) bt_set(bu, gen_entry(L, iy, ix, dyu, dx));
      const int jyl = (i - 1) * q + c / n, dyl = jyl - iy;
      if (i > 0 && dyl >= -L.b && dx >= -L.b && dx <= L.b) bt_set(cl, gen_entry(L, iy, ix, dyl, dx));
    } else if (a == c) {
      d = bt_one(T());  // padding unknown
    }
    D[e] = d;
    Bu[e] = bu;
    Cl[e] = cl;
  }
}

// One matrix row (m entries, lane-strided into KR registers).
template <class T, int KR>
__device__ __forceinline__ void btri_row_load(const T* __restrict__ row, int m, T (&r)[KR]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int c = lane + 32 * k;
    r[k] = c < m ? __ldcs(row + c) : bt_zero(T());
  }
}

__device__ __forceinline__ void btri_arrive(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
  }
}

__device__ __forceinline__ void btri_wait(unsigned* bar, unsigned target) {
  if (threadIdx.x == 0) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar));
    } while (v < target);
    __threadfence();
  }
  __syncthreads();
}

// The step's input vector (planar: re plane at v, im plane at v + plane),
// written by other CTAs before the last barrier, staged once per CTA into
// shared memory (vs: m re values, then m im values).
__device__ __forceinline__ void btri_stage(const double* v, size_t plane, int m, double* vs) {
  for (int c = threadIdx.x; c < m; c += blockDim.x) {
    vs[c] = __ldcg(v + c);
    vs[m + c] = __ldcg(v + plane + c);
  }
  __syncthreads();
}

// Row dot with the staged vector.
template <class T, int KR>
__device__ __forceinline__ double2 btri_row_dot(const T (&r)[KR], const double* vs, int m) {
  const int lane = threadIdx.x & 31;
  double sr0 = 0.0, si0 = 0.0, sr1 = 0.0, si1 = 0.0;
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int c = lane + 32 * k;
    if (c < m) {
      const double vr = vs[c], vi = vs[m + c];
      if (k & 1) bt_fma(r[k], vr, vi, sr1, si1);
      else bt_fma(r[k], vr, vi, sr0, si0);
    }
  }
  double sr = sr0 + sr1, si = si0 + si1;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, o);
    si += __shfl_xor_sync(0xffffffffu, si, o);
  }
  return cmk(sr, si);
}

// One group of m row tasks of a solve step: out row = (rhs) - mat * vec (+ second product).
struct BtGroup {
  int kind;       // 0 none, 1 y/z (rhs - A v), 2 w (A v), 3 middle y_k (rhs - A v - A2 v2), 4 x_k (A v), 5 x (w - A v)
  int blk;        // block of the output rows
  int vec, vec2;  // staged vector slots (0, 1) read by the products
  int mat, mat2;  // matrix: 0 none, 1 GT[blk], 2 SinvT[blk'], 3 HT[blk], 4 G2 ; blk' = mblk
  int mblk;       // block of the (first) matrix
};

// Step s of the twisted solve: up to 4 groups and the (up to 2) input vectors
// to stage (block index and buffer: 0 = y, 1 = x; -1 = none).
struct BtStep {
  BtGroup g[4];
  int ng;
  int sv_blk[2], sv_buf[2];
};

// word offsets inside the step table (BtStep as ints), used where a single field is read from global memory
constexpr int kGroupWords = (int)(sizeof(BtGroup) / sizeof(int));
constexpr int kGroupMatWord = 4, kGroupMblkWord = 6;  // BtGroup::mat, BtGroup::mblk
constexpr int kStepNgWord = 4 * kGroupWords;          // BtStep::ng
static_assert(sizeof(BtGroup) == 7 * sizeof(int) && sizeof(BtStep) == (4 * 7 + 5) * sizeof(int), "step table layout");

__host__ __device__ inline BtStep btri_step(int s, int nb, int k) {
  BtStep st;
  st.ng = 0;
  st.sv_blk[0] = st.sv_blk[1] = -1;
  st.sv_buf[0] = st.sv_buf[1] = 0;
  const int F = k > nb - 1 - k ? k : nb - 1 - k;  // forward steps
  auto add = [&](int kind, int blk, int vec, int mat, int mblk, int vec2 = 0, int mat2 = 0) {
    BtGroup& g = st.g[st.ng++];
    g.kind = kind;
    g.blk = blk;
    g.vec = vec;
    g.vec2 = vec2;
    g.mat = mat;
    g.mat2 = mat2;
    g.mblk = mblk;
  };
  if (s < F) {  // forward: top block i = s (< k), bottom block i = nb-1-s (> k)
    const int it = s, ib = nb - 1 - s;
    if (it < k) {
      if (it > 0) {
        st.sv_blk[0] = it - 1;
        add(1, it, 0, 1, it);       // y_it = r - G_it y_{it-1}
        add(2, it - 1, 0, 2, it - 1);  // w_{it-1} = S^-1 y_{it-1}
      } else {
        add(1, it, 0, 0, it);       // y_0 = r_0
      }
    }
    if (ib > k) {
      if (ib < nb - 1) {
        st.sv_blk[1] = ib + 1;
        add(1, ib, 1, 1, ib);       // z_ib = r - G'_ib z_{ib+1}
        add(2, ib + 1, 1, 2, ib + 1);  // w'_{ib+1} = T^-1 z_{ib+1}
      } else {
        add(1, ib, 1, 0, ib);       // z_{nb-1} = r_{nb-1}
      }
    }
    return st;
  }
  if (s == F) {  // middle right-hand side and the last w / w'
    if (k > 0) st.sv_blk[0] = k - 1;
    if (k < nb - 1) st.sv_blk[1] = k + 1;
    add(3, k, 0, k > 0 ? 1 : 0, k, 1, k < nb - 1 ? 4 : 0);
    if (k > 0) add(2, k - 1, 0, 2, k - 1);
    if (k < nb - 1) add(2, k + 1, 1, 2, k + 1);
    return st;
  }
  if (s == F + 1) {  // x_k = M^-1 y_k
    st.sv_blk[0] = k;
    add(4, k, 0, 2, k);
    return st;
  }
  const int t = s - F - 1;  // backward step t >= 1: x_{k-t} (top) and x_{k+t} (bottom)
  const int it = k - t, ib = k + t;
  if (it >= 0) {
    st.sv_blk[0] = it + 1;
    st.sv_buf[0] = 1;
    add(5, it, 0, 3, it);
  }
  if (ib <= nb - 1) {
    st.sv_blk[1] = ib - 1;
    st.sv_buf[1] = 1;
    add(5, ib, 1, 3, ib);
  }
  return st;
}

template <class T>
__device__ __forceinline__ const T* bt_mat(const BtriArgs& a, int mat, int blk, int row) {
  const size_t mm = (size_t)a.m * a.m, off = (size_t)blk * mm + (size_t)row * a.m;
  switch (mat) {
    case 1: return static_cast<const T*>(a.GT) + off;
    case 2: return static_cast<const T*>(a.SinvT) + off;
    case 3: return static_cast<const T*>(a.HT) + off;
    case 4: return static_cast<const T*>(a.G2) + (size_t)row * a.m;
    default: return nullptr;
  }
}

template <class T, int KR>
__global__ void __launch_bounds__(btri_threads(KR * (int)(sizeof(T) / 8)), 1) k_btri_solve(BtriArgs a) {
  const int lane = threadIdx.x & 31;
  const int wpb = blockDim.x >> 5;
  const int gw = blockIdx.x * wpb + (threadIdx.x >> 5);
  const int W = gridDim.x * wpb;
  const int m = a.m, nb = a.nb, k = a.k;
  const size_t P = (size_t)nb * m;
  const unsigned G = gridDim.x;
  const int nsteps = a.nsteps;
  unsigned phase = 0;
  T r[KR];
  extern __shared__ double vs[];  // two staged vectors, 2m doubles each
  // The step table was built on the host (btri_step): the descriptor of the current step and, loaded between
  // arriving at and waiting on the barrier, of the next one live in shared memory -- no per-thread recomputation
  // of the schedule and no local-memory copy of it (round 2: 16% of the kernel's instructions were the
  // schedule's integer arithmetic and 8% its local-memory traffic).
  __shared__ BtStep sst[2];
  constexpr int kStepWords = (int)(sizeof(BtStep) / sizeof(int));
  const int* steps_w = static_cast<const int*>(a.steps);
  if (threadIdx.x < kStepWords) reinterpret_cast<int*>(&sst[0])[threadIdx.x] = __ldg(steps_w + threadIdx.x);
  __syncthreads();
  int pre = -1;                   // task whose matrix row r holds (prefetched), -1: none
  const int gw0 = gw / m, gr0 = gw % m;  // group and row of this warp's first task of any step
  for (int s = 0; s < nsteps; ++s) {
    const BtStep& st = sst[s & 1];
    const int ntask = st.ng * m;
    // stage this step's input vectors (every CTA with tasks)
    if (blockIdx.x * wpb < ntask) {
      for (int v = 0; v < 2; ++v) {
        if (st.sv_blk[v] < 0) continue;
        const double* src = (st.sv_buf[v] ? a.x : a.y) + (size_t)st.sv_blk[v] * m;
        for (int c = threadIdx.x; c < m; c += blockDim.x) {
          vs[v * 2 * m + c] = __ldcg(src + c);
          vs[v * 2 * m + m + c] = __ldcg(src + P + c);
        }
      }
      __syncthreads();
    }
    // tasks t = gw, gw + W, ...: group t / m and row t % m advanced without divisions
    int grp = gw0, row = gr0;
    for (int t = gw; t < ntask; t += W) {
      const BtGroup& g = st.g[grp];
      const size_t gi = (size_t)g.blk * m + row;
      double br = 0.0, bi = 0.0;  // rhs (kinds 1, 3) or w (kind 5)
      if (lane == 0) {
        if ((g.kind == 1 || g.kind == 3) && gi < a.NN) {
          br = a.io[gi];
          bi = a.io[a.NN + gi];
        } else if (g.kind == 5) {
          br = __ldcg(a.w + gi);
          bi = __ldcg(a.w + P + gi);
        }
      }
      double2 acc = cmk(0.0, 0.0);
      if (g.mat) {
        if (t != pre) btri_row_load<T, KR>(bt_mat<T>(a, g.mat, g.mblk, row), m, r);
        acc = btri_row_dot<T, KR>(r, vs + g.vec * 2 * m, m);
      }
      if (g.kind == 3 && g.mat2) {
        btri_row_load<T, KR>(bt_mat<T>(a, g.mat2, g.mblk, row), m, r);
        const double2 a2 = btri_row_dot<T, KR>(r, vs + g.vec2 * 2 * m, m);
        acc = cadd(acc, a2);
      }
      pre = -1;
      if (lane == 0) {
        double xr, xi;
        double* dst;
        if (g.kind == 1 || g.kind == 3) {
          xr = br - acc.x; xi = bi - acc.y; dst = a.y;
        } else if (g.kind == 2) {
          xr = acc.x; xi = acc.y; dst = a.w;
        } else if (g.kind == 4) {
          xr = acc.x; xi = acc.y; dst = a.x;
        } else {
          xr = br - acc.x; xi = bi - acc.y; dst = a.x;
        }
        dst[gi] = xr;
        dst[P + gi] = xi;
        if ((g.kind == 4 || g.kind == 5) && gi < a.NN) {
          a.io[gi] = xr;
          a.io[a.NN + gi] = xi;
        }
      }
      row += W;
      while (row >= m) {
        row -= m;
        ++grp;
      }
    }
    if (s + 1 < nsteps) {
      btri_arrive(a.bar);
      // the next step's descriptor (read by this CTA only after the barrier's closing __syncthreads)
      if (threadIdx.x < kStepWords)
        reinterpret_cast<int*>(&sst[(s + 1) & 1])[threadIdx.x] = __ldg(steps_w + (size_t)(s + 1) * kStepWords + threadIdx.x);
      {  // prefetch the first task's row of the next step (its group comes straight from the table)
        const int ng1 = __ldg(steps_w + (size_t)(s + 1) * kStepWords + kStepNgWord);
        if (gw < ng1 * m) {
          const int* gwd = steps_w + (size_t)(s + 1) * kStepWords + gw0 * kGroupWords;
          const int mat = __ldg(gwd + kGroupMatWord), mblk = __ldg(gwd + kGroupMblkWord);
          if (mat) {
            btri_row_load<T, KR>(bt_mat<T>(a, mat, mblk, gr0), m, r);
            pre = gw;
          }
        }
      }
      btri_wait(a.bar, ++phase * G);
    }
  }
}

}  // namespace hd
