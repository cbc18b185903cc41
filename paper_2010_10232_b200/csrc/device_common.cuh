// Device-side helpers shared by the solver kernels: complex double arithmetic
// on double2 (interleaved, the layout of Eigen::VectorXcd), cp.async staging
// and the deterministic block / grid reductions used by every inner product.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace hd {

__host__ __device__ __forceinline__ double2 cmk(double r, double i) { return make_double2(r, i); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return cmk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return cmk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return cmk(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// conj(a) * b
__device__ __forceinline__ double2 cconjmul(double2 a, double2 b) {
  return cmk(fma(a.x, b.x, a.y * b.y), fma(a.x, b.y, -a.y * b.x));
}
__device__ __forceinline__ double2 cscale(double s, double2 a) { return cmk(s * a.x, s * a.y); }
// acc + s * a (s real)
__device__ __forceinline__ double2 cfma_r(double s, double2 a, double2 acc) {
  return cmk(fma(s, a.x, acc.x), fma(s, a.y, acc.y));
}
// acc + a * b (complex)
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  return cmk(fma(a.x, b.x, fma(-a.y, b.y, acc.x)), fma(a.x, b.y, fma(a.y, b.x, acc.y)));
}
__device__ __forceinline__ double2 cinv(double2 d) {
  const double s = 1.0 / fma(d.x, d.x, d.y * d.y);
  return cmk(d.x * s, -d.y * s);
}
__device__ __forceinline__ double cnorm2(double2 a) { return fma(a.x, a.x, a.y * a.y); }

// ---- cp.async (LDGSTS) 16-byte staging with zero fill --------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- streaming loads that do not pollute L2 (basis vectors in MGS) -------
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.cs.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// ---- warp / block reductions (fixed order => deterministic) -------------
__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// Sums v over the block; result valid in thread 0.  scratch: >= 32 double2.
__device__ __forceinline__ double2 block_sum2(double2 v, double2* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum2(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < nw ? scratch[lane] : cmk(0.0, 0.0);
    v = warp_sum2(v);
  }
  return v;
}

// Grid reduction by "last block done": every block stores its partial, the
// last block to arrive sums all partials in index order (deterministic for a
// fixed grid) and returns true in thread 0 with the total in *total.
// counter must be zero on entry; it is reset by the last block.
__device__ __forceinline__ bool grid_sum2(double2 v, double2* partials, unsigned* counter, double2* scratch,
                                          double2* total) {
  __shared__ bool am_last;
  const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
  v = block_sum2(v, scratch);
  if (threadIdx.x == 0) {
    partials[bid] = v;
    __threadfence();
    const unsigned ticket = atomicAdd(counter, 1u);
    am_last = (ticket == nb - 1);
  }
  __syncthreads();
  if (!am_last) return false;
  __threadfence();
  double2 s = cmk(0.0, 0.0);
  for (unsigned i = threadIdx.x; i < nb; i += blockDim.x) s = cadd(s, __ldcg(&partials[i]));
  s = block_sum2(s, scratch);
  if (threadIdx.x == 0) {
    *total = s;
    *counter = 0u;
  }
  return threadIdx.x == 0;
}

}  // namespace hd
