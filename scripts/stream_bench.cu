// Read-only streaming bandwidth on the B200 (the ceiling for Arnoldi pass 1):
// (0) grid-stride double2 loads, (1) the same with 8 independent vectors per
// warp (dot-product shape), (2) cp.async.bulk (TMA) 16 KB chunks into a
// 4-stage shared-memory ring with mbarriers, consumed by the CTA.
#include <cstdio>
#include <string>
#include <cuda_runtime.h>

__global__ void k_plain(const double2* __restrict__ a, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldg(a + i);
    s += v.x + v.y;
  }
  if (s == 12345.678) *out = s;
}

// V vectors of length n (contiguous), chunked like k_lsa_dots: CTA owns chunk, warp owns vectors
template <int CE>
__global__ void k_chunks(const double2* __restrict__ U, size_t n, int nv, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, NW = blockDim.x >> 5;
  double s = 0;
  const size_t nch = (n + CE - 1) / CE;
  for (size_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    for (int i = warp; i < nv; i += NW) {
      const double2* u = U + (size_t)i * n + ch * CE;
#pragma unroll 8
      for (int q = 0; q < CE / 32; ++q) {
        double2 v = __ldg(u + q * 32 + lane);
        s += v.x + v.y;
      }
    }
  }
  if (s == 12345.678) *out = s;
}

__device__ __forceinline__ void mbar_init(unsigned long long* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(b)),
      "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* g, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)),
               "l"(g), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b))
               : "memory");
}

template <int CE, int ST>
__global__ void k_tma(const double2* __restrict__ U, size_t n, int nv, double* out) {
  extern __shared__ __align__(128) double2 ring[];  // ST x CE
  __shared__ __align__(8) unsigned long long full[ST];
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0)
    for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  const size_t nch = (n + CE - 1) / CE;
  // work items: (chunk, vector) in CTA order
  const size_t my_chunks = nch > blockIdx.x ? (nch - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const size_t items = my_chunks * nv;
  auto src = [&](size_t it) {
    const size_t ch = blockIdx.x + (it / nv) * gridDim.x;
    const int i = (int)(it % nv);
    return U + (size_t)i * n + ch * CE;
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < ST && s < (int)items; ++s) {
      mbar_expect(&full[s], CE * 16);
      bulk_g2s(ring + (size_t)s * CE, src(s), CE * 16, &full[s]);
    }
  double acc = 0;
  for (size_t it = 0; it < items; ++it) {
    const int s = (int)(it % ST);
    const unsigned ph = (unsigned)((it / ST) & 1);
    mbar_wait(&full[s], ph);
    for (int e = threadIdx.x; e < CE; e += blockDim.x) {
      const double2 v = ring[(size_t)s * CE + e];
      acc += v.x + v.y;
    }
    __syncthreads();  // slot consumed
    if (threadIdx.x == 0 && it + ST < items) {
      mbar_expect(&full[s], CE * 16);
      bulk_g2s(ring + (size_t)s * CE, src(it + ST), CE * 16, &full[s]);
    }
  }
  if (acc == 12345.678) *out = acc + lane;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t n = 2563201 / 1024 * 1024;  // C5-sized vectors
  const int nv = 64;
  double2* U;
  double* out;
  cudaMalloc(&U, sizeof(double2) * n * nv);
  cudaMalloc(&out, 8);
  cudaMemset(U, 0, sizeof(double2) * n * nv);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = 16.0 * n * nv;
  auto run = [&](const char* name, auto launch) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("%-40s %8.1f GB/s  (%s)\n", name, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  for (int g : {nsm * 4, nsm * 8, nsm * 16})
    run((std::string("plain grid ") + std::to_string(g)).c_str(), [&] { k_plain<<<g, 256>>>(U, n * nv, out); });
  for (int cpb : {2, 4})
    run((std::string("chunks 1024, CTAs/SM ") + std::to_string(cpb)).c_str(),
        [&] { k_chunks<1024><<<nsm * cpb, 256>>>(U, n, nv, out); });
  cudaFuncSetAttribute(k_tma<1024, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 1024 * 16);
  cudaFuncSetAttribute(k_tma<2048, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 2048 * 16);
  cudaFuncSetAttribute(k_tma<1024, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 1024 * 16);
  for (int cpb : {1, 2, 3})
    run((std::string("tma 16KB x4, CTAs/SM ") + std::to_string(cpb)).c_str(),
        [&] { k_tma<1024, 4><<<nsm * cpb, 256, 4 * 1024 * 16>>>(U, n, nv, out); });
  for (int cpb : {1, 2})
    run((std::string("tma 32KB x4, CTAs/SM ") + std::to_string(cpb)).c_str(),
        [&] { k_tma<2048, 4><<<nsm * cpb, 256, 4 * 2048 * 16>>>(U, n, nv, out); });
  for (int cpb : {1, 2})
    run((std::string("tma 16KB x8, CTAs/SM ") + std::to_string(cpb)).c_str(),
        [&] { k_tma<1024, 8><<<nsm * cpb, 256, 8 * 1024 * 16>>>(U, n, nv, out); });
  return 0;
}
