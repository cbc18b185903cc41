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

#include <cuda.h>  // CUtensorMap (type only)

#include "device_common.cuh"

namespace hd {

constexpr int kLsaBD = 256;  // threads per CTA
constexpr int kLsaTE = 4;    // elements per thread per tile
#ifndef HD_LSA_VPS
#define HD_LSA_VPS 2
#endif
constexpr int kLsaVPS = HD_LSA_VPS;  // basis vectors per step of pass 2
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
  int jlag;           // Givens only: work on iteration (j - jlag) (graph mode: the previous
                      // iteration's Givens overlaps this iteration's operator)
  int part_offset;    // row slabs: this slab's first CTA slot in `partials` (0: single domain)
  int partial_only;   // row slabs: pass 1 writes its CTA partials and stops (k_lsa_dots_finish
                      // combines the slabs' partials in slab order)
  int rev;            // pass 2 walks its tiles from the end of the vectors: pass 1 read them front to
                      // back, so the tail of every basis vector is what the L2 still holds
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
__device__ __forceinline__ double2 lsa_collect(const double2* partials, int nslot, int q, int nparts) {
  double2 s = cmk(0.0, 0.0);
  const int lane = threadIdx.x & 31;
  for (int b = lane; b < nparts; b += 32) s = cadd(s, __ldcg(&partials[(size_t)b * nslot + q]));
  s = lsa_warp_sum(s);
  return cmk(__shfl_sync(0xffffffffu, s.x, 0), __shfl_sync(0xffffffffu, s.y, 0));
}

// ---------------------------------------------------------------------------
// pass 1: dots against w and u_j as a chunked GEMV-T.  Each CTA stages a chunk
// of w and u_j in shared memory; its warps stream whole basis vectors over the
// chunk (coalesced, 8 loads in flight per lane) and reduce once per chunk and
// vector into per-CTA shared accumulators (one warp owns each vector slot).
// ---------------------------------------------------------------------------
constexpr int kLsaCE = 1024;  // chunk elements

struct LsaArgs;
__device__ void lsa_dots_finish(const LsaArgs& a, int j, int nparts, double2* sh_s, double2* sh_lj, double2* hsm);

// basis loads in flight per lane in pass 1 (16: C5 90.0 -> 89.3 ms against 8, with the
// double-buffered w / u_j chunks; a split of each vector chunk over two warps needs
// per-item partial slots and was not pursued)
#ifndef HD_LSA_UNROLL
#define HD_LSA_UNROLL 16
#endif
constexpr int kLsaUnroll = HD_LSA_UNROLL;

// Items per chunk and vector: each staged chunk's vector products are split into
// kLsaSplit sub-chunk items so that the j+1 vectors spread evenly over the warps
// between the chunk barriers; every split has its own accumulator slots, summed
// in split order at the end (deterministic).
#ifndef HD_LSA_SPLIT
#define HD_LSA_SPLIT 1
#endif
constexpr int kLsaSplit = HD_LSA_SPLIT;

constexpr size_t lsa_dots_smem() { return sizeof(double2) * (4 * kLsaCE + kLsaSplit * 2 * (kLsaMaxJ + 1)); }

__global__ void __launch_bounds__(kLsaBD, 2) k_lsa_dots(LsaArgs a) {
  constexpr int NW = kLsaBD / 32;
  constexpr int PER = kLsaCE / 32 / kLsaSplit;  // elements per lane per item
  extern __shared__ __align__(16) double2 dsm[];
  // w and u_j chunks, double-buffered: the next chunk's pair is copied (cp.async)
  // while the warps stream the basis vectors against the current one
  double2* wsb = dsm;                   // [2][kLsaCE] w chunks
  double2* usb = dsm + 2 * kLsaCE;      // [2][kLsaCE] u_j chunks
  double2* acc = dsm + 4 * kLsaCE;      // [0..j]: s_i ; [kLsaMaxJ+1 ..]: G_ji
  __shared__ double2 sh_s[kLsaMaxJ + 1];
  __shared__ double2 sh_lj[kLsaMaxJ];
  __shared__ double2 hsm[kLsaMaxJ + 1];
  if (a.done && *((volatile const int*)a.done)) return;
  const int j = a.dj ? *a.dj : a.j;
  const int nd = j + 1;
  const int nslot = 2 * kLsaMaxJ + 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = threadIdx.x; q < kLsaSplit * nslot; q += kLsaBD) acc[q] = cmk(0.0, 0.0);
  const size_t N = a.N;
  const double2* uj = a.U + (size_t)j * N;
  const size_t nchunks = (N + kLsaCE - 1) / kLsaCE;
  auto stage = [&](size_t ch, int buf) {
    if (ch < nchunks) {
      const size_t c0 = ch * kLsaCE;
      const int len = (int)min((size_t)kLsaCE, N - c0);
      for (int e = threadIdx.x; e < kLsaCE; e += kLsaBD) {
        const bool v = e < len;
        cp_async16(wsb + buf * kLsaCE + e, v ? a.w + c0 + e : a.w, v);
        cp_async16(usb + buf * kLsaCE + e, v && j > 0 ? uj + c0 + e : a.w, v && j > 0);
      }
    }
    cp_async_commit();
  };
  stage(blockIdx.x, 0);
  int buf = 0;
  for (size_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x, buf ^= 1) {
    const size_t c0 = ch * kLsaCE;
    const int len = (int)min((size_t)kLsaCE, N - c0);
    stage(ch + gridDim.x, buf ^ 1);  // its buffer was last read before the previous chunk's closing barrier
    cp_async_wait<1>();
    __syncthreads();  // this chunk's w and u_j visible to every warp
    const double2* ws = wsb + buf * kLsaCE;
    const double2* us = usb + buf * kLsaCE;
    for (int t = warp; t < nd * kLsaSplit; t += NW) {
      const int i = t / kLsaSplit, hs = t % kLsaSplit;
      const double2* ui = a.U + (size_t)i * N + c0;
      double2* acch = acc + hs * nslot;
      double2 sa = cmk(0.0, 0.0), sb = cmk(0.0, 0.0), ga = cmk(0.0, 0.0), gb = cmk(0.0, 0.0);
#pragma unroll kLsaUnroll
      for (int q = 0; q < PER; ++q) {
        const int e = (hs * PER + q) * 32 + lane;
        const double2 v = e < len ? __ldg(ui + e) : cmk(0.0, 0.0);
        if (q & 1) {
          sb = cadd(sb, cconjmul(v, ws[e]));
          gb = cadd(gb, cconjmul(us[e], v));
        } else {
          sa = cadd(sa, cconjmul(v, ws[e]));
          ga = cadd(ga, cconjmul(us[e], v));
        }
      }
      double2 s_ = lsa_warp_sum(cadd(sa, sb));
      double2 g_ = (i < j) ? lsa_warp_sum(cadd(ga, gb)) : cmk(0.0, 0.0);
      if (lane == 0) {
        acch[i] = cadd(acch[i], s_);
        if (i < j) acch[kLsaMaxJ + 1 + i] = cadd(acch[kLsaMaxJ + 1 + i], g_);
      }
    }
    __syncthreads();  // every warp done with this chunk's buffers before they are refilled
  }
  cp_async_wait<0>();
  __syncthreads();
  for (int q = threadIdx.x; q < nslot; q += kLsaBD) {
    const bool used = q < nd || (q >= kLsaMaxJ + 1 && q < kLsaMaxJ + 1 + j);
    if (used) {
      double2 v = acc[q];
#pragma unroll
      for (int h = 1; h < kLsaSplit; ++h) v = cadd(v, acc[h * nslot + q]);
      a.partials[(size_t)(a.part_offset + blockIdx.x) * nslot + q] = v;
    }
  }
  if (a.partial_only) return;
  if (!lsa_last_block(a.counter)) return;
  lsa_dots_finish(a, j, gridDim.x, sh_s, sh_lj, hsm);
  if (threadIdx.x == 0) *a.counter = 0u;
}

// ---------------------------------------------------------------------------
// pass 1 on the Blackwell bulk-copy engine (HD_LSA_TMA=1; default: k_lsa_dots).
// One CTA per SM, 8 warps.  The CTA's chunks of w and u_j (kTCE elements) go
// through a 3-deep ring of cp.async.bulk copies issued by thread 0 and
// completed on mbarriers; every warp streams its own items -- (chunk, vector)
// pairs t = c (j+1) + i, dealt round-robin over the warps so any j splits
// evenly -- through its own 2-stage ring of bulk copies of u_i's chunk.  No
// register staging and no CTA barrier in the stream: up to 3 chunks x 8 warps
// of copies are in flight per SM, what the DRAM latency needs at this per-SM
// share of the bandwidth.  A w / u_j buffer is refilled once all 8 warps have
// left its chunk (an "empty" mbarrier of count 8).  Per-warp accumulators,
// summed over the warps in fixed order at the end (deterministic).
// Measured at C5: both passes 48.6 ms per solve against 48.3 ms with the
// register-streaming pass 1 -- the stream was not short of bytes in flight.
// ---------------------------------------------------------------------------
constexpr int kTCE = 512;   // chunk elements (8 KB)
constexpr int kTNW = 8;     // warps per CTA
constexpr int kTWU = 3;     // w / u_j chunk buffers
constexpr int kTST = 2;     // u_i ring stages per warp

__host__ __device__ constexpr size_t lsa_tma_smem() {
  return sizeof(double2) * ((size_t)2 * kTWU * kTCE + (size_t)kTNW * kTST * kTCE + (size_t)kTNW * 2 * (kLsaMaxJ + 1)) +
         sizeof(unsigned long long) * (2 * kTWU + kTNW * kTST);
}

__device__ __forceinline__ unsigned tma_sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void tma_mbar_init(unsigned long long* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tma_sa(b)), "r"(count));
}
__device__ __forceinline__ void tma_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tma_sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tma_sa(b)) : "memory");
}
__device__ __forceinline__ void tma_wait(unsigned long long* b, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(tma_sa(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_g2s(void* smem, const void* g, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tma_sa(smem)),
               "l"(g), "r"(bytes), "r"(tma_sa(b))
               : "memory");
}

__global__ void __launch_bounds__(kTNW * 32, 1) k_lsa_dots_tma(LsaArgs a) {
  extern __shared__ __align__(128) double2 dsm[];
  double2* wub = dsm;                                   // [kTWU][2][kTCE]: w chunk, u_j chunk
  double2* ring = wub + 2 * kTWU * kTCE;                // [kTNW][kTST][kTCE]
  double2* acc = ring + kTNW * kTST * kTCE;             // [kTNW][2][kLsaMaxJ+1]: s_i, G_ji
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(acc + kTNW * 2 * (kLsaMaxJ + 1));
  unsigned long long* full_wu = bar;                    // [kTWU]
  unsigned long long* empty_wu = bar + kTWU;            // [kTWU], count kTNW
  unsigned long long* full_r = bar + 2 * kTWU;          // [kTNW][kTST]
  __shared__ double2 sh_s[kLsaMaxJ + 1];
  __shared__ double2 sh_lj[kLsaMaxJ];
  __shared__ double2 hsm[kLsaMaxJ + 1];
  if (a.done && *((volatile const int*)a.done)) return;
  const int j = a.dj ? *a.dj : a.j;
  const int nd = j + 1;
  const int nslot = 2 * kLsaMaxJ + 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t N = a.N;
  const double2* uj = a.U + (size_t)j * N;
  const size_t nchunks = (N + kTCE - 1) / kTCE;
  const int nch = nchunks > blockIdx.x ? (int)((nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
  auto chunk0 = [&](int c) { return ((size_t)blockIdx.x + (size_t)c * gridDim.x) * kTCE; };
  auto chunk_len = [&](int c) { return (int)min((size_t)kTCE, N - chunk0(c)); };
  for (int q = threadIdx.x; q < kTNW * 2 * (kLsaMaxJ + 1); q += blockDim.x) acc[q] = cmk(0.0, 0.0);
  if (threadIdx.x == 0) {
    for (int b = 0; b < kTWU; ++b) {
      tma_mbar_init(&full_wu[b], 1);
      tma_mbar_init(&empty_wu[b], kTNW);
    }
    for (int r = 0; r < kTNW * kTST; ++r) tma_mbar_init(&full_r[r], 1);
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  auto load_wu = [&](int c) {  // thread 0: chunk c of w and u_j into buffer c % kTWU
    const int b = c % kTWU, len = chunk_len(c);
    const unsigned bytes = (unsigned)len * 16u;
    tma_expect(&full_wu[b], (j > 0 ? 2u : 1u) * bytes);
    tma_g2s(wub + (size_t)(2 * b) * kTCE, a.w + chunk0(c), bytes, &full_wu[b]);
    if (j > 0) tma_g2s(wub + (size_t)(2 * b + 1) * kTCE, uj + chunk0(c), bytes, &full_wu[b]);
  };
  if (threadIdx.x == 0)
    for (int c = 0; c < kTWU && c < nch; ++c) load_wu(c);
  // this warp's items t = warp + k kTNW < nch nd: chunk t / nd, vector t % nd
  const long nitems = (long)nch * nd;
  auto load_item = [&](long t, int slot) {  // lane 0: u_i's chunk into the warp's ring slot
    const int c = (int)(t / nd), i = (int)(t % nd);
    const unsigned bytes = (unsigned)chunk_len(c) * 16u;
    unsigned long long* fb = &full_r[warp * kTST + slot];
    tma_expect(fb, bytes);
    tma_g2s(ring + (size_t)(warp * kTST + slot) * kTCE, a.U + (size_t)i * N + chunk0(c), bytes, fb);
  };
  if (lane == 0)
    for (int s2 = 0; s2 < kTST; ++s2) {
      const long t = warp + (long)s2 * kTNW;
      if (t < nitems) load_item(t, s2);
    }
  double2* myacc = acc + (size_t)warp * 2 * (kLsaMaxJ + 1);
  int left = 0;  // chunks this warp has left (arrived on their empty barrier)
  // arrive on the chunks before c_excl (after their load landed, so the arrival
  // counts toward that use of the buffer even when the warp had no item in the
  // chunk); warp 0 then refills each buffer once all warps have left it
  auto leave_until = [&](int c_excl) {
    for (; left < c_excl; ++left) {
      tma_wait(&full_wu[left % kTWU], (unsigned)((left / kTWU) & 1));
      __syncwarp();
      if (lane == 0) tma_arrive(&empty_wu[left % kTWU]);
      if (warp == 0 && lane == 0 && left + kTWU < nch) {
        tma_wait(&empty_wu[left % kTWU], (unsigned)((left / kTWU) & 1));
        load_wu(left + kTWU);
      }
    }
  };
  long k = 0;
  // the chunk's w and u_j stay in registers while the warp's items stay in that
  // chunk (consecutive items t, t + 8, ... are vectors i, i + 8, ... of one chunk),
  // so a vector costs one shared-memory read per element
  constexpr int PL = kTCE / 32;
  double2 wr[PL], ur[PL];
  int cur = -1;
  for (long t = warp; t < nitems; t += kTNW, ++k) {
    const int c = (int)(t / nd), i = (int)(t % nd);
    leave_until(c);
    const int slot = (int)(k % kTST);
    const int len = chunk_len(c);
    if (c != cur) {
      tma_wait(&full_wu[c % kTWU], (unsigned)((c / kTWU) & 1));
      const double2* ws = wub + (size_t)(2 * (c % kTWU)) * kTCE;
      const double2* us = ws + kTCE;
#pragma unroll
      for (int q = 0; q < PL; ++q) {
        const int e = q * 32 + lane;
        wr[q] = e < len ? ws[e] : cmk(0.0, 0.0);
        ur[q] = (e < len && j > 0) ? us[e] : cmk(0.0, 0.0);
      }
      cur = c;
    }
    tma_wait(&full_r[warp * kTST + slot], (unsigned)((k / kTST) & 1));
    const double2* ui = ring + (size_t)(warp * kTST + slot) * kTCE;
    double2 sa = cmk(0.0, 0.0), sb = cmk(0.0, 0.0), ga = cmk(0.0, 0.0), gb = cmk(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < PL; ++q) {
      const int e = q * 32 + lane;
      const double2 v = e < len ? ui[e] : cmk(0.0, 0.0);
      if (q & 1) {
        sb = cadd(sb, cconjmul(v, wr[q]));
        gb = cadd(gb, cconjmul(ur[q], v));
      } else {
        sa = cadd(sa, cconjmul(v, wr[q]));
        ga = cadd(ga, cconjmul(ur[q], v));
      }
    }
    const double2 s_ = lsa_warp_sum(cadd(sa, sb));
    const double2 g_ = lsa_warp_sum(cadd(ga, gb));
    __syncwarp();  // every lane done with the slot before it is refilled
    if (lane == 0) {
      myacc[i] = cadd(myacc[i], s_);
      if (i < j) myacc[kLsaMaxJ + 1 + i] = cadd(myacc[kLsaMaxJ + 1 + i], g_);
      const long tn = t + (long)kTST * kTNW;
      if (tn < nitems) load_item(tn, slot);
    }
  }
  leave_until(nch);
  __syncthreads();
  // CTA partials: the warps' accumulators in warp order
  for (int q = threadIdx.x; q < nslot; q += blockDim.x) {
    const bool used = q < nd || (q >= kLsaMaxJ + 1 && q < kLsaMaxJ + 1 + j);
    if (used) {
      double2 v = cmk(0.0, 0.0);
      for (int w2 = 0; w2 < kTNW; ++w2) v = cadd(v, acc[(size_t)w2 * 2 * (kLsaMaxJ + 1) + q]);
      a.partials[(size_t)(a.part_offset + blockIdx.x) * nslot + q] = v;
    }
  }
  if (a.partial_only) return;
  if (!lsa_last_block(a.counter)) return;
  lsa_dots_finish(a, j, gridDim.x, sh_s, sh_lj, hsm);
  if (threadIdx.x == 0) *a.counter = 0u;
}

// ---- totals, Gram row j, triangular solve (I + L) h = s (one CTA) ----------
__device__ void lsa_dots_finish(const LsaArgs& a, int j, int nparts, double2* sh_s, double2* sh_lj, double2* hsm) {
  constexpr int NW = kLsaBD / 32;
  const int nd = j + 1;
  const int nslot = 2 * kLsaMaxJ + 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double sj = a.sig[j];
  for (int q = warp; q < nd; q += NW) {
    const double2 s = lsa_collect(a.partials, nslot, q, nparts);
    if (lane == 0) sh_s[q] = cscale(a.sig[q] * sj, s);
  }
  for (int q = warp; q < j; q += NW) {
    const double2 gsum = lsa_collect(a.partials, nslot, kLsaMaxJ + 1 + q, nparts);
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
    double2* hs = hsm;
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
}

// ---------------------------------------------------------------------------
// pass 1 as a tall-skinny FP64 tensor-core GEMM fed by the bulk-copy engine
// (HD_LSA_MMA=1).  All dots of an iteration are one contraction over the N
// elements,
//
//   [ s_i , G_ji ] = sum_e  conj(u_i[e]) w[e] ,  conj(u_j[e]) u_i[e]      (i = 0 .. j),
//
// i.e. C = A B with A the basis as a real (j+1) x 2N matrix (exactly its memory
// layout) and B a 2N x 4 matrix built from w and u_j.  mma.sync.m8n8k4.f64
// (DMMA) takes 8 basis vectors x 4 values of K per instruction: lane
// (r = lane/4, q = lane%4) feeds A[r][q] and B[q][r], and the 8 x 8 accumulator
// (2 doubles per lane per group of 8 vectors) stays in registers over the
// warp's whole share of N: no per-chunk reduction and no block barrier in the
// loop.  The contraction index may be permuted freely as long as A and B
// agree, so a lane takes one whole complex element (16 bytes) of its vector
// and feeds its real part to one DMMA step and its imaginary part to the next:
//   "re" step B column r: wr, wi, ur, -ui      "im" step: wi, -wr, ui, ur     (r = 0..3; 4..7 zero).
// Every warp is its own pipeline: a unit is (tile of kMmaTE elements, group of
// 8 vectors) = an 8-row box of the basis seen as a 2D tensor (2N doubles x
// vectors), fetched by ONE cp.async.bulk.tensor (UTMALDG) into a kMmaST-deep
// ring completed on mbarriers; elements past N and vectors past the allocation
// are zero-filled.  The data in flight lives in shared memory (kMmaST x 8 KB
// per warp), not in registers.
// The (w, u_j) tile arrives by two cp.async.bulk copies; its fragments go to
// registers at once, so one buffer suffices.  The per-CTA and grid reductions
// at the end are the fixed-order ones of k_lsa_dots (same partial slots, same
// finishing step).
//
// Measured at C5 (round 2): correct (tests/test_gpu_switches.py) and SLOWER:
// pass 1 takes 32.5 ms per solve against 24.8 ms for k_lsa_dots (the solve
// 94.6 vs 88.7 ms).  History: fragments loaded straight into registers (one
// 8-warp CTA per SM at 240+ registers, 8 KB in flight per warp): 106-116 ms;
// this ring with eight 512-byte cp.async.bulk rows per unit: 106.7 ms; one
// 4 KB tensor box per unit: 97.6 ms; 8 KB boxes (kMmaTE = 64): 94.6 ms.  With
// the DMMAs replaced by two FMAs the pipeline alone streams at 4.6 TB/s for
// 4 KB and 8 KB boxes alike, below k_lsa_dots' 5.5 TB/s: boxes of eight rows
// from eight vectors (eight DRAM pages) are what the copy engine is slow on,
// and that shape is what the DMMA operand layout asks for.  Opt-in.
// ---------------------------------------------------------------------------
#ifndef HD_MMA_TE
#define HD_MMA_TE 64
#endif
#ifndef HD_MMA_ST
#define HD_MMA_ST 3
#endif
constexpr int kMmaTE = HD_MMA_TE;               // complex elements per tile (1 KB per vector)
constexpr int kMmaNG = (kLsaMaxJ + 1 + 7) / 8;  // groups of 8 basis vectors
constexpr int kMmaST = HD_MMA_ST;               // ring stages per warp
constexpr int kMmaRS = kMmaTE * 16;             // row pitch in shared memory (bytes): a dense tensor-copy box
constexpr int kMmaWarp = kMmaST * 8 * kMmaRS + 2 * kMmaTE * 16 + 128;  // ring + the (w, u_j) tile + barriers
constexpr size_t lsa_mma_smem() { return (size_t)(kLsaBD / 32) * kMmaWarp + 128; }

__device__ __forceinline__ void lsa_dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 lsa_lds16(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}

__global__ void __launch_bounds__(kLsaBD, 1) k_lsa_dots_mma(LsaArgs a, const __grid_constant__ CUtensorMap tmU) {
  constexpr int NW = kLsaBD / 32;
  constexpr int NT = kMmaTE / 4;  // element quads per tile
  extern __shared__ __align__(128) unsigned char msm_raw[];
  __shared__ double2 acc[2 * kLsaMaxJ + 2];  // [0..j]: s_i ; [kLsaMaxJ+1 ..]: G_ji  (k_lsa_dots' slots)
  __shared__ double2 sh_s[kLsaMaxJ + 1];
  __shared__ double2 sh_lj[kLsaMaxJ];
  __shared__ double2 hsm[kLsaMaxJ + 1];
  if (a.done && *((volatile const int*)a.done)) return;
  const int j = a.dj ? *a.dj : a.j;
  const int nd = j + 1, ng = (nd + 7) >> 3;
  const int nslot = 2 * kLsaMaxJ + 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = lane >> 2, q = lane & 3;
  for (int t = threadIdx.x; t < nslot; t += kLsaBD) acc[t] = cmk(0.0, 0.0);
  const size_t N = a.N;
  const double2* uj = a.U + (size_t)j * N;
  unsigned char* wbase = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(msm_raw) + 127) & ~uintptr_t(127)) +
                         (size_t)warp * kMmaWarp;
  unsigned char* bbuf = wbase + kMmaST * 8 * kMmaRS;                             // [w tile | u_j tile]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(bbuf + 2 * kMmaTE * 16);  // [kMmaST]
  unsigned long long* bfull = full + kMmaST;                                     // the (w, u_j) tile's barrier
  if (lane == 0) {
    for (int s = 0; s < kMmaST; ++s) tma_mbar_init(&full[s], 1);
    tma_mbar_init(&bfull[0], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  const size_t ntiles = (N + kMmaTE - 1) / kMmaTE;
  const size_t gw = (size_t)blockIdx.x * NW + warp, W = (size_t)gridDim.x * NW;
  const int nt = gw < ntiles ? (int)((ntiles - gw + W - 1) / W) : 0;  // this warp's tiles gw, gw + W, ...
  const int nunits = nt * ng;
  auto tile_bytes = [&](int k) {  // bytes of tile k of a vector (the last tile of the grid may be short)
    const size_t e0 = (gw + (size_t)k * W) * kMmaTE;
    return (unsigned)(min((size_t)kMmaTE, N - e0) * 16);
  };
  auto issue_unit = [&](int u) {  // lane 0: unit u = (tile u / ng, group u % ng) as one 8-row tensor-copy box
    const int k = u / ng, g = u - k * ng, slot = u % kMmaST;
    const size_t e0 = (gw + (size_t)k * W) * kMmaTE;
    if (lane == 0) {
      tma_expect(&full[slot], 8 * kMmaRS);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              tma_sa(wbase + (size_t)slot * 8 * kMmaRS)),
          "l"(&tmU), "r"((int)(2 * e0)), "r"(8 * g), "r"(tma_sa(&full[slot]))
          : "memory");
    }
  };
  auto issue_b = [&](int k) {  // lanes 0, 1: the w and u_j tiles of tile k (its fragments go to registers at once)
    const size_t e0 = (gw + (size_t)k * W) * kMmaTE;
    const unsigned bytes = tile_bytes(k);
    if (lane == 0) tma_expect(&bfull[0], 2 * bytes);
    if (lane == 0) tma_g2s(bbuf, a.w + e0, bytes, &bfull[0]);
    if (lane == 1) tma_g2s(bbuf + kMmaTE * 16, uj + e0, bytes, &bfull[0]);
  };
  if (lane == 0)
    for (int u = 0; u < kMmaST && u < nunits; ++u) issue_unit(u);
  if (lane < 2 && nt > 0) issue_b(0);
  double C[kMmaNG][2];
#pragma unroll
  for (int g = 0; g < kMmaNG; ++g) C[g][0] = C[g][1] = 0.0;
  const bool buse = r < 4;
  const unsigned boff = (unsigned)((buse ? (r >> 1) : 0) * kMmaTE * 16 + q * 16);  // this lane's element of quad 0 in a (w | u_j) tile
  const unsigned aoff = (unsigned)(r * kMmaRS + q * 16);              // ... in a ring stage
  int uc = 0, slot = 0;
  unsigned ph = 0;
  for (int k = 0; k < nt; ++k) {
    const size_t e0 = (gw + (size_t)k * W) * kMmaTE + q;
    tma_wait(&bfull[0], (unsigned)(k & 1));
    double bre[NT], bim[NT];
    const unsigned bb = tma_sa(bbuf) + boff;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      double2 v = lsa_lds16(bb + t * 64);
      if (!buse || e0 + 4 * t >= N) v = cmk(0.0, 0.0);  // columns 4..7 and the tail of the last tile
      bre[t] = r == 0 ? v.x : (r == 1 ? v.y : (r == 2 ? v.x : -v.y));
      bim[t] = r == 0 ? v.y : (r == 1 ? -v.x : (r == 2 ? v.y : v.x));
    }
    __syncwarp();
    if (lane < 2 && k + 1 < nt) issue_b(k + 1);
#pragma unroll
    for (int g = 0; g < kMmaNG; ++g) {
      if (g < ng) {  // warp-uniform
        tma_wait(&full[slot], ph);
        const unsigned ab = tma_sa(wbase) + (unsigned)slot * 8 * kMmaRS + aoff;
        double T[2] = {0.0, 0.0};  // second chain: halves the dependent DMMA chain on C[g]
        const bool row_ok = 8 * g + r <= j;  // rows beyond the basis hold other memory: mask them
#pragma unroll
        for (int h = 0; h < NT; h += 8) {
          double2 av[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            av[t] = lsa_lds16(ab + (h + t) * 64);
            if (!row_ok) av[t] = cmk(0.0, 0.0);
          }
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            lsa_dmma(C[g], av[t].x, bre[h + t]);
            lsa_dmma(T, av[t].y, bim[h + t]);
          }
        }
        C[g][0] += T[0];
        C[g][1] += T[1];
        __syncwarp();  // every lane has read the stage before it is refilled
        if (lane == 0 && uc + kMmaST < nunits) issue_unit(uc + kMmaST);
        ++uc;
        if (++slot == kMmaST) {
          slot = 0;
          ph ^= 1u;
        }
      }
    }
  }
  // CTA sums in warp order (fixed => deterministic): C[g] of lane (r, q): q = 0 -> s_i, q = 1 -> G_ji, i = 8 g + r
  __syncthreads();
  for (int wq = 0; wq < NW; ++wq) {
    if (warp == wq && q < 2) {
#pragma unroll
      for (int g = 0; g < kMmaNG; ++g) {
        const int i = 8 * g + r;
        if (g < ng && i <= j) {
          if (q == 0) acc[i] = cadd(acc[i], cmk(C[g][0], C[g][1]));
          else if (i < j) acc[kLsaMaxJ + 1 + i] = cadd(acc[kLsaMaxJ + 1 + i], cmk(C[g][0], C[g][1]));
        }
      }
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < nslot; t += kLsaBD) {
    const bool used = t < nd || (t >= kLsaMaxJ + 1 && t < kLsaMaxJ + 1 + j);
    if (used) a.partials[(size_t)(a.part_offset + blockIdx.x) * nslot + t] = acc[t];
  }
  if (a.partial_only) return;
  if (!lsa_last_block(a.counter)) return;
  lsa_dots_finish(a, j, gridDim.x, sh_s, sh_lj, hsm);
  if (threadIdx.x == 0) *a.counter = 0u;
}

// row slabs: combine the partials of all slabs (nparts CTA slots, slab order)
__global__ void __launch_bounds__(kLsaBD) k_lsa_dots_finish(LsaArgs a, int nparts) {
  __shared__ double2 sh_s[kLsaMaxJ + 1];
  __shared__ double2 sh_lj[kLsaMaxJ];
  __shared__ double2 hsm[kLsaMaxJ + 1];
  if (a.done && *((volatile const int*)a.done)) return;
  const int j = a.dj ? *a.dj : a.j;
  lsa_dots_finish(a, j, nparts, sh_s, sh_lj, hsm);
}

// ---------------------------------------------------------------------------
// pass 2: u_{j+1} = sigma_j w - sum_i c_i u_i,  hnew = ||u_{j+1}||, Givens
// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 lsa_cdiv(double2 a, double2 b) { return cmul(a, cinv(b)); }

// mode 0: u_{j+1} = sigma_j w - sum_{i<=j} c_i u_i (+ norm) and, for j >= 1, the
// lagged iterate x_{j-1} = x0 + sum_{i<j} c'_i u_i (src/linalg.cpp:78-80);
// mode 1 (budget exhausted): only x_j = x0 + sum_{i<=j} c'_i u_i.
__global__ void __launch_bounds__(kLsaBD) k_lsa_update(LsaArgs a) {
  constexpr int NW = kLsaBD / 32;
  __shared__ double2 sh_c[kLsaMaxJ + 1];
  __shared__ double2 sh_x[kLsaMaxJ + 1];
  __shared__ double red[NW];
  if (a.done && *((volatile const int*)a.done)) return;
  const int j = a.dj ? *a.dj : a.j;
  const bool upd = a.mode == 0;
  const bool iter = a.mode == 1 || j >= 1;
  const int mi = a.mode == 1 ? j + 1 : j;      // iterate terms
  const int nv = upd ? j + 1 : mi;             // vectors streamed
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = threadIdx.x; q <= j; q += kLsaBD) {
    sh_c[q] = upd ? __ldcg(&a.ch[q]) : cmk(0.0, 0.0);
    sh_x[q] = (iter && q < mi) ? __ldcg(&a.cx[q]) : cmk(0.0, 0.0);
  }
  __syncthreads();
  const double sj = upd ? a.sig[j] : 0.0;
  const size_t N = a.N;
  const size_t tile = (size_t)kLsaBD * kLsaTE;
  double2* un = a.Uw + (size_t)(j + 1) * N;
  double nrm = 0.0;
  const size_t ntiles = (N + tile - 1) / tile;
  for (size_t tt = blockIdx.x; tt < ntiles; tt += gridDim.x) {
    const size_t t0 = (a.rev ? ntiles - 1 - tt : tt) * tile;
    double2 wv[kLsaTE], xv[kLsaTE];
#pragma unroll
    for (int u = 0; u < kLsaTE; ++u) {
      const size_t e = t0 + (size_t)u * kLsaBD + threadIdx.x;
      wv[u] = (upd && e < N) ? cscale(sj, ld_stream(a.w + e)) : cmk(0.0, 0.0);
      xv[u] = (iter && e < N) ? ld_stream(a.x0 + e) : cmk(0.0, 0.0);
    }
    // kLsaVPS vectors per step: 4 kLsaVPS outstanding 16-B loads per thread; the
    // products are accumulated in vector order (as two per step did)
    for (int i = 0; i < nv; i += kLsaVPS) {
      double2 v[kLsaVPS][kLsaTE];
#pragma unroll
      for (int b = 0; b < kLsaVPS; ++b) {
        const double2* ub = a.U + (size_t)(i + b) * N;
#pragma unroll
        for (int u = 0; u < kLsaTE; ++u) {
          const size_t e = t0 + (size_t)u * kLsaBD + threadIdx.x;
          v[b][u] = (i + b < nv && e < N) ? __ldg(ub + e) : cmk(0.0, 0.0);
        }
      }
#pragma unroll
      for (int b = 0; b < kLsaVPS; ++b) {
        if (i + b >= nv) break;
        const double2 cb = sh_c[i + b], db = sh_x[i + b];
#pragma unroll
        for (int u = 0; u < kLsaTE; ++u) {
          if (upd) wv[u] = csub(wv[u], cmul(cb, v[b][u]));
          if (iter) xv[u] = cfma(db, v[b][u], xv[u]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kLsaTE; ++u) {
      const size_t e = t0 + (size_t)u * kLsaBD + threadIdx.x;
      if (e < N) {
        if (upd) {
          un[e] = wv[u];
          nrm += cnorm2(wv[u]);
        }
        if (iter) a.x[e] = xv[u];
      }
    }
  }
  if (!upd) return;
  // CTA partial of ||u_{j+1}||^2
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nrm += __shfl_down_sync(0xffffffffu, nrm, o);
  if (lane == 0) red[warp] = nrm;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < NW; ++q) s += red[q];
    a.partials[a.part_offset + blockIdx.x] = cmk(s, 0.0);
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
  const int j = (a.dj ? *a.dj : a.j) - a.jlag;
  if (j < 0) return;
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
  int breakdown;  // side-branch monitor: Krylov breakdown, the host monitors x_{iters-1}
  int nonfinite;  // NaN/Inf residual or hnew: stopped, the host reports an error
  double hprev;   // row slabs: hnew of the previous iteration (the body's Givens runs last)
};

// Row-slab loop control, last kernel of the slab graph body (after the monitor
// of x_{j-1} and the Givens of column j): the host loop's decisions of
// run_solve_slabs on the device -- record rr(x_{j-1}), stop on tolerance, on a
// non-finite value or on the breakdown of iteration j-1, stop at the budget,
// else step to j+1.  Every rank computes the same scalars (slab-order sums),
// so every rank takes the same decision.
__global__ void k_slab_loop_step(LoopState* s, const double* dres, double* res_hist, double tol, int maxit) {
  if (s->done) return;
  const int j = s->j;
  if (j >= 1) {
    const double rr = dres[0];
    res_hist[j - 1] = rr;
    if (!isfinite(rr) || !isfinite(s->hprev)) {
      s->nonfinite = 1;
      s->done = 1;
      s->iters = j;
      return;
    }
    if (rr <= tol || s->hprev < 1e-300) {
      s->conv = rr <= tol;
      s->done = 1;
      s->iters = j;
      return;
    }
  }
  s->hprev = dres[1];
  if (j + 1 >= maxit) {
    s->done = 1;
    s->need_tail = 1;
    s->iters = maxit;
    return;
  }
  s->j = j + 1;
}

// After the monitor of x_{j-1} (src/linalg.cpp:82-88): record the residual,
// stop on tolerance or Krylov breakdown of the previous step.
__device__ __forceinline__ void loop_check(LoopState* s, const double* dres, double* res_hist, double tol,
                                           cudaGraphConditionalHandle h) {
  if (s->done) return;
  const int j = s->j;
  if (j < 1) return;
  const double rr = dres[0];
  res_hist[j - 1] = rr;
  if (!isfinite(rr) || !isfinite(dres[1])) {  // poisoned solve: stop instead of running to maxit
    s->nonfinite = 1;
    s->done = 1;
    s->iters = j;
    cudaGraphSetConditional(h, 0);
    return;
  }
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

__global__ void k_loop_check(LoopState* s, const double* dres, double* res_hist, double tol,
                             cudaGraphConditionalHandle h) {
  loop_check(s, dres, res_hist, tol, h);
}

// Side-branch monitor (HD_MON_SIDE): body j monitors x_{j-2} concurrently with
// op(u_j); x_{j-2} is still in place because pass 2 of body j (which writes
// x_{j-1}) runs after the branch joins, and exits early once done is set.
__global__ void k_loop_check_lag2(LoopState* s, const double* dres, double* res_hist, double tol,
                                  cudaGraphConditionalHandle h) {
  if (s->done) return;
  const int j = s->j;
  if (j < 2) return;
  const double rr = dres[0];
  res_hist[j - 2] = rr;
  if (rr <= tol) {
    s->conv = 1;
    s->done = 1;
    s->iters = j - 1;
    cudaGraphSetConditional(h, 0);
  }
}

// Side-branch monitor: breakdown of iteration j-1 (hnew from its Givens) stops
// the loop with x_{j-1} formed but not yet monitored (the host does that).
__global__ void k_loop_breakdown(LoopState* s, const double* dres, cudaGraphConditionalHandle h) {
  if (s->done) return;
  const int j = s->j;
  if (j >= 1 && dres[1] < 1e-300) {
    s->done = 1;
    s->breakdown = 1;
    s->iters = j;
    cudaGraphSetConditional(h, 0);
  }
}

__device__ __forceinline__ void loop_next(LoopState* s, int maxit, cudaGraphConditionalHandle h) {
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

__global__ void k_loop_next(LoopState* s, int maxit, cudaGraphConditionalHandle h) {
  loop_next(s, maxit, h);
}

// The graph body's tail in one launch: monitor scaling (raw norm / ||f||),
// convergence / breakdown check of x_{j-1}, and the step to j+1.
__global__ void k_loop_step(LoopState* s, double* dres, double* res_hist, double tol, int maxit,
                            cudaGraphConditionalHandle h) {
  const double f = dres[3];
  dres[0] = dres[0] / (f > 0.0 ? f : 1.0);
  loop_check(s, dres, res_hist, tol, h);
  loop_next(s, maxit, h);
}

}  // namespace hd
