// Row-slab decomposition: transports (local copies, virtual ranks, NCCL), slab operators, the split E solve, the slab GMRES loop.
// (part of solver.cu, a single translation unit: included in order)
#pragma once

namespace hd {

// ===========================================================================
// Row-slab decomposition (plan: paper_2010_10232_b200/slabs.py)
//
// The 2D grid is cut into S bands of iy rows.  Every distributed level vector
// is held per slab with H halo rows above and below ([r0-H, r1+H) of the
// global rows); kernels address it through a "virtual" pointer shifted by the
// slab origin, so they index global rows and read the halo rows where a
// stencil or transfer crosses the slab edge.  Communication happens exactly
// where the multi-GPU program communicates:
//   * halo exchange before every apply / transfer on a distributed level
//     (here: device copies between the slabs' buffers; multi-GPU: neighbour
//     send/recv of H rows);
//   * the gather level's restricted rhs and the deflation coarse vector are
//     written into one global buffer (multi-GPU: allgather), the levels below
//     the gather level and the E solve run once (multi-GPU: redundantly);
//   * reductions: each slab writes its partial sums (norms: a raw sum of
//     squares; Arnoldi: its CTAs' partials at its own offset) and one kernel
//     combines them in slab order (multi-GPU: allreduce).
// On one GPU the slabs run in sequence on one stream (no kernel waits on
// another); the result is the single-domain solve up to the association of
// the sums, which tests/test_gpu_parity.py checks.
// ===========================================================================
struct SlabLevel {
  int n = 0, b = 0, H = 0;
  bool dist = false;
  std::vector<int> bounds;  // S+1 row boundaries (distributed levels)
};

// NCCL, resolved at run time (dlopen) so the library loads without it; only
// the multi-process slab program (hd_create_dist) needs it.
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  if (api.h) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw Error(HD_ERR_INVALID, "multi-process row slabs need NCCL (libnccl.so.2 not found)");
  auto sym = [&](const char* n) {
    void* f = dlsym(h, n);
    if (!f) throw Error(HD_ERR_INVALID, std::string("NCCL symbol missing: ") + n);
    return f;
  };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
  api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
  api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  api.h = h;
  return api;
}

#define CKN(x)                                                                                    \
  do {                                                                                            \
    ncclResult_t e_ = (x);                                                                        \
    if (e_ != ncclSuccess) throw Error(HD_ERR_CUDA, std::string(#x) + ": " + nccl().GetErrorString(e_)); \
  } while (0)

// A point-to-point transfer of the slab program (halo rows).
struct SlabPost {
  const double2* src;
  double2* dst;
  size_t count;  // double2 elements
  int peer;      // the other slab
};

struct hd_slabs {
  int S = 0, g = 0, Gs = 0;
  // transport.  nranks == 1: every slab lives in this process (one GPU, the
  // exchanges are device copies); nranks > 1: this process owns slab `rank`
  // (one process per GPU) and the exchanges are NCCL send/recv, the shared
  // coarse vectors NCCL broadcasts and the reduction partials NCCL allgathers.
  // vranks (HD_SLAB_VRANKS=1, one process): every slab is its own virtual
  // rank and halo rows go through the same posted send/recv records as the
  // NCCL path, matched and copied at group end -- the offsets and sizes of
  // the multi-process program exercised on one GPU.
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  bool vranks = false;
  std::vector<int> mine;                        // slabs of this process
  std::vector<SlabPost> sends, recvs;           // posted in the current group (vranks)
  double2* red = nullptr;                       // S x nslot per-slab Arnoldi pass-1 sums
  // distributed E solve (plain fast diagonalisation): per-slab transform
  // buffers (one shared buffer when all slabs are local and not virtual
  // ranks) and all-to-all staging (pack -> send/recv -> unpack)
  bool dist_e = false;
  std::vector<double*> eT1, eT2;                // [slab] 2 planes x nc^2
  std::vector<double*> esend, erecv;            // [slab] staging, 2 planes x nc x own columns
  // graph-resident iteration (HD_GRAPH != 0): one captured body per (maxit),
  // launched once per iteration with the iteration index in device memory
  int* dj = nullptr;                            // device iteration index
  int* hj = nullptr;                            // pinned mirror
  cudaGraphExec_t body = nullptr;
  int body_maxit = -1;
  double body_tol = -1.0;
  unsigned body_epoch = ~0u;  // hd_ctx::buf_epoch the body graph captured
  const int* done = nullptr;  // while capturing the body: the loop state's done flag (early exit)
  long body_delta[6] = {0, 0, 0, 0, 0, 0};      // counters one body adds (matvecs .. lib_calls)
  std::vector<SlabLevel> lv;                    // MG levels
  std::vector<std::vector<double2*>> X, Y, B, R;  // [level][slab], levels < g
  std::vector<int> cur;                         // ping-pong state of X/Y per level
  // fine-level vectors, per slab, halo'd with H = lv[0].H
  std::vector<double2*> f, w, t1, t2, t3, x, x0, rhsp, vin;
  std::vector<double2*> V;                      // per slab: basis u_0..u_maxit (own rows, flat)
  int maxit = -1;
  double* slots = nullptr;                      // per-slab raw sums
  double2* parts = nullptr;                     // S x Gs Arnoldi partials
};

__global__ void k_slab_sumsq(const double2* __restrict__ x, size_t N, RedOut red) {
  __shared__ double2 scratch[32];
  double acc = 0.0;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < N; g += (size_t)gridDim.x * blockDim.x)
    acc += cnorm2(x[g]);
  double2 total;
  if (grid_sum2(cmk(acc, 0.0), red.partials, red.counter, scratch, &total)) *red.dst = total.x;
}

// norm = sqrt(sum of the slabs' raw sums, slab order) / scale -> dst (and cdst = (norm, 0))
__global__ void k_slab_norm(const double* slots, int S, const double* scale_src, double* dst, double2* cdst) {
  double s = 0.0;
  for (int i = 0; i < S; ++i) s += slots[i];
  double sc = 1.0;
  if (scale_src) sc = *scale_src > 0.0 ? *scale_src : 1.0;
  const double nrm = sqrt(s) / sc;
  *dst = nrm;
  if (cdst) *cdst = cmk(nrm, 0.0);
}

// Arnoldi pass 1 of one slab: its Gs CTA partials summed per used slot in CTA
// order (deterministic), so a process contributes one row of kLsaNslot sums
constexpr int kLsaNslot = 2 * kLsaMaxJ + 2;
__global__ void k_lsa_slab_reduce(const double2* __restrict__ parts, int Gs, int j, const int* dj,
                                  double2* __restrict__ out) {
  if (dj) j = *dj;
  for (int q = threadIdx.x; q < kLsaNslot; q += blockDim.x) {
    const bool used = q < j + 1 || (q >= kLsaMaxJ + 1 && q < kLsaMaxJ + 1 + j);
    double2 acc = cmk(0.0, 0.0);
    if (used)
      for (int b = 0; b < Gs; ++b) acc = cadd(acc, parts[(size_t)b * kLsaNslot + q]);
    out[q] = acc;
  }
}

static hd_slabs* slabs_of(hd_ctx* c) { return reinterpret_cast<hd_slabs*>(c->slabs); }
static inline bool is_local(const hd_slabs* sl, int s) { return sl->nranks == 1 || s == sl->rank; }

// virtual pointer of a halo'd slab buffer: global row r of the slab lives at v + r*n
static inline double2* vptr(double2* buf, int r0, int H, int n) {
  return buf - static_cast<ptrdiff_t>(r0 - H) * n;
}
static inline int own(const SlabLevel& L, int s) { return L.bounds[s + 1] - L.bounds[s]; }

// ---- transport -------------------------------------------------------------
// halo rows: slab s receives from a neighbour t.  Local pairs are device copies;
// remote pairs (other process, or a virtual rank) are posted send/recv.
static void xp_send(hd_ctx* c, const double2* src, size_t count, int from, int to) {
  hd_slabs* sl = slabs_of(c);
  if (sl->vranks) {
    sl->sends.push_back({src, nullptr, count, to});
    (void)from;
  } else {
    CKN(nccl().Send(src, 2 * count, ncclDouble, to, sl->comm, c->st));
  }
}
static void xp_recv(hd_ctx* c, double2* dst, size_t count, int from, int to) {
  hd_slabs* sl = slabs_of(c);
  if (sl->vranks) {
    sl->recvs.push_back({nullptr, dst, count, from});
    (void)to;
  } else {
    CKN(nccl().Recv(dst, 2 * count, ncclDouble, from, sl->comm, c->st));
  }
}
static bool remote_pairs(const hd_slabs* sl) { return sl->nranks > 1 || sl->vranks; }
static void xp_group_start(hd_ctx* c) {
  hd_slabs* sl = slabs_of(c);
  if (sl->nranks > 1) CKN(nccl().GroupStart());
  sl->sends.clear();
  sl->recvs.clear();
}
// vranks: the k-th send from slab a to slab b pairs with the k-th receive of b from a
static void xp_group_end(hd_ctx* c, const std::vector<int>& send_from, const std::vector<int>& recv_to) {
  hd_slabs* sl = slabs_of(c);
  if (sl->nranks > 1) {
    CKN(nccl().GroupEnd());
    return;
  }
  if (!sl->vranks) return;
  std::vector<bool> used(sl->sends.size(), false);
  for (size_t r = 0; r < sl->recvs.size(); ++r) {
    const SlabPost& rv = sl->recvs[r];
    bool found = false;
    for (size_t q = 0; q < sl->sends.size() && !found; ++q) {
      if (used[q] || send_from[q] != rv.peer || sl->sends[q].peer != recv_to[r]) continue;
      if (sl->sends[q].count != rv.count) throw Error(HD_ERR_INVALID, "slab transport: send/recv size mismatch");
      CK(cudaMemcpyAsync(rv.dst, sl->sends[q].src, rv.count * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
      used[q] = found = true;
    }
    if (!found) throw Error(HD_ERR_INVALID, "slab transport: receive without a matching send");
  }
  for (bool u : used)
    if (!u) throw Error(HD_ERR_INVALID, "slab transport: send without a matching receive");
}

// halo exchange of one distributed level vector (slab s <- neighbours' own rows)
static void slab_exchange(hd_ctx* c, const SlabLevel& L, const std::vector<double2*>& v) {
  hd_slabs* sl = slabs_of(c);
  const size_t row = static_cast<size_t>(L.n), hrows = static_cast<size_t>(L.H) * row;
  const bool remote = remote_pairs(sl);
  std::vector<int> send_from, recv_to;
  if (remote) xp_group_start(c);
  for (int s : sl->mine) {
    const size_t ownr = static_cast<size_t>(own(L, s));
    double2* top_halo = v[s];
    double2* bot_halo = v[s] + (L.H + ownr) * row;
    const double2* first_own = v[s] + hrows;
    const double2* last_own = v[s] + ownr * row;  // rows own-H .. own-1 (after the H halo rows)
    if (s > 0) {
      if (!remote && is_local(sl, s - 1)) {
        CK(cudaMemcpyAsync(top_halo, v[s - 1] + static_cast<size_t>(own(L, s - 1)) * row, hrows * sizeof(double2),
                           cudaMemcpyDeviceToDevice, c->st));
      } else {
        xp_send(c, first_own, hrows, s, s - 1);
        send_from.push_back(s);
        xp_recv(c, top_halo, hrows, s - 1, s);
        recv_to.push_back(s);
      }
    }
    if (s + 1 < sl->S) {
      if (!remote && is_local(sl, s + 1)) {
        CK(cudaMemcpyAsync(bot_halo, v[s + 1] + hrows, hrows * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
      } else {
        xp_send(c, last_own, hrows, s, s + 1);
        send_from.push_back(s);
        xp_recv(c, bot_halo, hrows, s + 1, s);
        recv_to.push_back(s);
      }
    }
  }
  if (remote) xp_group_end(c, send_from, recv_to);
}

// rows [bounds[s], bounds[s+1]) of a whole-grid buffer (planes of `plane`
// double2, or planar doubles when planar) written by their owners -> every
// process (multi-process: one NCCL broadcast per owner and plane)
static void slab_share_rows(hd_ctx* c, const SlabLevel& L, void* buf, bool planar) {
  hd_slabs* sl = slabs_of(c);
  if (sl->nranks == 1) return;  // one process: the buffer is already whole
  const size_t NN = static_cast<size_t>(L.n) * L.n;
  CKN(nccl().GroupStart());
  for (int s = 0; s < sl->S; ++s) {
    const size_t r0 = static_cast<size_t>(L.bounds[s]) * L.n, cnt = static_cast<size_t>(own(L, s)) * L.n;
    if (planar) {
      double* d = static_cast<double*>(buf);
      for (int pl = 0; pl < 2; ++pl)
        CKN(nccl().Broadcast(d + pl * NN + r0, d + pl * NN + r0, cnt, ncclDouble, s, sl->comm, c->st));
    } else {
      double2* d = static_cast<double2*>(buf);
      CKN(nccl().Broadcast(d + r0, d + r0, 2 * cnt, ncclDouble, s, sl->comm, c->st));
    }
  }
  CKN(nccl().GroupEnd());
}

// per-slab blocks of `per` doubles at slab offsets (slab s at s*per) -> every process
static void slab_allgather(hd_ctx* c, double* buf, size_t per) {
  hd_slabs* sl = slabs_of(c);
  if (sl->nranks == 1) return;
  CKN(nccl().AllGather(buf + static_cast<size_t>(sl->rank) * per, buf, per, ncclDouble, sl->comm, c->st));
}

static std::vector<double2*> slab_alloc(const SlabLevel& L, int S, const hd_slabs* sl) {
  std::vector<double2*> v(S, nullptr);
  for (int s = 0; s < S; ++s) {
    if (!is_local(sl, s)) continue;
    const size_t rows = static_cast<size_t>(own(L, s) + 2 * L.H);
    v[s] = dalloc<double2>(rows * L.n);
    CK(cudaMemset(v[s], 0, rows * L.n * sizeof(double2)));
  }
  return v;
}

// ---- level operators on slabs ------------------------------------------------
static void s_apply(hd_ctx* c, int mode, const LevelDev& L, const SlabLevel& G, std::vector<double2*>& x,
                    const std::vector<double2*>* b, std::vector<double2*>* out, double omega) {
  hd_slabs* sl = slabs_of(c);
  slab_exchange(c, G, x);
  for (int s : sl->mine) {
    const int r0 = G.bounds[s], r1 = G.bounds[s + 1];
    op_apply(c, mode, L, vptr(x[s], r0, G.H, G.n), b ? vptr((*b)[s], r0, G.H, G.n) : nullptr,
             out ? vptr((*out)[s], r0, G.H, G.n) : nullptr, omega, mode == OP_RESNORM ? sl->slots + s : nullptr, 1.0,
             nullptr, 0, r0, r1, mode == OP_RESNORM ? 1 : 0);
  }
  if (mode == OP_RESNORM) slab_allgather(c, sl->slots, 1);
}

static void s_jacobi0(hd_ctx* c, const LevelDev& L, const SlabLevel& G, const std::vector<double2*>& b,
                      std::vector<double2*>& out) {
  hd_slabs* sl = slabs_of(c);
  for (int s : sl->mine) {
    const int r0 = G.bounds[s], r1 = G.bounds[s + 1];
    jacobi0(c, L, vptr(b[s], r0, G.H, G.n), vptr(out[s], r0, G.H, G.n), c->spec.omega, r0, r1);
  }
}

static std::vector<double2*>& sX(hd_slabs* sl, int l) { return sl->cur[l] ? sl->Y[l] : sl->X[l]; }
static std::vector<double2*>& sY(hd_slabs* sl, int l) { return sl->cur[l] ? sl->X[l] : sl->Y[l]; }

// one V-cycle at distributed level l (src/precond.cpp:144-153); rhs per slab;
// the result is in sX(l)
static void s_cycle(hd_ctx* c, int l, std::vector<double2*>& b, bool x_zero) {
  hd_slabs* sl = slabs_of(c);
  const SlabLevel& G = sl->lv[l];
  const LevelDev L = levM(c, l);
  const int nu = c->spec.smooth_steps;
  int st = 0;
  if (x_zero) {
    if (nu == 0) {
      for (int s : sl->mine)
        CK(cudaMemsetAsync(sX(sl, l)[s], 0, static_cast<size_t>(own(G, s) + 2 * G.H) * G.n * sizeof(double2), c->st));
    } else {
      s_jacobi0(c, L, G, b, sX(sl, l));
      st = 1;
    }
  }
  for (; st < nu; ++st) {
    s_apply(c, OP_JACOBI, L, G, sX(sl, l), &b, &sY(sl, l), c->spec.omega);
    sl->cur[l] ^= 1;
  }
  s_apply(c, OP_RESID, L, G, sX(sl, l), &b, &sl->R[l], 0.0);
  // restriction into level l+1: its slabs, or the global buffer at the gather level
  const SlabLevel& Gc = sl->lv[l + 1];
  slab_exchange(c, G, sl->R[l]);
  const bool coarse_dist = l + 1 < sl->g;
  for (int s : sl->mine) {
    const int q0 = Gc.bounds[s], q1 = Gc.bounds[s + 1];
    double2* out = coarse_dist ? vptr(sl->B[l + 1][s], q0, Gc.H, Gc.n) : c->mg_b[l + 1];
    restrict_(c, Stencil{0, 0.0}, vptr(sl->R[l][s], G.bounds[s], G.H, G.n), G.n, Gc.n, out, nullptr, q0, q1);
  }
  if (!coarse_dist) slab_share_rows(c, Gc, c->mg_b[l + 1], false);  // the gather level: allgather
  const double2* eglob = nullptr;
  if (coarse_dist) {
    s_cycle(c, l + 1, sl->B[l + 1], true);
    slab_exchange(c, Gc, sX(sl, l + 1));
  } else {
    eglob = cycle_at(c, l + 1, c->mg_b[l + 1], true);  // the small levels, once (multi-GPU: on every rank)
  }
  for (int s : sl->mine) {
    const int r0 = G.bounds[s], r1 = G.bounds[s + 1];
    const double2* ec = coarse_dist ? vptr(sX(sl, l + 1)[s], Gc.bounds[s], Gc.H, Gc.n) : eglob;
    prolong_<0>(c, Stencil{0, 0.0}, ec, nullptr, G.n, Gc.n, nullptr, vptr(sX(sl, l)[s], r0, G.H, G.n), r0, r1);
  }
  for (int k = 0; k < nu; ++k) {
    s_apply(c, OP_JACOBI, L, G, sX(sl, l), &b, &sY(sl, l), c->spec.omega);
    sl->cur[l] ^= 1;
  }
}

// out = MG^-1 b on the slabs (src/precond.cpp:159-163)
static void s_mg_solve(hd_ctx* c, std::vector<double2*>& b, std::vector<double2*>& out) {
  hd_slabs* sl = slabs_of(c);
  const SlabLevel& G = sl->lv[0];
  const LevelDev L = levM(c, 0);
  for (int cy = 0; cy < c->spec.cycles; ++cy) {
    if (cy == 0) {
      s_cycle(c, 0, b, true);
    } else {  // later cycles from the current iterate
      for (int k = 0; k < c->spec.smooth_steps; ++k) {
        s_apply(c, OP_JACOBI, L, G, sX(sl, 0), &b, &sY(sl, 0), c->spec.omega);
        sl->cur[0] ^= 1;
      }
      // residual, restriction, coarse cycle, correction, post-smoothing: as s_cycle from a nonzero start
      s_apply(c, OP_RESID, L, G, sX(sl, 0), &b, &sl->R[0], 0.0);
      const SlabLevel& Gc = sl->lv[1];
      slab_exchange(c, G, sl->R[0]);
      const bool coarse_dist = 1 < sl->g;
      for (int s : sl->mine) {
        double2* o = coarse_dist ? vptr(sl->B[1][s], Gc.bounds[s], Gc.H, Gc.n) : c->mg_b[1];
        restrict_(c, Stencil{0, 0.0}, vptr(sl->R[0][s], G.bounds[s], G.H, G.n), G.n, Gc.n, o, nullptr, Gc.bounds[s],
                  Gc.bounds[s + 1]);
      }
      if (!coarse_dist) slab_share_rows(c, Gc, c->mg_b[1], false);
      const double2* eglob = nullptr;
      if (coarse_dist) {
        s_cycle(c, 1, sl->B[1], true);
        slab_exchange(c, Gc, sX(sl, 1));
      } else {
        eglob = cycle_at(c, 1, c->mg_b[1], true);
      }
      for (int s : sl->mine) {
        const int r0 = G.bounds[s], r1 = G.bounds[s + 1];
        const double2* ec = coarse_dist ? vptr(sX(sl, 1)[s], Gc.bounds[s], Gc.H, Gc.n) : eglob;
        prolong_<0>(c, Stencil{0, 0.0}, ec, nullptr, G.n, Gc.n, nullptr, vptr(sX(sl, 0)[s], r0, G.H, G.n), r0, r1);
      }
      for (int k = 0; k < c->spec.smooth_steps; ++k) {
        s_apply(c, OP_JACOBI, L, G, sX(sl, 0), &b, &sY(sl, 0), c->spec.omega);
        sl->cur[0] ^= 1;
      }
    }
  }
  const size_t row = static_cast<size_t>(G.n) * sizeof(double2);
  for (int s : sl->mine)
    CK(cudaMemcpyAsync(out[s] + static_cast<size_t>(G.H) * G.n, sX(sl, 0)[s] + static_cast<size_t>(G.H) * G.n,
                       own(G, s) * row, cudaMemcpyDeviceToDevice, c->st));
}

// rows [r0, r1) of both planes of a column-major n x n transform buffer scaled by Dinv
__global__ void k_fd_scale_rows(double* __restrict__ T, const double2* __restrict__ Dinv, int n, int r0, int r1) {
  const size_t NN = (size_t)n * n;
  const int h = r1 - r0;
  const size_t tot = (size_t)h * n;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    const size_t g = (e / h) * n + r0 + e % h;
    const double2 v = cmul(cmk(T[g], T[g + NN]), Dinv[g]);
    T[g] = v.x;
    T[g + NN] = v.y;
  }
}

// All-to-all of the distributed E solve.  to_rows: block (rows R_t, cols C_s)
// of slab s's buffer goes to slab t (cols -> rows); else block (rows R_s,
// cols C_t) of slab s goes to slab t (rows -> cols).  R and C both follow the
// deflation grid's slab rows.  Pack (2D copies into a contiguous staging
// block per peer), transfer (NCCL send/recv, or the virtual-rank matcher),
// unpack; with every slab local and no virtual ranks the buffer is shared and
// nothing moves.
static void e_alltoall(hd_ctx* c, bool to_rows) {
  hd_slabs* sl = slabs_of(c);
  if (!remote_pairs(sl)) return;
  const int nc = c->nc;
  const size_t NN = static_cast<size_t>(nc) * nc;
  const SlabLevel& Gc = sl->lv[1];
  auto lo = [&](int t) { return Gc.bounds[t]; };
  auto cnt = [&](int t) { return Gc.bounds[t + 1] - Gc.bounds[t]; };
  const size_t dp = sizeof(double);
  // pack: for each local s and each peer t != s, the block for t, both planes, contiguous
  for (int s : sl->mine) {
    size_t off = 0;
    for (int t = 0; t < sl->S; ++t) {
      if (t == s) continue;
      const int rr0 = to_rows ? lo(t) : lo(s), rh = to_rows ? cnt(t) : cnt(s);
      const int cc0 = to_rows ? lo(s) : lo(t), cw = to_rows ? cnt(s) : cnt(t);
      for (int pl = 0; pl < 2; ++pl) {
        CK(cudaMemcpy2DAsync(sl->esend[s] + off, rh * dp, sl->eT1[s] + pl * NN + static_cast<size_t>(cc0) * nc + rr0,
                             nc * dp, rh * dp, cw, cudaMemcpyDeviceToDevice, c->st));
        off += static_cast<size_t>(rh) * cw;
      }
    }
  }
  // transfer
  std::vector<int> send_from, recv_to;
  xp_group_start(c);
  for (int s : sl->mine) {
    size_t so = 0, ro = 0;
    for (int t = 0; t < sl->S; ++t) {
      if (t == s) continue;
      const size_t ns = 2 * static_cast<size_t>(to_rows ? cnt(t) * cnt(s) : cnt(s) * cnt(t));
      const size_t nr = ns;  // the block from t has the same shape (|R_s| x |C_t| or |R_t| x |C_s| swapped)
      // double2 counts for the transport (2 doubles each); blocks have an even double count (2 planes)
      xp_send(c, reinterpret_cast<const double2*>(sl->esend[s] + so), ns / 2, s, t);
      send_from.push_back(s);
      xp_recv(c, reinterpret_cast<double2*>(sl->erecv[s] + ro), nr / 2, t, s);
      recv_to.push_back(s);
      so += ns;
      ro += nr;
    }
  }
  xp_group_end(c, send_from, recv_to);
  // unpack: the block from t lands at (rows R_s, cols C_t) (to_rows) or (rows R_t, cols C_s)
  for (int s : sl->mine) {
    size_t off = 0;
    for (int t = 0; t < sl->S; ++t) {
      if (t == s) continue;
      const int rr0 = to_rows ? lo(s) : lo(t), rh = to_rows ? cnt(s) : cnt(t);
      const int cc0 = to_rows ? lo(t) : lo(s), cw = to_rows ? cnt(t) : cnt(s);
      for (int pl = 0; pl < 2; ++pl) {
        CK(cudaMemcpy2DAsync(sl->eT1[s] + pl * NN + static_cast<size_t>(cc0) * nc + rr0, nc * dp, sl->erecv[s] + off,
                             rh * dp, rh * dp, cw, cudaMemcpyDeviceToDevice, c->st));
        off += static_cast<size_t>(rh) * cw;
      }
    }
  }
}

// E^-1 on the slabs by the fast diagonalisation with the work split by slab:
// x transforms of the slab's own coarse rows (columns of the column-major
// planes), all-to-all to kx-row blocks, y transforms and the scaling of the
// own kx rows, all-to-all back, inverse x transforms of the own rows.  ep
// holds each slab's restricted rows on entry and its rows of E^-1 r on exit.
static void s_e_solve_dist(hd_ctx* c) {
  hd_slabs* sl = slabs_of(c);
  ExactSolver& X = c->E;
  const int n = X.n;
  const long nn = static_cast<long>(n) * n;
  const double one = 1.0, zero = 0.0;
  const SlabLevel& Gc = sl->lv[1];
  auto gemm_b = [&](cublasOperation_t ta, cublasOperation_t tb, int m, int nn_, const double* A, int lda, long sA,
                    const double* B, int ldb, long sB, double* C2, int ldc, long sC) {
    const size_t mk = prof_mark(c);
    CKB(cublasDgemmStridedBatched(c->cb, ta, tb, m, nn_, n, &one, A, lda, sA, B, ldb, sB, &zero, C2, ldc, sC, 2));
    launched(c, HD_K_LIBGEMM, mk, 16.0 * nn, true);
  };
  for (int s : sl->mine) {  // x transforms of the own columns
    const int q0 = Gc.bounds[s], w = Gc.bounds[s + 1] - q0;
    gemm_b(CUBLAS_OP_T, CUBLAS_OP_N, n, w, X.V, n, 0, c->ep + static_cast<size_t>(q0) * n, n, nn,
           sl->eT1[s] + static_cast<size_t>(q0) * n, n, nn);
  }
  e_alltoall(c, true);
  for (int s : sl->mine) {  // y transforms, scaling, inverse y transforms of the own kx rows
    const int r0 = Gc.bounds[s], h = Gc.bounds[s + 1] - r0;
    gemm_b(CUBLAS_OP_N, CUBLAS_OP_N, h, n, sl->eT1[s] + r0, n, nn, X.V, n, 0, sl->eT2[s] + r0, n, nn);
    HD_LAUNCH(HD_K_EXACT, 48.0 * h * n,
              k_fd_scale_rows<<<grid_for(static_cast<size_t>(h) * n), 256, 0, c->st>>>(sl->eT2[s], X.Dinv, n, r0,
                                                                                        r0 + h));
    gemm_b(CUBLAS_OP_N, CUBLAS_OP_T, h, n, sl->eT2[s] + r0, n, nn, X.V, n, 0, sl->eT1[s] + r0, n, nn);
  }
  e_alltoall(c, false);
  for (int s : sl->mine) {  // inverse x transforms of the own columns
    const int q0 = Gc.bounds[s], w = Gc.bounds[s + 1] - q0;
    gemm_b(CUBLAS_OP_N, CUBLAS_OP_N, n, w, X.V, n, 0, sl->eT1[s] + static_cast<size_t>(q0) * n, n, nn,
           c->ep + static_cast<size_t>(q0) * n, n, nn);
  }
  slab_share_rows(c, Gc, c->ep, true);  // the prolongation reads coarse rows around the slab
}

// deflation on the slabs: out = v - Z E^-1 Z^T (A v) (project) or Z E^-1 Z^T v (Q)
static void s_deflate(hd_ctx* c, std::vector<double2*>& v, std::vector<double2*>& out, bool project) {
  hd_slabs* sl = slabs_of(c);
  const SlabLevel& G = sl->lv[0];
  const Stencil z{1, c->spec.drop};
  std::vector<double2*>* src = &v;
  if (project) {
    s_apply(c, OP_APPLY, opA(c), G, v, nullptr, &sl->t3, 0.0);
    src = &sl->t3;
  }
  slab_exchange(c, G, *src);
  const SlabLevel& Gc = sl->lv[1];  // the deflation coarse grid (per_dim / 2) shares level 1's rows
  for (int s : sl->mine)
    restrict_(c, z, vptr((*src)[s], G.bounds[s], G.H, G.n), c->n, c->nc, nullptr, c->ep, Gc.bounds[s],
              Gc.bounds[s + 1]);
  if (sl->dist_e) {
    s_e_solve_dist(c);                    // the E solve split by slab (two all-to-alls)
  } else {
    slab_share_rows(c, Gc, c->ep, true);  // the deflation coarse vector: allgather (both planes)
    exact_solve_planar(c, c->E, c->ep);    // redundantly on every process
  }
  for (int s : sl->mine) {
    const int r0 = G.bounds[s], r1 = G.bounds[s + 1];
    if (project)
      prolong_<1>(c, z, nullptr, c->ep, c->n, c->nc, vptr(v[s], r0, G.H, G.n), vptr(out[s], r0, G.H, G.n), r0, r1);
    else
      prolong_<2>(c, z, nullptr, c->ep, c->n, c->nc, nullptr, vptr(out[s], r0, G.H, G.n), r0, r1);
  }
}

// op(v) = P MG^-1 A v on the slabs (src/precond.cpp:236-245)
static void s_op(hd_ctx* c, std::vector<double2*>& v, std::vector<double2*>& out) {
  hd_slabs* sl = slabs_of(c);
  ++c->matvecs;
  s_apply(c, OP_APPLY, opA(c), sl->lv[0], v, nullptr, &sl->t1, 0.0);
  std::vector<double2*>* cur = &sl->t1;
  if (c->spec.shift) {
    ++c->shift_solves;
    c->vcycles += c->spec.cycles;
    s_mg_solve(c, sl->t1, sl->t2);
    cur = &sl->t2;
  }
  if (c->spec.deflate) {
    ++c->coarse_solves;
    s_deflate(c, *cur, out, true);
  } else {
    const SlabLevel& G = sl->lv[0];
    for (int s : sl->mine)
      CK(cudaMemcpyAsync(out[s], (*cur)[s], static_cast<size_t>(own(G, s) + 2 * G.H) * G.n * sizeof(double2),
                         cudaMemcpyDeviceToDevice, c->st));
  }
}

// ||v|| over the slabs -> dst (raw sums in slab order; scale_src: divide by it)
static void s_norm(hd_ctx* c, std::vector<double2*>& v, double* dst, double2* cdst = nullptr,
                   const double* scale_src = nullptr) {
  hd_slabs* sl = slabs_of(c);
  const SlabLevel& G = sl->lv[0];
  for (int s : sl->mine) {
    RedOut r = red_of(c, sl->slots + s);
    r.raw = 1;
    const size_t N = static_cast<size_t>(own(G, s)) * G.n;
    HD_LAUNCH(HD_K_VEC, 16.0 * N,
              k_slab_sumsq<<<std::min(grid_for(N), c->red_blocks), 256, 0, c->st>>>(v[s] + static_cast<size_t>(G.H) * G.n, N, r));
  }
  slab_allgather(c, sl->slots, 1);
  HD_LAUNCH(HD_K_VEC, 0.0, k_slab_norm<<<1, 1, 0, c->st>>>(sl->slots, sl->S, scale_src, dst, cdst));
}

static void s_monitor(hd_ctx* c, std::vector<double2*>& x) {  // ||f - A x|| / ||f||
  hd_slabs* sl = slabs_of(c);
  s_apply(c, OP_RESNORM, opA(c), sl->lv[0], x, &sl->f, nullptr, 0.0);
  HD_LAUNCH(HD_K_VEC, 0.0, k_slab_norm<<<1, 1, 0, c->st>>>(sl->slots, sl->S, c->dres + 3, c->dres + 0, nullptr));
}

// whole-grid vector <-> slabs (own rows)
static void s_scatter(hd_ctx* c, const double2* full, std::vector<double2*>& v) {
  hd_slabs* sl = slabs_of(c);
  const SlabLevel& G = sl->lv[0];
  for (int s : sl->mine)
    CK(cudaMemcpyAsync(v[s] + static_cast<size_t>(G.H) * G.n, full + static_cast<size_t>(G.bounds[s]) * G.n,
                       static_cast<size_t>(own(G, s)) * G.n * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
}
static void s_gather(hd_ctx* c, const std::vector<double2*>& v, double2* full) {
  hd_slabs* sl = slabs_of(c);
  const SlabLevel& G = sl->lv[0];
  for (int s : sl->mine)
    CK(cudaMemcpyAsync(full + static_cast<size_t>(G.bounds[s]) * G.n, v[s] + static_cast<size_t>(G.H) * G.n,
                       static_cast<size_t>(own(G, s)) * G.n * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));  slab_share_rows(c, G, full, false);
}

// basis vector u_j of slab s <-> halo'd slab vectors
__global__ void k_copy_basis(double2* __restrict__ dst, const double2* __restrict__ V, size_t Ns, const int* dj) {
  const double2* src = V + (size_t)(*dj) * Ns;
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < Ns; g += (size_t)gridDim.x * blockDim.x)
    dst[g] = src[g];
}

static void s_basis_to(hd_ctx* c, int j, std::vector<double2*>& v, const int* dj = nullptr) {
  hd_slabs* sl = slabs_of(c);
  const SlabLevel& G = sl->lv[0];
  for (int s : sl->mine) {
    const size_t Ns = static_cast<size_t>(own(G, s)) * G.n;
    if (dj)
      HD_LAUNCH(HD_K_VEC, 32.0 * Ns,
                k_copy_basis<<<grid_for(Ns), 256, 0, c->st>>>(v[s] + static_cast<size_t>(G.H) * G.n, sl->V[s], Ns, dj));
    else
      CK(cudaMemcpyAsync(v[s] + static_cast<size_t>(G.H) * G.n, sl->V[s] + static_cast<size_t>(j) * Ns,
                         Ns * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
  }
}

static LsaArgs s_lsa(hd_ctx* c, int s, int j, int mode, int maxit) {
  hd_slabs* sl = slabs_of(c);
  const SlabLevel& G = sl->lv[0];
  LsaArgs a = lsa_args(c, sl->x[s] + static_cast<size_t>(G.H) * G.n, j, mode, maxit);
  a.U = a.Uw = sl->V[s];
  a.w = sl->w[s] + static_cast<size_t>(G.H) * G.n;
  a.x0 = sl->x0[s] + static_cast<size_t>(G.H) * G.n;
  a.N = static_cast<size_t>(own(G, s)) * G.n;
  a.partials = sl->parts;
  a.part_offset = s * sl->Gs;
  a.partial_only = 1;
  a.done = sl->done;
  return a;
}

// Slab Arnoldi iteration, part a: u_j -> w = op(u_j), pass 1 (per-slab partials,
// per-slab sums, gathered, combined in slab order), pass 2 (u_{j+1} and the
// lagged x_{j-1}; partials gathered).  dj: device iteration index (graph body).
static void slab_iteration_a(hd_ctx* c, int j, int maxit, const int* dj) {
  hd_slabs* sl = slabs_of(c);
  s_basis_to(c, j, sl->vin, dj);
  s_op(c, sl->vin, sl->w);
  for (int s : sl->mine) {
    LsaArgs a = s_lsa(c, s, j, 0, maxit);
    a.dj = dj;
    HD_LAUNCH(HD_K_MGS, (j + 3.0) * 16.0 * a.N, k_lsa_dots<<<sl->Gs, kLsaBD, lsa_dots_smem(), c->st>>>(a));
  }
  for (int s : sl->mine)
    HD_LAUNCH(HD_K_MGS, 0.0, k_lsa_slab_reduce<<<1, kLsaBD, 0, c->st>>>(sl->parts + static_cast<size_t>(s) * sl->Gs * kLsaNslot,
                                                                     sl->Gs, j, dj, sl->red + static_cast<size_t>(s) * kLsaNslot));
  slab_allgather(c, reinterpret_cast<double*>(sl->red), 2 * static_cast<size_t>(kLsaNslot));
  LsaArgs af = s_lsa(c, sl->mine[0], j, 0, maxit);
  af.dj = dj;
  af.partials = sl->red;
  HD_LAUNCH(HD_K_MGS, 0.0, k_lsa_dots_finish<<<1, kLsaBD, 0, c->st>>>(af, sl->S));
  for (int s : sl->mine) {
    LsaArgs a = s_lsa(c, s, j, 0, maxit);
    a.dj = dj;
    HD_LAUNCH(HD_K_MGS, (j >= 1 ? j + 5.0 : 3.0) * 16.0 * a.N, k_lsa_update<<<sl->Gs, kLsaBD, 0, c->st>>>(a));
  }
  slab_allgather(c, reinterpret_cast<double*>(sl->parts), 2 * static_cast<size_t>(sl->Gs));
}

// part b: Givens + back substitution of column j, hnew to the host mirror
static void slab_iteration_b(hd_ctx* c, int j, int maxit, int nparts, const int* dj) {
  hd_slabs* sl = slabs_of(c);
  LsaArgs a0 = s_lsa(c, sl->mine[0], j, 0, maxit);
  a0.dj = dj;
  HD_LAUNCH(HD_K_GIVENS, 0.0, k_lsa_givens<<<1, kLsaBD, c->lsa_givens_smem, c->st>>>(a0, nparts));
  if (!dj) CK(cudaMemcpyAsync(c->hres + 1, c->dres + 1, sizeof(double), cudaMemcpyDeviceToHost, c->st));
}

// Capture one iteration (parts a and b with the monitor of x_{j-1} between
// them, the scalars copied to the pinned mirror at the end) as a graph; the
// counters it adds per launch are recorded.  NCCL calls are captured too.
constexpr int kSlabChunk = 8;  // slab bodies launched per host synchronisation

static void build_slab_body(hd_ctx* c, int maxit, double tol, int nparts) {
  hd_slabs* sl = slabs_of(c);
  if (!c->loop_state) {
    c->loop_state = dalloc<LoopState>(1);
    CK(cudaMallocHost(&c->loop_host, sizeof(LoopState)));
  }
  dfree(c->res_hist);
  if (c->res_host) cudaFreeHost(c->res_host);
  c->res_hist = dalloc<double>(maxit + 1);
  CK(cudaMallocHost(&c->res_host, (maxit + 1) * sizeof(double)));
  if (sl->body) {
    cudaGraphExecDestroy(sl->body);
    sl->body = nullptr;
  }
  const long before[6] = {c->matvecs, c->coarse_solves, c->shift_solves, c->vcycles, c->launches, c->lib_calls};
  cudaGraph_t g = nullptr;
  int* dj = &c->loop_state->j;
  sl->done = &c->loop_state->done;
  CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeRelaxed));
  slab_iteration_a(c, 0, maxit, dj);
  s_monitor(c, sl->x);  // x_{j-1} (recorded by the loop step for j >= 1)
  slab_iteration_b(c, 0, maxit, nparts, dj);
  k_slab_loop_step<<<1, 1, 0, c->st>>>(c->loop_state, c->dres, c->res_hist, tol, maxit);
  CK(cudaStreamEndCapture(c->st, &g));
  sl->done = nullptr;
  CK(cudaGraphInstantiate(&sl->body, g, 0));
  cudaGraphDestroy(g);
  const long after[6] = {c->matvecs, c->coarse_solves, c->shift_solves, c->vcycles, c->launches, c->lib_calls};
  for (int k = 0; k < 6; ++k) sl->body_delta[k] = after[k] - before[k];
  c->matvecs = before[0];
  c->coarse_solves = before[1];
  c->shift_solves = before[2];
  c->vcycles = before[3];
  c->launches = static_cast<int>(before[4]);
  c->lib_calls = static_cast<int>(before[5]);
  sl->body_maxit = maxit;
  sl->body_tol = tol;
  sl->body_epoch = c->buf_epoch;
}

static SolveOut run_solve_slabs(hd_ctx* c, const hd_gmres& opt, const double2* f_full, double2* xout_full) {
  hd_slabs* sl = slabs_of(c);
  const int maxit = std::max(opt.max_iterations, 1);
  if (maxit + 1 > kLsaMaxJ) throw Error(HD_ERR_INVALID, "row slabs: max_iterations above the Arnoldi limit");
  ensure_gmres(c, maxit);
  const SlabLevel& G = sl->lv[0];
  if (sl->maxit < maxit) {
    ++c->buf_epoch;
    for (auto* p : sl->V) dfree(p);
    for (int s : sl->mine) sl->V[s] = dalloc<double2>(static_cast<size_t>(maxit + 1) * own(G, s) * G.n);
    sl->maxit = maxit;
  }
  c->matvecs = c->coarse_solves = c->shift_solves = c->vcycles = 0;
  c->launches = c->lib_calls = 0;
  s_scatter(c, f_full, sl->f);
  s_norm(c, sl->f, c->dres + 3);
  // rhs' = P MG^-1 f, start = Q f  (src/precond.cpp:247-256)
  std::vector<double2*>* b = &sl->f;
  if (c->spec.shift) {
    ++c->shift_solves;
    c->vcycles += c->spec.cycles;
    s_mg_solve(c, sl->f, sl->t2);
    b = &sl->t2;
  }
  if (c->spec.deflate) {
    ++c->coarse_solves;
    s_deflate(c, *b, sl->rhsp, true);
    s_deflate(c, sl->f, sl->x0, false);
    ++c->coarse_solves;
  } else {
    for (int s : sl->mine) {
      CK(cudaMemcpyAsync(sl->rhsp[s], (*b)[s], static_cast<size_t>(own(G, s) + 2 * G.H) * G.n * sizeof(double2),
                         cudaMemcpyDeviceToDevice, c->st));
      CK(cudaMemsetAsync(sl->x0[s], 0, static_cast<size_t>(own(G, s) + 2 * G.H) * G.n * sizeof(double2), c->st));
    }
  }
  SolveOut res;
  s_monitor(c, sl->x0);
  read_scalars(c);
  if (c->hres[0] <= opt.tolerance) {
    res.converged = true;
    res.residuals.push_back(c->hres[0]);
    s_gather(c, sl->x0, xout_full);
    return res;
  }
  // r = rhs' - op(x0), beta = ||r||, u_0 = r, sigma_0 = 1/beta
  s_op(c, sl->x0, sl->w);
  for (int s : sl->mine) {
    const size_t o = static_cast<size_t>(G.H) * G.n, Ns = static_cast<size_t>(own(G, s)) * G.n;
    HD_LAUNCH(HD_K_VEC, 48.0 * Ns, k_sub<<<grid_for(Ns), 256, 0, c->st>>>(sl->rhsp[s] + o, sl->w[s] + o, sl->w[s] + o, Ns));
  }
  s_norm(c, sl->w, c->dres + 2, c->g);
  read_scalars(c);
  if (c->hres[2] == 0.0) {
    s_monitor(c, sl->x0);
    read_scalars(c);
    res.converged = c->hres[0] <= opt.tolerance;
    s_gather(c, sl->x0, xout_full);
    return res;
  }
  CK(cudaMemsetAsync(c->H, 0, sizeof(double2) * (maxit + 1) * maxit, c->st));
  CK(cudaMemsetAsync(c->g + 1, 0, sizeof(double2) * maxit, c->st));
  for (int s : sl->mine) {
    const size_t Ns = static_cast<size_t>(own(G, s)) * G.n;
    CK(cudaMemcpyAsync(sl->V[s], sl->w[s] + static_cast<size_t>(G.H) * G.n, Ns * sizeof(double2),
                       cudaMemcpyDeviceToDevice, c->st));
  }
  HD_LAUNCH(HD_K_VEC, 0.0, k_inv_scalar<<<1, 1, 0, c->st>>>(c->lsa_sig, c->dres + 2));
  const int nparts = sl->S * sl->Gs;  // pass-2 partials (one per CTA of every slab)
  const bool graph = c->graph_enabled && !c->prof_on;
  if (graph) {
    // The whole iteration (op, pass 1, pass 2, monitor of x_{j-1}, Givens, loop
    // step) is one captured graph reading j and done from device memory.  It is
    // launched in chunks of kSlabChunk with one host synchronisation per chunk:
    // bodies past the stopping iteration exit early (their collectives still
    // run, the same number on every rank, since every rank takes the same
    // device decision).  No per-iteration host round trip.
    if (sl->body_maxit != maxit || sl->body_tol != opt.tolerance || sl->body_epoch != c->buf_epoch)
      build_slab_body(c, maxit, opt.tolerance, nparts);
    k_loop_init<<<1, 1, 0, c->st>>>(c->loop_state);
    int bodies = 0;
    for (;;) {
      const int chunk = std::min(kSlabChunk, maxit - bodies + 1);
      for (int q = 0; q < chunk; ++q) CK(cudaGraphLaunch(sl->body, c->st));
      bodies += chunk;
      CK(cudaMemcpyAsync(c->loop_host, c->loop_state, sizeof(LoopState), cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      if (c->loop_host->done) break;
      if (bodies > maxit + 1) throw Error(HD_ERR_INVALID, "row slabs: loop state did not terminate");
    }
    const LoopState ls = *c->loop_host;
    CK(cudaMemcpyAsync(c->res_host, c->res_hist, maxit * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    if (ls.nonfinite)
      throw Error(HD_ERR_NONFINITE, "non-finite residual or Arnoldi norm at GMRES iteration " + std::to_string(ls.iters));
    const int it = ls.iters;
    res.iterations = it;
    res.converged = ls.conv != 0;
    const int recorded = ls.need_tail ? maxit - 1 : it;
    for (int q = 0; q < recorded; ++q) res.residuals.push_back(c->res_host[q]);
    // counts of the ops GMRES used (speculative ops past the stop are not counted,
    // as the host loop's rollback); launches of every body that ran
    c->matvecs += static_cast<long>(it) * sl->body_delta[0];
    c->coarse_solves += static_cast<long>(it) * sl->body_delta[1];
    c->shift_solves += static_cast<long>(it) * sl->body_delta[2];
    c->vcycles += static_cast<long>(it) * sl->body_delta[3];
    c->launches += static_cast<int>(bodies * sl->body_delta[4]);
    c->lib_calls += static_cast<int>(bodies * sl->body_delta[5]);
    if (ls.need_tail) {  // budget exhausted: x_{maxit-1}, then its monitor
      for (int s : sl->mine) {
        LsaArgs bq = s_lsa(c, s, maxit - 1, 1, maxit);
        HD_LAUNCH(HD_K_ITERATE, (maxit + 2.0) * 16.0 * bq.N, k_lsa_update<<<sl->Gs, kLsaBD, 0, c->st>>>(bq));
      }
      s_monitor(c, sl->x);
      read_scalars(c);
      res.residuals.push_back(c->hres[0]);
      res.converged = c->hres[0] <= opt.tolerance;
    }
    s_gather(c, sl->x, xout_full);
    return res;
  }
  bool stop = false;
  double hnew_prev = 1.0;
  for (int j = 0; j < maxit && !stop; ++j) {
    const long snap[4] = {c->matvecs, c->coarse_solves, c->shift_solves, c->vcycles};
    auto rollback = [&]() {
      c->matvecs = snap[0];
      c->coarse_solves = snap[1];
      c->shift_solves = snap[2];
      c->vcycles = snap[3];
    };
    slab_iteration_a(c, j, maxit, nullptr);
    if (j >= 1) {  // x_{j-1} is ready
      s_monitor(c, sl->x);
      read_scalars(c);
      const double rr = c->hres[0];
      res.iterations = j;
      res.residuals.push_back(rr);
      if (rr <= opt.tolerance) {
        res.converged = true;
        rollback();
        break;
      }
      if (hnew_prev < 1e-300) {
        rollback();
        break;
      }
    }
    slab_iteration_b(c, j, maxit, nparts, nullptr);
    if (j + 1 == maxit) {  // budget exhausted: x_{maxit-1}, then its monitor
      for (int s : sl->mine) {
        LsaArgs bq = s_lsa(c, s, j, 1, maxit);
        HD_LAUNCH(HD_K_ITERATE, (j + 3.0) * 16.0 * bq.N, k_lsa_update<<<sl->Gs, kLsaBD, 0, c->st>>>(bq));
      }
      s_monitor(c, sl->x);
      read_scalars(c);
      const double rr = c->hres[0];
      res.iterations = j + 1;
      res.residuals.push_back(rr);
      res.converged = rr <= opt.tolerance;
      stop = true;
    }
    CK(cudaStreamSynchronize(c->st));
    hnew_prev = c->hres[1];
  }
  s_gather(c, sl->x, xout_full);
  return res;
}

// plan of slabs.py (gather level, doubled boundaries), built from the context's hierarchy
static void create_slabs(hd_ctx* c, int S, int rank = 0, int nranks = 1, ncclComm_t comm = nullptr) {
  if (c->dim != 2) throw Error(HD_ERR_INVALID, "row slabs: 2D only (1D configs run as replicas)");
  if (c->lev.size() < 2 || !c->spec.shift || c->spec.cycles < 1)
    throw Error(HD_ERR_INVALID, "row slabs: needs the multigrid-CSLP preconditioner (shift, cycles >= 1)");
  // layered and wedge fields: the G-term / stored-stencil level operators take
  // row ranges like the Kronecker-sum stencil; their exact E solves (dense or
  // block tridiagonal) run redundantly on the gathered coarse vector
  const int L = static_cast<int>(c->lev.size());
  const char* e = std::getenv("HD_SLAB_AGGLOMERATE");
  const int agg = e ? std::atoi(e) : 200;
  auto split = [&](int n) {
    std::vector<int> q(S + 1);
    for (int r = 0; r <= S; ++r) q[r] = static_cast<int>((static_cast<long>(r) * n + S / 2) / S);
    return q;
  };
  int g = 1;
  while (g < L - 1 && c->lev[g].n > agg) ++g;
  std::vector<std::vector<int>> bnd;
  for (;; --g) {
    const std::vector<int> q = split(c->lev[g].n);
    bnd.assign(L, {});
    bool ok = true;
    for (int l = 0; l <= g; ++l) {
      const int f = 1 << (g - l);
      std::vector<int> b(S + 1);
      for (int r = 0; r < S; ++r) b[r] = q[r] * f;
      b[S] = c->lev[l].n;
      bnd[l] = b;
      if (l < g)
        for (int r = 0; r < S; ++r)
          if (b[r + 1] - b[r] < std::max(8, std::max(c->lev[l].b, 2) + 2)) ok = false;
    }
    if (ok) break;
    if (g == 1) throw Error(HD_ERR_INVALID, "row slabs: grid too small for " + std::to_string(S) + " slabs");
  }
  auto* sl = new hd_slabs();
  c->slabs = sl;
  sl->S = S;
  sl->g = g;
  sl->rank = rank;
  sl->nranks = nranks;
  sl->comm = comm;
  const char* vr = std::getenv("HD_SLAB_VRANKS");
  sl->vranks = nranks == 1 && vr && std::atoi(vr) == 1;
  for (int s = 0; s < S; ++s)
    if (nranks == 1 || s == rank) sl->mine.push_back(s);
  sl->lv.resize(L);
  for (int l = 0; l < L; ++l) {
    SlabLevel& G = sl->lv[l];
    G.n = c->lev[l].n;
    G.b = c->lev[l].b;
    G.H = std::max({G.b, c->fine.b, 2});
    G.dist = l < g;
    G.bounds = bnd[l];
  }
  sl->X.resize(g);
  sl->Y.resize(g);
  sl->B.resize(g);
  sl->R.resize(g);
  sl->cur.assign(L, 0);
  for (int l = 0; l < g; ++l) {
    sl->X[l] = slab_alloc(sl->lv[l], S, sl);
    sl->Y[l] = slab_alloc(sl->lv[l], S, sl);
    if (l > 0) sl->B[l] = slab_alloc(sl->lv[l], S, sl);
    sl->R[l] = slab_alloc(sl->lv[l], S, sl);
  }
  for (auto* v : {&sl->f, &sl->w, &sl->t1, &sl->t2, &sl->t3, &sl->x, &sl->x0, &sl->rhsp, &sl->vin})
    *v = slab_alloc(sl->lv[0], S, sl);
  sl->V.assign(S, nullptr);
  sl->slots = dalloc<double>(S);
  // Arnoldi grid per slab and the partials of all slabs
  const size_t Nmax = static_cast<size_t>(*std::max_element(bnd[0].begin() + 1, bnd[0].end())) * c->n;
  sl->Gs = std::max(1, std::min(c->lsa_G > 0 ? c->lsa_G : 296, static_cast<int>((Nmax + 1023) / 1024)));
  sl->parts = dalloc<double2>(static_cast<size_t>(S) * sl->Gs * (2 * kLsaMaxJ + 2) + 8);
  sl->red = dalloc<double2>(static_cast<size_t>(S) * kLsaNslot);
  // distributed E solve when E is the plain fast diagonalisation (HD_DIST_E=0: redundant)
  {
    const ExactSolver& X = c->E;
    const char* de = std::getenv("HD_DIST_E");
    sl->dist_e = c->spec.deflate && X.dim == 2 && X.V && !X.folded && !X.pfd && !X.dense && !X.btri &&
                 !(de && std::atoi(de) == 0);
    if (sl->dist_e) {
      const int nc = c->nc;
      const size_t NN = static_cast<size_t>(nc) * nc;
      const SlabLevel& Gc = sl->lv[1];
      sl->eT1.assign(S, nullptr);
      sl->eT2.assign(S, nullptr);
      sl->esend.assign(S, nullptr);
      sl->erecv.assign(S, nullptr);
      for (int s2 : sl->mine) {
        if (sl->vranks || sl->nranks > 1) {
          sl->eT1[s2] = dalloc<double>(2 * NN);
          sl->eT2[s2] = dalloc<double>(2 * NN);
        } else {
          sl->eT1[s2] = X.T1;
          sl->eT2[s2] = X.T2;
        }
        const size_t own_c = static_cast<size_t>(Gc.bounds[s2 + 1] - Gc.bounds[s2]);
        sl->esend[s2] = dalloc<double>(2 * static_cast<size_t>(nc) * own_c);
        sl->erecv[s2] = dalloc<double>(2 * static_cast<size_t>(nc) * own_c);
      }
    }
  }
  CK(cudaDeviceSynchronize());
}

static void destroy_slabs(hd_ctx* c) {
  hd_slabs* sl = slabs_of(c);
  if (!sl) return;
  auto fr = [](std::vector<double2*>& v) {
    for (auto* p : v) dfree(p);
  };
  for (auto& v : sl->X) fr(v);
  for (auto& v : sl->Y) fr(v);
  for (auto& v : sl->B) fr(v);
  for (auto& v : sl->R) fr(v);
  for (auto* v : {&sl->f, &sl->w, &sl->t1, &sl->t2, &sl->t3, &sl->x, &sl->x0, &sl->rhsp, &sl->vin, &sl->V}) fr(*v);
  dfree(sl->slots);
  dfree(sl->parts);
  dfree(sl->red);
  if (sl->vranks || sl->nranks > 1)
    for (int s : sl->mine) {
      dfree(sl->eT1[s]);
      dfree(sl->eT2[s]);
    }
  for (int s : sl->mine) {
    if (!sl->esend.empty()) dfree(sl->esend[s]);
    if (!sl->erecv.empty()) dfree(sl->erecv[s]);
  }
  if (sl->body) cudaGraphExecDestroy(sl->body);
  dfree(sl->dj);
  if (sl->hj) cudaFreeHost(sl->hj);
  if (sl->comm) nccl().CommDestroy(sl->comm);
  delete sl;
  c->slabs = nullptr;
}


}  // namespace hd
