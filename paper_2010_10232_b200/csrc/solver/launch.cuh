// Launch helpers, per-launch profiling, level operators, transfers, exact solves, the V-cycle, deflation, the composed operator, the Arnoldi engines and the single-domain GMRES loop (host-driven and graph-resident).
// (part of solver.cu, a single translation unit: included in order)
#pragma once

namespace hd {

// ---------------------------------------------------------------------------
// launch helpers + per-launch profiling (CUDA events on the launch stream)
// ---------------------------------------------------------------------------
static size_t prof_mark(hd_ctx* c) {
  if (!c->prof_on) return static_cast<size_t>(-1);
  if (c->prof_used >= c->prof_ev.size()) {
    const size_t grow = std::max<size_t>(1024, c->prof_ev.size());
    for (size_t i = 0; i < grow; ++i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      c->prof_ev.push_back(e);
    }
  }
  CK(cudaEventRecord(c->prof_ev[c->prof_used], c->st));
  return c->prof_used++;
}

// source line of the launch being checked (error messages; HD_LAUNCH sets it)
static thread_local int g_launch_line = 0;

// called right after a launch: error check, launch count, profile record
static void launched(hd_ctx* c, int kind, size_t mark, double bytes, bool library = false) {
  const cudaError_t le = cudaGetLastError();
  if (le != cudaSuccess)
    throw Error(HD_ERR_CUDA, std::string("kernel launch (kind ") + std::to_string(kind) + ", launch.cuh:" +
                                 std::to_string(g_launch_line) + "): " + cudaGetErrorString(le));
  g_launch_line = 0;
  if (library) ++c->lib_calls;
  else ++c->launches;
  if (mark == static_cast<size_t>(-1)) return;
  prof_mark(c);
  c->prof_recs.push_back({kind, mark, bytes});
}

#define HD_LAUNCH(kind, bytes, ...)        \
  do {                                     \
    const size_t mk_ = prof_mark(c);       \
    g_launch_line = __LINE__;              \
    __VA_ARGS__;                           \
    launched(c, (kind), mk_, (bytes));     \
  } while (0)
static int grid_for(size_t N, int threads = 256, int cap = 148 * 8) {
  const size_t g = (N + threads - 1) / threads;
  return static_cast<int>(std::max<size_t>(1, std::min<size_t>(g, cap)));
}

// algorithmic bytes of one operator launch: x read + output (+ b read)
static double op_bytes(int mode, size_t NL) {
  const double P = 16.0 * static_cast<double>(NL);
  switch (mode) {
    case OP_APPLY: return 2 * P;
    case OP_RESNORM: return 2 * P;
    case OP_JACOBIP: return 3.25 * P;  // + the coarse correction, a quarter of a fine pass
    default: return 3 * P;
  }
}

// Per instantiation: opt in to the dynamic shared memory of the tallest strip
// and query how many CTAs are resident per SM.
template <int B, int MODE>
static int stencil_occupancy() {
  // per device: the opt-in and the resident-CTA count (cached per (device, kernel))
  static std::mutex mu;
  static std::map<int, int> per_dev;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = per_dev.find(dev);
    if (it != per_dev.end()) return it->second;
  }
  constexpr size_t sm = stencil_smem<B, MODE>(kSRowsMax);
  smem_optin(reinterpret_cast<const void*>(k_stencil2d<B, MODE>), sm);
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_stencil2d<B, MODE>, kSW * kSWarps, sm));
  per = std::max(per, 1);
  std::lock_guard<std::mutex> lk(mu);
  per_dev[dev] = per;
  return per;
}

// Strip height: fill whole waves of resident CTAs, discounted by the 2B halo
// rows each strip re-reads.
static int pick_rows(int n, int rows, int slots, int B) {
  const int colblocks = (n + kSW * kSWarps - 1) / (kSW * kSWarps);
  static const int cand[] = {8, 12, 16, 20, 24, 28, 32, 40, 48, 56, 64, 80, 96, 112, 128};
  int best = 32;
  double best_score = -1.0;
  for (int ry : cand) {
    if (ry > kSRowsMax) break;
    const long tiles = static_cast<long>(colblocks) * ((rows + ry - 1) / ry);
    const long waves = (tiles + slots - 1) / slots;
    const double util = static_cast<double>(tiles) / (static_cast<double>(waves) * slots);
    const double score = util * ry / (ry + 2.0 * B);
    if (score > best_score + 1e-9) {
      best_score = score;
      best = ry;
    }
  }
  return best;
}

// ---- tensor-copy stencil (stencil_tma.cuh): tensor maps, CT tables, launch -------------------
typedef CUresult (*TmaEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled through the runtime (the library does not link libcuda); null when the driver lacks it
static TmaEncodeFn tma_encode_fn() {
  static TmaEncodeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<TmaEncodeFn>(f);
  }();
  return fn;
}

// Map of `nvec` consecutive n x n complex grids at `base` viewed as doubles (2n, n, nvec), box
// (2 cols, kTSR rows, 1); rows and columns outside a grid read as zero.  Cached per context.
static const CUtensorMap& tma_map(hd_ctx* c, const double2* base, int n, int nvec, int cols) {
  const hd_ctx::TmaKey key{base, n, nvec, cols};
  auto it = c->tma_maps.find(key);
  if (it != c->tma_maps.end()) return it->second;
  CUtensorMap m;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(2) * n, static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(nvec)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(16) * n, static_cast<cuuint64_t>(16) * n * n};
  const cuuint32_t box[3] = {static_cast<cuuint32_t>(2 * cols), static_cast<cuuint32_t>(kTSR), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = tma_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2*>(base), dims, strides,
                                     box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(HD_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return c->tma_maps.emplace(key, m).first->second;
}

// CT of a level (y coefficients per input row, stencil_tma.cuh); setup builds the tables of
// every eligible level (tma_prepare), so no allocation happens inside a graph capture
static const double2* tma_ct(hd_ctx* c, const LevelDev& L) {
  auto key = std::make_pair(L.S, L.M);
  auto it = c->tma_ct.find(key);
  if (it != c->tma_ct.end()) return it->second;
  const int rows = L.n + 2 * L.b + kTSR;
  double2* ct = dalloc<double2>(static_cast<size_t>(rows) * (2 * L.b + 2));
  k_build_ct<<<64, 256, 0, c->st>>>(L, ct, rows);
  CK(cudaGetLastError());
  c->tma_ct[key] = ct;
  return ct;
}

// the modes and levels the tensor-copy kernel takes: whole-grid operators (no row slab) of 2D
// Kronecker-sum levels with at least tma_min_n rows.  The Jacobi mode stays on the cp.async
// kernel (its centre-value queue spills at two columns per lane).
template <int MODE>
static bool stencil_tma_ok(hd_ctx* c, const LevelDev& L, int rb, int re) {
  return c->stencil_tma && MODE != OP_JACOBI && MODE != OP_JACOBIP && rb == 0 && re == L.n && L.n >= c->tma_min_n && L.b <= 6 &&
         tma_encode_fn() != nullptr;
}

template <int B, int MODE>
static int stencil_tma_occupancy() {
  static std::mutex mu;
  static std::map<int, int> per_dev;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = per_dev.find(dev);
    if (it != per_dev.end()) return it->second;
  }
  constexpr size_t sm = TmaLayout<B, MODE>::total;
  smem_optin(reinterpret_cast<const void*>(k_stencil2d_tma<B, MODE>), sm);
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_stencil2d_tma<B, MODE>, 32 * kTWarps, sm));
  per = std::max(per, 1);
  std::lock_guard<std::mutex> lk(mu);
  per_dev[dev] = per;
  return per;
}

// strip height of the tensor-copy kernel: the warp tasks fill whole waves of resident warps,
// discounted by the 2B halo rows every strip recomputes
static int pick_rows_tma(int n, int warp_slots, int B, int* strips_x, int* ntasks) {
  const int sx = (n + kTW - 1) / kTW;
  int best = 32;
  double best_score = -1.0;
  for (int ry = 8; ry <= 256; ++ry) {
    const long tasks = static_cast<long>(sx) * ((n + ry - 1) / ry);
    const long waves = (tasks + warp_slots - 1) / warp_slots;
    const double util = static_cast<double>(tasks) / (static_cast<double>(waves) * warp_slots);
    const double score = util * ry / (ry + 2.0 * B);
    if (score > best_score + 1e-9) {
      best_score = score;
      best = ry;
    }
  }
  *strips_x = sx;
  *ntasks = sx * ((n + best - 1) / best);
  return best;
}

template <int B, int MODE>
static void launch_stencil_tma(hd_ctx* c, const LevelDev& L, const double2* x, const double2* b, double2* out,
                               double omega, RedOut red, const int* xidx, size_t xstride, double2* out2, double2 c2) {
  const int per = stencil_tma_occupancy<B, MODE>();
  int strips_x = 0, ntasks = 0;
  const int ry = pick_rows_tma(L.n, per * kTWarps * c->n_sms, B, &strips_x, &ntasks);
  // x: one grid, or (graph mode, x = V + j N with j on the device) the whole basis as a 3D map
  const bool basis = xidx != nullptr;
  if (basis && xstride != static_cast<size_t>(L.n) * L.n) throw Error(HD_ERR_INVALID, "stencil: basis stride");
  const CUtensorMap& tmx = tma_map(c, x, L.n, basis ? c->v_cap : 1, tma_xc<B>());
  const bool need_b = TmaLayout<B, MODE>::NEED_B;
  const CUtensorMap& tmb = need_b ? tma_map(c, b, L.n, 1, kTBC) : tmx;
  const double2* ct = tma_ct(c, L);
  const int grid = (ntasks + kTWarps - 1) / kTWarps;
  k_stencil2d_tma<B, MODE><<<grid, 32 * kTWarps, TmaLayout<B, MODE>::total, c->st>>>(tmx, tmb, L, ct, out, omega, ry,
                                                                                      strips_x, ntasks, red, xidx, out2, c2);
}

template <int B, int MODE>
static void launch_stencil(hd_ctx* c, const LevelDev& L, const double2* x, const double2* b, double2* out,
                           double omega, RedOut red, const int* xidx, size_t xstride, int rb, int re,
                           double2* out2 = nullptr, double2 c2 = double2{0.0, 0.0}, const double2* ec = nullptr,
                           int nc = 0) {
  if constexpr (MODE != OP_JACOBI && MODE != OP_JACOBIP) {  // (the Jacobi modes have no tensor-copy instantiation)
    if (stencil_tma_ok<MODE>(c, L, rb, re)) {
      launch_stencil_tma<B, MODE>(c, L, x, b, out, omega, red, xidx, xstride, out2, c2);
      return;
    }
  }
  const int per = stencil_occupancy<B, MODE>();
  const int ry = pick_rows(L.n, re - rb, per * c->n_sms, B);
  dim3 grid((L.n + kSW * kSWarps - 1) / (kSW * kSWarps), (re - rb + ry - 1) / ry);
  k_stencil2d<B, MODE><<<grid, kSW * kSWarps, stencil_smem<B, MODE>(ry), c->st>>>(L, x, b, out, omega, ry, red,
                                                                               xidx, xstride, rb, re, out2, c2, ec, nc);
}

template <int MODE>
static void launch_op2d_mode(hd_ctx* c, const LevelDev& L, const double2* x, const double2* b, double2* out,
                             double omega, RedOut red, int kind, const int* xidx, size_t xstride, int rb = 0,
                             int re = -1, double2* out2 = nullptr, double2 c2 = double2{0.0, 0.0},
                             const double2* ec = nullptr, int nc = 0) {
  if (re < 0) re = L.n;
  const size_t mk = prof_mark(c);
  g_launch_line = __LINE__ + 1000 * MODE;
  switch (L.b) {
#define HD_CASE(BB) \
  case BB: launch_stencil<BB, MODE>(c, L, x, b, out, omega, red, xidx, xstride, rb, re, out2, c2, ec, nc); break;
    HD_CASE(1) HD_CASE(2) HD_CASE(3) HD_CASE(4) HD_CASE(5) HD_CASE(6)
#undef HD_CASE
    default: throw Error(HD_ERR_INVALID, "band half-width " + std::to_string(L.b) + " unsupported");
  }
  launched(c, kind, mk, op_bytes(MODE, static_cast<size_t>(L.n) * (re - rb)) + (MODE == OP_APPLYJ0 ? 16.0 * L.n * (re - rb) : 0.0));
}

// layered field: G-term Kronecker-sum operator (layered.cuh)
template <int MODE>
static void launch_gen_mode(hd_ctx* c, const GenLevel& G, const double2* x, const double2* b, double2* out,
                            double omega, RedOut red, int kind, const int* xidx, size_t xstride, int rb, int re) {
  smem_optin(reinterpret_cast<const void*>(k_kron2d<MODE>), gen_smem(6, kGenMaxG));
  if (G.b > 6 || G.G > kGenMaxG) throw Error(HD_ERR_INVALID, "layered operator exceeds the kernel limits");
  if (re < 0) re = G.n;
  const dim3 grid((G.n + kGenTX - 1) / kGenTX, (re - rb + kGenTY - 1) / kGenTY);
  // algorithmic bytes: the vector passes plus, for a stored stencil, its (2b+1)^2 coefficient planes
  const double bytes = op_bytes(MODE, static_cast<size_t>(G.n) * (re - rb)) +
                       (G.K ? 8.0 * (2 * G.b + 1) * (2 * G.b + 1) * G.n * (re - rb) : 0.0);
  HD_LAUNCH(kind, bytes,
            k_kron2d<MODE><<<grid, kGenThreads, gen_smem(G.b, G.G), c->st>>>(G, x, b, out, omega, red, xidx,
                                                                               xstride, rb, re));
}

static RedOut red_of(hd_ctx* c, double* dst = nullptr, double scale = 1.0) {
  RedOut r;
  r.raw = 0;
  r.partials = c->partials;
  r.counter = c->counter;
  r.dst = dst;
  r.scale = scale;
  return r;
}

// out = L x | b - L x | x + w D^-1 (b - L x) | ||b - L x|| * scale -> dst
static void op_apply(hd_ctx* c, int mode, const LevelDev& L, const double2* x, const double2* b, double2* out,
                     double omega = 0.0, double* dst = nullptr, double scale = 1.0, const int* xidx = nullptr,
                     size_t xstride = 0, int rb = 0, int re = -1, int raw = 0) {
  RedOut red = red_of(c, dst, scale);
  red.raw = raw;
  const int kind = L.n == c->n ? HD_K_OP_FINE : HD_K_OP_COARSE;
  if (L.gen) {
    const GenLevel& G = *static_cast<const GenLevel*>(L.gen);
    switch (mode) {
      case OP_APPLY: launch_gen_mode<OP_APPLY>(c, G, x, b, out, omega, red, kind, xidx, xstride, rb, re); break;
      case OP_RESID: launch_gen_mode<OP_RESID>(c, G, x, b, out, omega, red, kind, xidx, xstride, rb, re); break;
      case OP_JACOBI: launch_gen_mode<OP_JACOBI>(c, G, x, b, out, omega, red, kind, xidx, xstride, rb, re); break;
      default: launch_gen_mode<OP_RESNORM>(c, G, x, b, out, omega, red, kind, xidx, xstride, rb, re); break;
    }
    return;
  }
  if (c->dim == 2) {
    switch (mode) {
      case OP_APPLY: launch_op2d_mode<OP_APPLY>(c, L, x, b, out, omega, red, kind, xidx, xstride, rb, re); break;
      case OP_RESID: launch_op2d_mode<OP_RESID>(c, L, x, b, out, omega, red, kind, xidx, xstride, rb, re); break;
      case OP_JACOBI: launch_op2d_mode<OP_JACOBI>(c, L, x, b, out, omega, red, kind, xidx, xstride, rb, re); break;
      default: launch_op2d_mode<OP_RESNORM>(c, L, x, b, out, omega, red, kind, xidx, xstride, rb, re); break;
    }
  } else {
    const int grid = mode == OP_RESNORM ? std::min(grid_for(L.n), c->red_blocks) : grid_for(L.n);
    const size_t mk = prof_mark(c);
    switch (mode) {
      case OP_APPLY: k_op1d<OP_APPLY><<<grid, 256, 0, c->st>>>(L, x, b, out, omega, red, xidx, xstride); break;
      case OP_RESID: k_op1d<OP_RESID><<<grid, 256, 0, c->st>>>(L, x, b, out, omega, red, xidx, xstride); break;
      case OP_JACOBI: k_op1d<OP_JACOBI><<<grid, 256, 0, c->st>>>(L, x, b, out, omega, red, xidx, xstride); break;
      default: k_op1d<OP_RESNORM><<<grid, 256, 0, c->st>>>(L, x, b, out, omega, red, xidx, xstride); break;
    }
    launched(c, kind, mk, op_bytes(mode, L.n));
  }
}

static void jacobi0(hd_ctx* c, const LevelDev& L, const double2* b, double2* out, double omega, int rb = 0,
                    int re = -1) {
  if (re < 0) re = L.n;
  const size_t NN = c->dim == 2 ? static_cast<size_t>(L.n) * L.n : L.n;
  if (L.gen) {
    const size_t NR = static_cast<size_t>(re - rb) * L.n;
    HD_LAUNCH(HD_K_JACOBI0, 32.0 * NR,
              k_jacobi0_gen<<<grid_for(NR), 256, 0, c->st>>>(*static_cast<const GenLevel*>(L.gen), b, out, omega, rb,
                                                             re));
    return;
  }
  HD_LAUNCH(HD_K_JACOBI0, 32.0 * NN,
            if (c->dim == 2) k_jacobi0_2d_t<<<dim3((L.n + 63) / 64, (re - rb + 15) / 16), 256, 0, c->st>>>(
                L, b, out, omega, rb, re);
            else k_jacobi0_1d<<<grid_for(NN), 256, 0, c->st>>>(L, b, out, omega));
}

static void restrict_(hd_ctx* c, Stencil z, const double2* r, int nf, int nc, double2* outc, double* outp,
                      int qb = 0, int qe = -1) {
  if (qe < 0) qe = nc;
  const size_t NC = c->dim == 2 ? static_cast<size_t>(nc) * nc : nc;
  const double NF = c->dim == 2 ? static_cast<double>(nf) * nf : nf;
  if (c->dim == 2) {
    dim3 grid((nc + kRQX - 1) / kRQX, (qe - qb + kRQY - 1) / kRQY);
    HD_LAUNCH(HD_K_TRANSFER, 16.0 * (NF + NC),
              if (z.kind == 0 && !outp) k_restrict2d<0, 0><<<grid, 256, 0, c->st>>>(z.drop, r, nf, nc, outc, outp, qb, qe);
              else if (z.kind == 0) k_restrict2d<0, 1><<<grid, 256, 0, c->st>>>(z.drop, r, nf, nc, outc, outp, qb, qe);
              else if (!outp) k_restrict2d<1, 0><<<grid, 256, 0, c->st>>>(z.drop, r, nf, nc, outc, outp, qb, qe);
              else k_restrict2d<1, 1><<<grid, 256, 0, c->st>>>(z.drop, r, nf, nc, outc, outp, qb, qe));
    return;
  }
  HD_LAUNCH(HD_K_TRANSFER, 16.0 * (NF + NC),
            k_restrict<1><<<grid_for(NC), 256, 0, c->st>>>(z, r, nf, nc, outc, outp));
}

// linear restriction fused with the coarse level's first Jacobi sweep from zero:
// outc = z^T r and x0 = omega D^-1 outc (2D Kronecker-sum levels)
// strip height of the streaming linear restriction: the warp tasks fill the resident warps in whole waves
static int restrict_stream_rows(hd_ctx* c, int nc, int* strips_x, int* ntasks) {
  static int per_sm = 0;  // resident warps per SM of the kernel (same for both J0 variants)
  if (!per_sm) {
    int ctas = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ctas, k_restrict_lin_stream<true>, 32 * kRSWarps, 0));
    per_sm = std::max(1, ctas) * kRSWarps;
  }
  const int sx = (nc + 31) / 32, slots = c->n_sms * per_sm;
  int best = 16;
  double best_score = -1.0;
  for (int qr = 4; qr <= 64; ++qr) {
    const long tasks = static_cast<long>(sx) * ((nc + qr - 1) / qr);
    const long waves = (tasks + slots - 1) / slots;
    const double score = static_cast<double>(tasks) / (static_cast<double>(waves) * slots) * (2.0 * qr) / (2.0 * qr + 1.0);
    if (score > best_score + 1e-9) best_score = score, best = qr;
  }
  *strips_x = sx;
  *ntasks = sx * ((nc + best - 1) / best);
  return best;
}

static void restrict_j0(hd_ctx* c, const double2* r, int nf, int nc, double2* outc, const LevelDev& Lc, double omega,
                        double2* x0) {
  if (c->restrict_stream && nf >= c->tma_min_n) {  // fine levels: the streaming kernel (same arithmetic)
    int sx = 0, nt = 0;
    const int qr = restrict_stream_rows(c, nc, &sx, &nt);
    HD_LAUNCH(HD_K_TRANSFER, 16.0 * (static_cast<double>(nf) * nf + 2.0 * nc * nc),
              k_restrict_lin_stream<true><<<(nt + kRSWarps - 1) / kRSWarps, 32 * kRSWarps, 0, c->st>>>(
                  r, nf, nc, qr, sx, nt, outc, Lc, omega, x0));
    return;
  }
  dim3 grid((nc + kRQX - 1) / kRQX, (nc + kRQY - 1) / kRQY);
  HD_LAUNCH(HD_K_TRANSFER, 16.0 * (static_cast<double>(nf) * nf + 2.0 * nc * nc),
            k_restrict2d<0, 0, true><<<grid, 256, 0, c->st>>>(0.0, r, nf, nc, outc, nullptr, 0, nc, Lc, omega, x0));
}

template <int PMODE>
static void prolong_(hd_ctx* c, Stencil z, const double2* ec, const double* ep, int nf, int nc, const double2* s,
                     double2* out, int fb = 0, int fe = -1) {
  if (fe < 0) fe = nf;
  const size_t NF = c->dim == 2 ? static_cast<size_t>(nf) * nf : nf;
  const double NC = c->dim == 2 ? static_cast<double>(nc) * nc : nc;
  if (c->dim == 2) {
    dim3 grid((nf + kPFX - 1) / kPFX, (fe - fb + kPFY - 1) / kPFY);
    HD_LAUNCH(HD_K_TRANSFER, 16.0 * (NC + (PMODE == 2 ? 1.0 : 2.0) * NF),
              if (z.kind == 0) k_prolong2d<0, PMODE><<<grid, 256, 0, c->st>>>(z.drop, ec, ep, nf, nc, s, out, fb, fe);
              else k_prolong2d<1, PMODE><<<grid, 256, 0, c->st>>>(z.drop, ec, ep, nf, nc, s, out, fb, fe));
    return;
  }
  HD_LAUNCH(HD_K_TRANSFER, 16.0 * (NC + (PMODE == 2 ? 1.0 : 2.0) * NF),
            k_prolong<1, PMODE><<<grid_for(NF), 256, 0, c->st>>>(z, ec, ep, nf, nc, s, out));
}

// Fused level operator + restriction (stencil_restrict.cuh): rc = Z^T (L x)
// (APPLY, the projection) or Z^T (b - L x) (RESID, the V-cycle), r never
// stored.  kind 0: linear MG transfer into outc (+ J0: x0 = omega D_c^-1 rc);
// kind 1: Bezier deflation transfer into the planar coarse vector outp.
static bool fused_restrict_ok(hd_ctx* c, const LevelDev& L) {
  static const bool off = std::getenv("HD_NOFUSE") != nullptr;
  return !off && c->dim == 2 && !L.gen && L.b >= 1 && L.b <= 6;
}

template <int B, int MODE, int KIND, int PLANAR, bool J0>
static void launch_sr(hd_ctx* c, const LevelDev& L, const double2* x, const double2* b, double drop, int nc,
                      double2* outc, double* outp, const LevelDev& Lc, double omega, double2* x0c) {
  constexpr int QW = sr_qw<KIND>();
  constexpr int nw = ZW<KIND>::nw;
  const int per = stencil_occupancy<B, MODE>();  // same ring and smem as the plain stencil
  const int slots = per * c->n_sms;
  const int cols = (nc + QW * kSWarps - 1) / (QW * kSWarps);
  // strip height in coarse rows: fill whole waves, discounting the recomputed rows
  int best = 16;
  double best_score = -1.0;
  for (int qr = 4; 2 * qr + nw - 1 <= kSRowsMax; qr += 2) {
    const long tiles = static_cast<long>(cols) * ((nc + qr - 1) / qr);
    const long waves = (tiles + slots - 1) / slots;
    const double util = static_cast<double>(tiles) / (static_cast<double>(waves) * slots);
    const double score = util * (2.0 * qr) / (2.0 * qr + nw - 2 + 2.0 * B);
    if (score > best_score + 1e-9) {
      best_score = score;
      best = qr;
    }
  }
  const int nout = 2 * best + nw - 1;
  smem_optin(reinterpret_cast<const void*>(k_stencil_restrict2d<B, MODE, KIND, PLANAR, J0>),
             stencil_smem<B, MODE>(kSRowsMax));
  const dim3 grid(cols, (nc + best - 1) / best);
  k_stencil_restrict2d<B, MODE, KIND, PLANAR, J0><<<grid, kSW * kSWarps, stencil_smem<B, MODE>(nout), c->st>>>(
      L, x, b, drop, nc, best, outc, outp, Lc, omega, x0c);
}

template <int MODE, int KIND, int PLANAR, bool J0>
static void op_restrict(hd_ctx* c, const LevelDev& L, const double2* x, const double2* b, double drop, int nc,
                        double2* outc, double* outp, const LevelDev& Lc = LevelDev{}, double omega = 0.0,
                        double2* x0c = nullptr) {
  const double NF = static_cast<double>(L.n) * L.n, NCd = static_cast<double>(nc) * nc;
  const double bytes = 16.0 * (NF * (MODE == OP_RESID ? 2.0 : 1.0) + NCd * (J0 ? 2.0 : 1.0));
  const size_t mk = prof_mark(c);
  g_launch_line = __LINE__;
  switch (L.b) {
#define HD_CASE(BB) \
  case BB: launch_sr<BB, MODE, KIND, PLANAR, J0>(c, L, x, b, drop, nc, outc, outp, Lc, omega, x0c); break;
    HD_CASE(1) HD_CASE(2) HD_CASE(3) HD_CASE(4) HD_CASE(5) HD_CASE(6)
#undef HD_CASE
    default: throw Error(HD_ERR_INVALID, "band half-width " + std::to_string(L.b) + " unsupported");
  }
  launched(c, L.n == c->n ? HD_K_OP_FINE : HD_K_OP_COARSE, mk, bytes);
}

// interleaved <-> planar (re plane, im plane) complex vectors
__global__ void k_to_planar(const double2* __restrict__ a, double* __restrict__ p, size_t N) {
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < N; g += (size_t)gridDim.x * blockDim.x) {
    const double2 v = a[g];
    p[g] = v.x;
    p[g + N] = v.y;
  }
}
__global__ void k_from_planar(const double* __restrict__ p, double2* __restrict__ a, size_t N) {
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < N; g += (size_t)gridDim.x * blockDim.x)
    a[g] = cmk(p[g], p[g + N]);
}

// y = Ainv x (dense exact solve of the layered field), interleaved
static void dense_apply(hd_ctx* c, const ExactSolver& X, const double2* x, double2* y) {
  const cuDoubleComplex one = make_cuDoubleComplex(1.0, 0.0), zero = make_cuDoubleComplex(0.0, 0.0);
  const size_t mk = prof_mark(c);
  CKB(cublasZgemv(c->cb, CUBLAS_OP_N, static_cast<int>(X.NN), static_cast<int>(X.NN), &one,
                  reinterpret_cast<const cuDoubleComplex*>(X.Ainv), static_cast<int>(X.NN),
                  reinterpret_cast<const cuDoubleComplex*>(x), 1, &zero, reinterpret_cast<cuDoubleComplex*>(y), 1));
  launched(c, HD_K_LIBGEMM, mk, 16.0 * X.NN * X.NN, true);
}

// Block tridiagonal exact solve (btri.cuh), in/out planar.
template <class T, int KR>
static void btri_launch_t(hd_ctx* c, ExactSolver& X) {
  const size_t smem = 4 * static_cast<size_t>(X.bt.m) * sizeof(double);  // two staged vectors
  smem_optin(reinterpret_cast<const void*>(k_btri_solve<T, KR>), smem);
  cudaLaunchConfig_t cfg{};
  cfg.dynamicSmemBytes = smem;
  cfg.gridDim = dim3(c->n_sms);
  cfg.blockDim = dim3(btri_threads(KR * static_cast<int>(sizeof(T) / 8)));
  cfg.stream = c->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_btri_solve<T, KR>, X.bt));
}

static void btri_solve(hd_ctx* c, ExactSolver& X, double* inout) {
  X.bt.io = inout;
  CK(cudaMemsetAsync(X.bt.bar, 0, sizeof(unsigned), c->st));
  const double mm = static_cast<double>(X.bt.m) * X.bt.m * (X.bt_cplx ? 2.0 : 1.0);
  HD_LAUNCH(HD_K_EXACT, 8.0 * mm * (3.0 * X.bt.nb - 1.0) + 32.0 * X.bt.NN,
            if (X.bt_cplx) switch (X.bt_kr) {
              case 8: btri_launch_t<double2, 8>(c, X); break;
              case 16: btri_launch_t<double2, 16>(c, X); break;
              case 24: btri_launch_t<double2, 24>(c, X); break;
              case 32: btri_launch_t<double2, 32>(c, X); break;
              default: btri_launch_t<double2, 48>(c, X); break;
            } else switch (X.bt_kr) {
              case 8: btri_launch_t<double, 8>(c, X); break;
              case 16: btri_launch_t<double, 16>(c, X); break;
              case 24: btri_launch_t<double, 24>(c, X); break;
              case 32: btri_launch_t<double, 32>(c, X); break;
              case 48: btri_launch_t<double, 48>(c, X); break;
              case 64: btri_launch_t<double, 64>(c, X); break;
              default: btri_launch_t<double, 96>(c, X); break;
            });
}

// C = op(A) op(B) (column-major, batched by strides) on the context stream:
// plain dense GEMMs of the fast diagonalisation, cuBLAS DGEMM by default
// (sm_100 DMMA kernels, 299 us per C5 E solve); HD_DGEMM=dmma selects this
// build's own FP64 tensor-core kernel (dgemm.cuh; 331 us at C5, 53 vs 36 us at
// C3 -- it does not beat the library yet).
static bool dgemm_cublas() {
  static const bool on = !(std::getenv("HD_DGEMM") && std::string(std::getenv("HD_DGEMM")) == "dmma");
  return on;
}

template <bool TA, bool TB>
static void dgemm(hd_ctx* c, int M, int N, int K, const double* A, int lda, long long sA, const double* B, int ldb,
                  long long sB, double* C, int ldc, long long sC, int batch, const double* const* Ap = nullptr,
                  const double* const* Bp = nullptr, double* const* Cp = nullptr) {
  const double flops = 2.0 * M * N * K * batch;
  if (Ap && dgemm_cublas()) {
    const double one = 1.0, zero = 0.0;
    const size_t mk = prof_mark(c);
    CKB(cublasDgemmBatched(c->cb, TA ? CUBLAS_OP_T : CUBLAS_OP_N, TB ? CUBLAS_OP_T : CUBLAS_OP_N, M, N, K, &one, Ap,
                           lda, Bp, ldb, &zero, const_cast<double**>(Cp), ldc, batch));
    launched(c, HD_K_LIBGEMM, mk, flops, true);
    return;
  }
  if (dgemm_cublas()) {
    const double one = 1.0, zero = 0.0;
    const size_t mk = prof_mark(c);
    CKB(cublasDgemmStridedBatched(c->cb, TA ? CUBLAS_OP_T : CUBLAS_OP_N, TB ? CUBLAS_OP_T : CUBLAS_OP_N, M, N, K,
                                  &one, A, lda, sA, B, ldb, sB, &zero, C, ldc, sC, batch));
    launched(c, HD_K_LIBGEMM, mk, flops, true);
    return;
  }
  DgemmArgs g{M, N, K, A, B, C, lda, ldb, ldc, sA, sB, sC, Ap, Bp, Cp};
  constexpr size_t sm = DgemmSmem<TA, TB>::bytes;
  // pointer-batched: the folded blocks are n2^2 doubles apart (16-byte aligned when n2 is even)
  const bool al16 = (reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) % 16 == 0 &&
                    (!Ap || ((static_cast<long long>(lda) * K) % 2 == 0 && (static_cast<long long>(ldb) * N) % 2 == 0));
  const bool even = ((M | N | K | lda | ldb) & 1) == 0 && ((sA | sB) & 1) == 0;
  // split K in two when one pass of tiles would leave the 148 SMs unevenly loaded
  const long tiles = static_cast<long>((N + kGBN - 1) / kGBN) * ((M + kGBM - 1) / kGBM) * batch;
  static const int ks_env = std::getenv("HD_DGEMM_KSPLIT") ? std::atoi(std::getenv("HD_DGEMM_KSPLIT")) : 1;
  const int ks = (ks_env == 2 && tiles < 4L * c->n_sms && K >= 8 * kGBK) ? 2 : 1;
  const dim3 grid((N + kGBN - 1) / kGBN, (M + kGBM - 1) / kGBM, batch * ks);
  if (ks == 2) {  // both halves add into C
    if (static_cast<long long>(ldc) == M && (batch == 1 || sC == static_cast<long long>(ldc) * N)) {
      CK(cudaMemsetAsync(C, 0, sizeof(double) * static_cast<size_t>(ldc) * N * batch, c->st));
    } else {
      for (int b = 0; b < batch; ++b)
        CK(cudaMemset2DAsync(C + b * sC, sizeof(double) * ldc, 0, sizeof(double) * M, N, c->st));
    }
  }
  // profiled as FLOPs (kind HD_K_DGEMM): the roofline of this kernel is the FP64 tensor rate
#define HD_DG(V, KS)                                                                      \
  smem_optin(reinterpret_cast<const void*>(k_dgemm<TA, TB, V, KS>), sm);                  \
  HD_LAUNCH(HD_K_DGEMM, flops, k_dgemm<TA, TB, V, KS><<<grid, 128, sm, c->st>>>(g));
  if (al16 && even) {
    if (ks == 2) { HD_DG(2, 2) } else { HD_DG(2, 1) }
  } else {
    if (ks == 2) { HD_DG(1, 2) } else { HD_DG(1, 1) }
  }
#undef HD_DG
}

static void exact_solve_planar(hd_ctx* c, ExactSolver& X, double* inout) {
  if (X.pfd) {
    const int n = X.n, np = X.np;
    // T = V^T [Bre | Bim]  (x modes; leading dimension np)
    dgemm<true, false>(c, n, 2 * n, n, X.V, n, 0, inout, n, 0, X.T1, np, 0, 1);
    PfdArgs a{X.T1, X.pfdF, X.pfdB, n, np};
    const int ng = np / kPG;
    const double tb = 8.0 * n * static_cast<double>(np) * ((X.pfd_kl + 1) + (2 * X.pfd_kl + 1)) + 64.0 * n * np;
    switch (X.pfd_kl) {
#define HD_PFD(KL)                                                                                   \
  case KL:                                                                                         \
    smem_optin(reinterpret_cast<const void*>(k_pfd_ysolve<KL>), pfd_smem<KL>());                    \
    HD_LAUNCH(HD_K_EXACT, tb, k_pfd_ysolve<KL><<<ng, 32, pfd_smem<KL>(), c->st>>>(a));             \
    break;
      HD_PFD(1) HD_PFD(2) HD_PFD(3) HD_PFD(4)
#undef HD_PFD
      default: throw Error(HD_ERR_INVALID, "partial diagonalisation: band half-width");
    }
    // X = V [Yre | Yim]
    dgemm<false, false>(c, n, 2 * n, n, X.V, n, 0, X.T1, np, 0, inout, n, 0, 1);
    return;
  }
  if (X.btri) {
    btri_solve(c, X, inout);
    return;
  }
  if (X.dense) {
    HD_LAUNCH(HD_K_VEC, 32.0 * X.NN, k_from_planar<<<grid_for(X.NN), 256, 0, c->st>>>(inout, X.dx, X.NN));
    dense_apply(c, X, X.dx, X.dy);
    HD_LAUNCH(HD_K_VEC, 32.0 * X.NN, k_to_planar<<<grid_for(X.NN), 256, 0, c->st>>>(X.dy, inout, X.NN));
    return;
  }
  if (X.dim == 2 && X.folded) {
    const int n = X.n, n2 = X.n2;
    const long long nn = static_cast<long long>(n2) * n2;
    HD_LAUNCH(HD_K_EXACT, 32.0 * n * n, k_fold_both<<<dim3((n2 + 255) / 256, n2, 2), 256, 0, c->st>>>(inout, X.F, n, n2));
    // x transform: Hh[yb] rows (2 xb + p) n2 = Vt_xb^T Q[xb][yb][p]  (8 pointer-batched n2^3 GEMMs)
    dgemm<true, false>(c, n2, n2, n2, nullptr, n2, 0, nullptr, n2, 0, nullptr, 4 * n2, 0, 8, X.xf_ptr, X.xf_ptr + 8,
                       const_cast<double* const*>(X.xf_ptr + 16));
    // y transform: R[yb] = Hh[yb] Vt_yb, Hh[yb] (4 n2) x n2 (x parity and plane stacked), batch over yb
    dgemm<false, false>(c, 4 * n2, n2, n2, X.Hh, 4 * n2, 4 * nn, X.Vt, n2, nn, X.R, 4 * n2, 4 * nn, 2);
    HD_LAUNCH(HD_K_EXACT, 48.0 * 4 * nn, k_scale_folded<<<dim3((n2 + 255) / 256, n2, 4), 256, 0, c->st>>>(X.R, X.Dinvf, n2));
    // inverse y: S[yb] = R[yb] Vt_yb^T  (into Hh)
    dgemm<false, true>(c, 4 * n2, n2, n2, X.R, 4 * n2, 4 * nn, X.Vt, n2, nn, X.Hh, 4 * n2, 4 * nn, 2);
    // inverse x: F blocks = Vt_xb Hh[yb] rows (2 xb + p) n2, then both reflections undone
    dgemm<false, false>(c, n2, n2, n2, nullptr, n2, 0, nullptr, 4 * n2, 0, nullptr, n2, 0, 8, X.xi_ptr, X.xi_ptr + 8,
                        const_cast<double* const*>(X.xi_ptr + 16));
    HD_LAUNCH(HD_K_EXACT, 32.0 * n * n, k_unfold_both<<<dim3((n2 + 255) / 256, n2, 2), 256, 0, c->st>>>(X.F, inout, n, n2));
    return;
  }
  if (X.dim == 2) {
    const int n = X.n;
    const long long nn = static_cast<long long>(n) * n;
    // T1 = V^T [Xre | Xim]
    dgemm<true, false>(c, n, 2 * n, n, X.V, n, 0, inout, n, 0, X.T1, n, 0, 1);
    // T2_plane = T1_plane V
    dgemm<false, false>(c, n, n, n, X.T1, n, nn, X.V, n, 0, X.T2, n, nn, 2);
    HD_LAUNCH(HD_K_EXACT, 48.0 * nn, k_fd_scale<<<grid_for(nn), 256, 0, c->st>>>(X.T2, X.Dinv, nn));
    // T1 = V [T2re | T2im]
    dgemm<false, false>(c, n, 2 * n, n, X.V, n, 0, X.T2, n, 0, X.T1, n, 0, 1);
    // out_plane = T1_plane V^T
    dgemm<false, true>(c, n, n, n, X.T1, n, nn, X.V, n, 0, inout, n, nn, 2);
  } else {
    HD_LAUNCH(HD_K_EXACT, 32.0 * X.n,
              bandlu_launch(c->st, X, nullptr, inout, nullptr, inout));
    if (X.seg.P) c->launches += 4;  // segmented sweeps: 5 kernels
  }
}

// coarsest multigrid level: interleaved in/out
static void coarsest_solve(hd_ctx* c, const double2* b, double2* out) {
  ExactSolver& X = c->coarsest;
  if (X.dense) {
    dense_apply(c, X, b, out);
    return;
  }
  const double NL = X.dim == 2 ? static_cast<double>(X.n) * X.n : X.n;
  HD_LAUNCH(HD_K_EXACT, 32.0 * NL,
            if (X.dim == 2) k_fd_small<<<1, 1024, 0, c->st>>>(X.V, X.Dinv, X.n, b, out);
            else bandlu_launch(c->st, X, b, nullptr, out, nullptr));
  if (X.dim != 2 && X.seg.P) c->launches += 4;
}

static size_t lsize(const hd_ctx* c, int n) { return c->dim == 2 ? static_cast<size_t>(n) * n : n; }

// level l of the shifted hierarchy
static LevelDev levM(hd_ctx* c, int l) {
  return level_dev(c->lev[l], c->cM, l == 0 ? c->corner : cmk(0.0, 0.0), c->lev[l].genM);
}

// x_out = (damped Jacobi)^steps from x (x_zero: x == 0), ping-pong through tmp
// x0_ready: xa already holds the first sweep from zero (fused into the producer of b)
// ec (with its grid side nc): the coarse correction still to be prolonged onto x; the first sweep
// then runs on x + Z ec without storing it (OP_JACOBIP)
static double2* smooth(hd_ctx* c, int l, const double2* b, double2* xa, double2* xb, bool x_zero, int steps,
                       bool x0_ready = false, const double2* ec = nullptr, int nc = 0) {
  const LevelDev L = levM(c, l);
  double2* cur = xa;
  double2* oth = xb;
  int s = 0;
  if (ec) {  // caller guarantees steps >= 1 and a 2D Kronecker-sum level
    launch_op2d_mode<OP_JACOBIP>(c, L, cur, b, oth, c->spec.omega, red_of(c), L.n == c->n ? HD_K_OP_FINE : HD_K_OP_COARSE,
                                 nullptr, 0, 0, -1, nullptr, double2{0.0, 0.0}, ec, nc);
    std::swap(cur, oth);
    s = 1;
  }
  if (x_zero) {
    if (steps == 0) {
      CK(cudaMemsetAsync(cur, 0, lsize(c, L.n) * sizeof(double2), c->st));
      return cur;
    }
    if (!x0_ready) jacobi0(c, L, b, cur, c->spec.omega);
    s = 1;
  }
  for (; s < steps; ++s) {
    op_apply(c, OP_JACOBI, L, cur, b, oth, c->spec.omega);
    std::swap(cur, oth);
  }
  return cur;
}

// One V-cycle at level l (src/precond.cpp:144-153); returns the buffer holding x.
// True when level l's first sweep from zero can ride with the kernel that
// produces its right-hand side: a 2D Kronecker-sum level that is smoothed
// (not the coarsest, not the 1D tail, not a layered/wedge level).
static bool j0_fusable(hd_ctx* c, int l) {
  const bool off = !c->j0_fuse;
  const int last = static_cast<int>(c->lev.size()) - 1;
  return !off && c->dim == 2 && l < last && l != c->tail_l && c->spec.smooth_steps >= 1 && !c->lev[l].genM &&
         !c->fine.genA;
}

// x0_ready: mg_x[l] already holds omega D^-1 b (see smooth)
static double2* cycle_at(hd_ctx* c, int l, const double2* b, bool x_zero, bool x0_ready = false) {
  const int last = static_cast<int>(c->lev.size()) - 1;
  if (l == c->tail_l && x_zero) {  // 1D: the remaining levels in one single-CTA kernel
    double nb = 0.0;
    for (int t = 0; t < c->tail.nl; ++t) nb += 64.0 * c->tail.n[t];
    HD_LAUNCH(HD_K_OP_COARSE, nb,
              k_tail1d<<<1, kTailThreads, c->tail_smem_bytes, c->st>>>(c->tail, b, c->mg_x[l]));
    return c->mg_x[l];
  }
  if (l == last) {
    coarsest_solve(c, b, c->mg_x[l]);
    return c->mg_x[l];
  }
  const LevelDev L = levM(c, l);
  double2* xcur = smooth(c, l, b, c->mg_x[l], c->mg_y[l], x_zero, c->spec.smooth_steps, x0_ready && x_zero);
  double2* xoth = xcur == c->mg_x[l] ? c->mg_y[l] : c->mg_x[l];
  const int nf = c->lev[l].n, ncl = c->lev[l + 1].n;
  const bool fuse = j0_fusable(c, l + 1);
  // residual + restriction (+ the coarse first sweep) in one pass on the levels with a
  // 2-wide band; at the p = 3 fine level the fused kernel (up to 174 registers) measured
  // 62 us against 52 us for the separate residual and restriction (ncu, C5), so it is split there
  if (fused_restrict_ok(c, L) && L.b <= 2) {
    if (fuse)
      op_restrict<OP_RESID, 0, 0, true>(c, L, xcur, b, 0.0, ncl, c->mg_b[l + 1], nullptr, levM(c, l + 1),
                                        c->spec.omega, c->mg_x[l + 1]);
    else
      op_restrict<OP_RESID, 0, 0, false>(c, L, xcur, b, 0.0, ncl, c->mg_b[l + 1], nullptr);
  } else {
    op_apply(c, OP_RESID, L, xcur, b, c->mg_r[l]);
    if (fuse) restrict_j0(c, c->mg_r[l], nf, ncl, c->mg_b[l + 1], levM(c, l + 1), c->spec.omega, c->mg_x[l + 1]);
    else restrict_(c, Stencil{0, 0.0}, c->mg_r[l], nf, ncl, c->mg_b[l + 1], nullptr);
  }
  double2* ec = cycle_at(c, l + 1, c->mg_b[l + 1], true, fuse);
  // prolongation + first post-smoothing sweep in one pass (K4) on 2D Kronecker-sum levels
  if (c->k4_fuse && c->dim == 2 && !L.gen && c->spec.smooth_steps >= 1 && L.b <= 6)
    return smooth(c, l, b, xcur, xoth, false, c->spec.smooth_steps, false, ec, ncl);
  prolong_<0>(c, Stencil{0, 0.0}, ec, nullptr, nf, ncl, nullptr, xcur);
  double2* res = smooth(c, l, b, xcur, xoth, false, c->spec.smooth_steps);
  return res;
}

// out = M^-1 b exactly (C_ex, src/precond.cpp:204-211): fast diagonalisation
// of the shifted Kronecker sum on the fine level (2D) or banded LU (1D)
static void shift_exact_solve(hd_ctx* c, const double2* b, double2* out) {
  const size_t N = c->N;
  ExactSolver& X = c->shift_exact;
  if (X.dim == 2) {
    HD_LAUNCH(HD_K_VEC, 32.0 * N, k_to_planar<<<grid_for(N), 256, 0, c->st>>>(b, c->sx_plan, N));
    exact_solve_planar(c, X, c->sx_plan);
    HD_LAUNCH(HD_K_VEC, 32.0 * N, k_from_planar<<<grid_for(N), 256, 0, c->st>>>(c->sx_plan, out, N));
  } else {
    HD_LAUNCH(HD_K_EXACT, 32.0 * X.n,
              bandlu_launch(c->st, X, b, nullptr, out, nullptr));
    if (X.seg.P) c->launches += 4;
  }
}

// MG^-1 b (Multigrid::solve, src/precond.cpp:159-163).  Returns the buffer that
// holds the result: `out` for C_ex, else the level-0 iterate buffer (mg_x[0] or
// mg_y[0]), valid until the next multigrid application.
static const double2* mg_solve_ptr(hd_ctx* c, const double2* b, double2* out, bool x0_ready = false) {
  const size_t N = c->N;
  if (c->spec.cycles <= 0) {
    shift_exact_solve(c, b, out);
    return out;
  }
  bool zero = true;
  double2* xb = nullptr;
  for (int cy = 0; cy < c->spec.cycles; ++cy) {
    if (!zero) {
      // level-0 iterate must live in mg_x[0] for the next cycle
      if (xb != c->mg_x[0]) CK(cudaMemcpyAsync(c->mg_x[0], xb, N * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
    }
    if (c->lev.size() == 1) {
      coarsest_solve(c, b, c->mg_x[0]);
      xb = c->mg_x[0];
    } else if (zero) {
      xb = cycle_at(c, 0, b, true, x0_ready);
    } else {
      // general cycle from a non-zero iterate held in mg_x[0]
      const LevelDev L = levM(c, 0);
      double2* xcur = smooth(c, 0, b, c->mg_x[0], c->mg_y[0], false, c->spec.smooth_steps);
      double2* xoth = xcur == c->mg_x[0] ? c->mg_y[0] : c->mg_x[0];
      if (fused_restrict_ok(c, L) && L.b <= 2) {
        op_restrict<OP_RESID, 0, 0, false>(c, L, xcur, b, 0.0, c->lev[1].n, c->mg_b[1], nullptr);
      } else {
        op_apply(c, OP_RESID, L, xcur, b, c->mg_r[0]);
        restrict_(c, Stencil{0, 0.0}, c->mg_r[0], c->lev[0].n, c->lev[1].n, c->mg_b[1], nullptr);
      }
      double2* ec = cycle_at(c, 1, c->mg_b[1], true);
      if (c->k4_fuse && c->dim == 2 && !L.gen && c->spec.smooth_steps >= 1 && L.b <= 6) {
        xb = smooth(c, 0, b, xcur, xoth, false, c->spec.smooth_steps, false, ec, c->lev[1].n);
      } else {
        prolong_<0>(c, Stencil{0, 0.0}, ec, nullptr, c->lev[0].n, c->lev[1].n, nullptr, xcur);
        xb = smooth(c, 0, b, xcur, xoth, false, c->spec.smooth_steps);
      }
    }
    zero = false;
  }
  return xb;
}

static void mg_solve(hd_ctx* c, const double2* b, double2* out) {
  const double2* r = mg_solve_ptr(c, b, out);
  if (r != out) CK(cudaMemcpyAsync(out, r, c->N * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
}


static LevelDev opA(hd_ctx* c) { return level_dev(c->fine, c->cA, c->corner, c->fine.genA); }

// out = Q v = Z E^-1 Z^T v  (Deflation::apply_Q, src/precond.cpp:102-104)
static void apply_Q(hd_ctx* c, const double2* v, double2* out) {
  const Stencil z{1, c->spec.drop};
  restrict_(c, z, v, c->n, c->nc, nullptr, c->ep);
  exact_solve_planar(c, c->E, c->ep);
  prolong_<2>(c, z, nullptr, c->ep, c->n, c->nc, nullptr, out);
}

// out = w - Q (A w)  (Deflation::project, src/precond.cpp:106-108)
static void project(hd_ctx* c, const double2* w, double2* out) {
  const Stencil z{1, c->spec.drop};
  const LevelDev A = opA(c);
  if (fused_restrict_ok(c, A)) {  // Z^T (A w) in one pass, A w never stored
    op_restrict<OP_APPLY, 1, 1, false>(c, A, w, nullptr, c->spec.drop, c->nc, nullptr, c->ep);
  } else {
    op_apply(c, OP_APPLY, A, w, nullptr, c->t3);
    restrict_(c, z, c->t3, c->n, c->nc, nullptr, c->ep);
  }
  exact_solve_planar(c, c->E, c->ep);
  prolong_<1>(c, z, nullptr, c->ep, c->n, c->nc, w, out);
}

// out = op(v) = P MG^-1 A v  (src/precond.cpp:236-245); v, out distinct from t1, t2, t3
static void compose_op(hd_ctx* c, const double2* v, double2* out, const int* vidx = nullptr) {
  NvtxRange nvtx_op("op = P MG^-1 A");
  ++c->matvecs;
  // A v also takes the fine level's first Jacobi sweep of the V-cycle (OP_APPLYJ0)
  const bool fuse = c->spec.shift && c->spec.cycles >= 1 && c->lev.size() > 1 && j0_fusable(c, 0);
  if (fuse) {
    RedOut red = red_of(c);
    launch_op2d_mode<OP_APPLYJ0>(c, opA(c), v, nullptr, c->t1, c->spec.omega, red, HD_K_OP_FINE, vidx, c->N, 0, -1,
                                 c->mg_x[0], c->cM);
  } else {
    op_apply(c, OP_APPLY, opA(c), v, nullptr, c->t1, 0.0, nullptr, 1.0, vidx, c->N);
  }
  const double2* cur = c->t1;
  if (c->spec.shift) {
    NvtxRange nvtx_mg("MG^-1 (V-cycles / C_ex)");
    ++c->shift_solves;
    c->vcycles += c->spec.cycles;
    cur = mg_solve_ptr(c, c->t1, c->t2, fuse);  // no copy: project reads it before the next V-cycle
  }
  if (c->spec.deflate) {
    NvtxRange nvtx_p("project (Z^T A, E^-1, Z)");
    ++c->coarse_solves;
    project(c, cur, out);
  } else {
    CK(cudaMemcpyAsync(out, cur, c->N * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
  }
}

static void ensure_gmres(hd_ctx* c, int maxit) {
  // every branch below that reallocates moves pointers the loop / prelude graphs captured
  if (maxit + 1 > c->v_cap) {
    ++c->buf_epoch;
    dfree(c->V);
    c->V = dalloc<double2>(static_cast<size_t>(maxit + 1) * c->N);
    c->v_cap = maxit + 1;
  }
  if (maxit > c->maxit_cap) {
    ++c->buf_epoch;
    dfree(c->H); dfree(c->g); dfree(c->cs); dfree(c->sn); dfree(c->y);
    c->H = dalloc<double2>(static_cast<size_t>(maxit + 1) * maxit);
    c->g = dalloc<double2>(maxit + 1);
    c->cs = dalloc<double2>(maxit);
    c->sn = dalloc<double2>(maxit);
    c->y = dalloc<double2>(maxit);
    c->maxit_cap = maxit;
  }
  if (maxit != c->lsa_maxit && maxit + 1 <= kLsaMaxJ) {
    ++c->buf_epoch;
    int sms = 0, per = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    smem_optin(reinterpret_cast<const void*>(k_lsa_dots), lsa_dots_smem());
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_lsa_dots, kLsaBD, lsa_dots_smem()));
    int per2 = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_lsa_update, kLsaBD, 0));
    per = std::max(1, std::min(per, per2));
    const size_t tiles = (c->N + static_cast<size_t>(kLsaBD) * kLsaTE - 1) / (static_cast<size_t>(kLsaBD) * kLsaTE);
    c->lsa_G = static_cast<int>(std::max<size_t>(1, std::min<size_t>(tiles, static_cast<size_t>(sms) * per)));
    dfree(c->lsa_sig); dfree(c->lsa_L); dfree(c->lsa_ch); dfree(c->lsa_cx); dfree(c->lsa_partials);
    c->lsa_sig = dalloc<double>(maxit + 2);
    c->lsa_L = dalloc<double2>(static_cast<size_t>(maxit + 1) * (maxit + 1));
    c->lsa_ch = dalloc<double2>(maxit + 2);
    c->lsa_cx = dalloc<double2>(maxit + 2);
    c->lsa_partials = dalloc<double2>(static_cast<size_t>(c->lsa_G) * (2 * kLsaMaxJ + 2) + 8);
    if (!c->lsa_counter) {
      c->lsa_counter = dalloc<unsigned>(4);
      CK(cudaMemset(c->lsa_counter, 0, 4 * sizeof(unsigned)));
    }
    const int m = maxit + 1;
    c->lsa_givens_smem = (static_cast<size_t>(m) * (m + 1) / 2 + 4 * (m + 2) + 8) * sizeof(double2);
    smem_optin(reinterpret_cast<const void*>(k_lsa_givens), c->lsa_givens_smem);
    c->lsa_maxit = maxit;
  }
}

// pass 1 of the one-reduction Arnoldi: the register-streaming k_lsa_dots, or
// (HD_LSA_TMA=1 at create) the bulk-copy ring kernel -- equal at C5 (48.6 vs
// 48.3 ms for both passes over a solve), so the round-1 kernel stays the default
static void launch_lsa_dots(hd_ctx* c, const LsaArgs& a, int G, cudaStream_t st) {
  if (c->lsa_mma) {  // one CTA per SM (never more CTAs than the partials buffer has slots)
    smem_optin(reinterpret_cast<const void*>(k_lsa_dots_mma), lsa_mma_smem());
    // the basis as a 2D tensor (2N doubles x v_cap vectors), box = kMmaTE elements x 8 vectors
    const hd_ctx::TmaKey key{a.U, static_cast<int>(a.N), c->v_cap, -kMmaTE};
    auto it = c->tma_maps.find(key);
    if (it == c->tma_maps.end()) {
      CUtensorMap m;
      const cuuint64_t dims[2] = {static_cast<cuuint64_t>(2) * a.N, static_cast<cuuint64_t>(c->v_cap)};
      const cuuint64_t strides[1] = {static_cast<cuuint64_t>(16) * a.N};
      const cuuint32_t box[2] = {2 * kMmaTE, 8};
      const cuuint32_t es[2] = {1, 1};
      const CUresult r = tma_encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double2*>(a.U), dims, strides, box,
                                         es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) throw Error(HD_ERR_CUDA, "cuTensorMapEncodeTiled (basis) failed: " + std::to_string(static_cast<int>(r)));
      it = c->tma_maps.emplace(key, m).first;
    }
    k_lsa_dots_mma<<<std::min(c->n_sms, G), kLsaBD, lsa_mma_smem(), st>>>(a, it->second);
  } else if (c->lsa_tma) {
    smem_optin(reinterpret_cast<const void*>(k_lsa_dots_tma), lsa_tma_smem());
    // one CTA per SM, never more CTAs than the partials buffer has slots (lsa_G)
    k_lsa_dots_tma<<<std::min(c->n_sms, G), kTNW * 32, lsa_tma_smem(), st>>>(a);
  } else {
    k_lsa_dots<<<G, kLsaBD, lsa_dots_smem(), st>>>(a);
  }
}

static LsaArgs lsa_args(hd_ctx* c, double2* xout, int j, int mode, int maxit) {
  LsaArgs a;
  a.jlag = 0;
  a.part_offset = 0;
  a.partial_only = 0;
  a.rev = c->lsa_rev ? 1 : 0;
  a.U = c->V;
  a.Uw = c->V;
  a.w = c->w;
  a.x0 = c->x0;
  a.x = xout;
  a.N = c->N;
  a.j = j;
  a.mode = mode;
  a.sig = c->lsa_sig;
  a.L = c->lsa_L;
  a.ldl = maxit + 1;
  a.H = c->H;
  a.ldh = maxit + 1;
  a.g = c->g;
  a.cs = c->cs;
  a.sn = c->sn;
  a.ch = c->lsa_ch;
  a.cx = c->lsa_cx;
  a.hnew_out = c->dres + 1;
  a.partials = c->lsa_partials;
  a.counter = c->lsa_counter;
  a.done = nullptr;
  a.dj = nullptr;
  return a;
}

__global__ void k_inv_scalar(double* dst, const double* src) { *dst = *src > 0.0 ? 1.0 / *src : 0.0; }

static void read_scalars(hd_ctx* c) {
  CK(cudaMemcpyAsync(c->hres, c->dres, 4 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
}

__global__ void k_loop_init(LoopState* s) {
  s->j = 0;
  s->done = 0;
  s->iters = 0;
  s->conv = 0;
  s->need_tail = 0;
  s->breakdown = 0;
  s->nonfinite = 0;
  s->hprev = 1.0;
}

__global__ void k_scale_monitor(double* dres) {
  // graph monitor: raw norm / (||f|| or 1)
  const double f = dres[3];
  dres[0] = dres[0] / (f > 0.0 ? f : 1.0);
}

static void monitor_raw(hd_ctx* c, const double2* x) {
  op_apply(c, OP_RESNORM, opA(c), x, c->f, nullptr, 0.0, c->dres + 0, 1.0);
}

// Captures the GMRES iteration body (device-side j) into the body of a WHILE
// conditional node: op(u_j) -> pass 1 (dots, x_{j-1}) -> monitor x_{j-1} ->
// convergence check -> pass 2 (u_{j+1}) -> Givens -> j++.
static void build_loop_graph(hd_ctx* c, int maxit, double tol) {
  if (c->loop_exec) cudaGraphExecDestroy(c->loop_exec);
  if (c->loop_graph) cudaGraphDestroy(c->loop_graph);
  c->loop_exec = nullptr;
  c->loop_graph = nullptr;
  if (!c->loop_state) {
    c->loop_state = dalloc<LoopState>(1);
    CK(cudaMallocHost(&c->loop_host, sizeof(LoopState)));
  }
  dfree(c->res_hist);
  if (c->res_host) cudaFreeHost(c->res_host);
  c->res_hist = dalloc<double>(maxit + 1);
  CK(cudaMallocHost(&c->res_host, (maxit + 1) * sizeof(double)));
  const long saved[4] = {c->matvecs, c->coarse_solves, c->shift_solves, c->vcycles};
  const int saved_l = c->launches, saved_b = c->lib_calls;
  const bool prof = c->prof_on;
  c->prof_on = false;
  cudaGraph_t g;
  CK(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, nullptr, 0, &p));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(c->st, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  const int G = c->lsa_G;
  int* dj = &c->loop_state->j;
  LsaArgs a = lsa_args(c, c->x, 0, 0, maxit);
  a.dj = dj;
  a.done = &c->loop_state->done;
  // side branch: the Givens rotation + back substitution of iteration j-1
  // (needed first by pass 2 of iteration j) overlaps the operator of iteration j
  if (!c->st2) {
    CK(cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  }
  CK(cudaEventRecord(c->ev_fork, c->st));
  CK(cudaStreamWaitEvent(c->st2, c->ev_fork, 0));
  LsaArgs ag = a;
  ag.jlag = 1;
  k_lsa_givens<<<1, kLsaBD, c->lsa_givens_smem, c->st2>>>(ag, G);
  if (c->mon_side) {
    // side branch, after the Givens: monitor x_{j-2} (written by pass 2 of the
    // previous body) with its own reduction scratch, record it, stop on tolerance
    std::swap(c->st, c->st2);
    std::swap(c->partials, c->mon_partials);
    std::swap(c->counter, c->mon_counter);
    monitor_raw(c, c->x);
    std::swap(c->st, c->st2);
    std::swap(c->partials, c->mon_partials);
    std::swap(c->counter, c->mon_counter);
    k_scale_monitor<<<1, 1, 0, c->st2>>>(c->dres);
    k_loop_check_lag2<<<1, 1, 0, c->st2>>>(c->loop_state, c->dres, c->res_hist, tol, h);
  }
  CK(cudaEventRecord(c->ev_join, c->st2));
  compose_op(c, c->V, c->w, dj);
  CK(cudaStreamWaitEvent(c->st, c->ev_join, 0));
  launch_lsa_dots(c, a, G, c->st);
  k_lsa_update<<<G, kLsaBD, 0, c->st>>>(a);  // u_{j+1} and the lagged x_{j-1}
  if (c->mon_side) {
    k_loop_breakdown<<<1, 1, 0, c->st>>>(c->loop_state, c->dres, h);
    k_loop_next<<<1, 1, 0, c->st>>>(c->loop_state, maxit, h);
  } else {
    monitor_raw(c, c->x);
    k_loop_step<<<1, 1, 0, c->st>>>(c->loop_state, c->dres, c->res_hist, tol, maxit, h);  // scale, check, next
  }
  cudaGraph_t captured = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(c->st, &captured);
  c->prof_on = prof;
  // op + monitor kernels + givens/dots/update/step (side monitor: scale/check/breakdown/next instead of step)
  c->graph_body_kernels = c->launches - saved_l + (c->mon_side ? 7 : 4);
  c->matvecs = saved[0];
  c->coarse_solves = saved[1];
  c->shift_solves = saved[2];
  c->vcycles = saved[3];
  c->launches = saved_l;
  c->lib_calls = saved_b;
  CK(ec);
  CK(cudaGetLastError());
  CK(cudaGraphInstantiate(&c->loop_exec, g, 0));
  c->loop_graph = g;
  c->loop_maxit = maxit;
  c->loop_tol = tol;
  c->loop_epoch = c->buf_epoch;
}

struct SolveOut {
  int iterations = 0;
  bool converged = false;
  std::vector<double> residuals;
};

// gmres(setup.op, setup.rhs, setup.start, setup.monitor, opt) after the
// compose() right-hand side / start transforms; f already in c->f.
// small 1D systems: the whole solve in one single-CTA kernel (small1d.cuh);
// the counters follow the reference's call pattern (compose: rhs and start,
// then one op per GMRES step plus the initial residual's)
static SolveOut run_solve_small1d(hd_ctx* c, const hd_gmres& opt, double2* xout) {
  const int maxit = opt.max_iterations;
  ensure_gmres(c, std::max(maxit, 1));
  c->matvecs = c->coarse_solves = c->shift_solves = c->vcycles = 0;
  c->launches = c->lib_calls = 0;
  SmallArgs a = c->small;
  a.maxit = maxit;
  a.tol = opt.tolerance;
  a.f = c->f;
  a.x = xout;
  a.V = c->V;
  a.H = c->H;
  a.res = c->small_res;
  a.state = c->small_state;
  const size_t smem = small_smem(a);
  smem_optin(reinterpret_cast<const void*>(k_solve1d_small), smem);
  // one warp per 32 unknowns (64..512 threads): fewer warps make the block barriers cheaper
  const int threads = static_cast<int>(std::min<size_t>(kSmallThreads, std::max<size_t>(64, (c->N + 31) / 32 * 32)));
  HD_LAUNCH(HD_K_OP_FINE, 16.0 * c->N * 10.0, k_solve1d_small<<<1, threads, smem, c->st>>>(a));
  int st[4] = {0, 0, 0, 0};
  std::vector<double> res(static_cast<size_t>(maxit) + 1, 0.0);
  CK(cudaMemcpyAsync(st, c->small_state, 3 * sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(res.data(), c->small_res, res.size() * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  const long cyc = c->spec.shift && c->spec.cycles > 0 ? c->spec.cycles : 0;
  auto one_op = [&]() {  // compose_op's counters
    ++c->matvecs;
    if (c->spec.shift) {
      ++c->shift_solves;
      c->vcycles += cyc;
    }
    if (c->spec.deflate) ++c->coarse_solves;
  };
  if (c->spec.shift) {  // rhs' = P MG^-1 f
    ++c->shift_solves;
    c->vcycles += cyc;
  }
  if (c->spec.deflate) c->coarse_solves += 2;  // project(rhs'), start = Q f
  SolveOut r;
  if (st[2] == 1) {  // monitor(x0) <= tol
    r.converged = true;
    r.residuals.push_back(res[0]);
    return r;
  }
  one_op();  // r = rhs' - op(x0)
  if (st[2] == 2) {  // beta == 0
    r.converged = st[1] != 0;
    return r;
  }
  r.iterations = st[0];
  r.converged = st[1] != 0;
  for (int j = 0; j < r.iterations; ++j) {
    r.residuals.push_back(res[j]);
    one_op();
  }
  return r;
}

static SolveOut run_solve(hd_ctx* c, const hd_gmres& opt, double2* xout) {
  if (c->small_ok && opt.max_iterations >= 1 && opt.max_iterations + 1 <= kLsaMaxJ && !c->prof_on)
    return run_solve_small1d(c, opt, xout);
  const size_t N = c->N;
  const int maxit = opt.max_iterations;
  ensure_gmres(c, std::max(maxit, 1));
  c->matvecs = c->coarse_solves = c->shift_solves = c->vcycles = 0;
  c->launches = c->lib_calls = 0;
  const int nb = c->red_blocks;
  const double P = 16.0 * static_cast<double>(N);
  // The prelude up to the one host synchronisation (no host decisions inside) is
  // captured once per context as a graph and replayed: small systems are
  // launch-bound there.  Counter and launch deltas of the capture are replayed too.
  long* cnt[4] = {&c->matvecs, &c->coarse_solves, &c->shift_solves, &c->vcycles};
  long snap0[4] = {0, 0, 0, 0};  // counters before the speculative op(x0)
  auto prelude = [&]() {
    NvtxRange nvtx_pre("GMRES prelude (rhs', x0, monitor, op(x0), beta)");
    // ||f|| (monitor scale, src/precond.cpp:258)
    HD_LAUNCH(HD_K_VEC, P, k_axpy_norm<<<nb, 256, 0, c->st>>>(c->f, nullptr, nullptr, N, red_of(c, c->dres + 3), c->scal + 2));
    // rhs' = P MG^-1 f   (src/precond.cpp:247-253)
    const double2* b = c->f;
    if (c->spec.shift) {
      ++c->shift_solves;
      c->vcycles += c->spec.cycles;
      mg_solve(c, c->f, c->t2);
      b = c->t2;
    }
    if (c->spec.deflate) {
      ++c->coarse_solves;
      project(c, b, c->rhsp);
    } else {
      CK(cudaMemcpyAsync(c->rhsp, b, N * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
    }
    // start = Q f (src/precond.cpp:255-256)
    if (c->spec.deflate) {
      apply_Q(c, c->f, c->x0);
      ++c->coarse_solves;
    } else {
      CK(cudaMemsetAsync(c->x0, 0, N * sizeof(double2), c->st));
    }
    // ||f||, monitor(x0) (scaled on the device, as in the graph body) and beta are
    // read with one host synchronisation after the prelude.  The operator of x0 is
    // speculative until monitor(x0) > tol is known; its counts are rolled back.
    monitor_raw(c, c->x0);
    HD_LAUNCH(HD_K_VEC, 0.0, k_scale_monitor<<<1, 1, 0, c->st>>>(c->dres));
    for (int q = 0; q < 4; ++q) snap0[q] = *cnt[q];
    // r = rhs' - op(x0); beta = ||r||; V0 = r / beta  (src/linalg.cpp:24-33)
    compose_op(c, c->x0, c->w);
    HD_LAUNCH(HD_K_VEC, 3 * P, k_sub<<<grid_for(N), 256, 0, c->st>>>(c->rhsp, c->w, c->w, N));
    HD_LAUNCH(HD_K_VEC, P, k_axpy_norm<<<nb, 256, 0, c->st>>>(c->w, nullptr, nullptr, N, red_of(c, c->dres + 2), c->g));
  };
  if (c->graph_enabled && !c->prof_on && c->pre_graph) {
    if (!c->pre_exec || c->pre_epoch != c->buf_epoch) {
      if (c->pre_exec) cudaGraphExecDestroy(c->pre_exec);
      c->pre_exec = nullptr;
      const long c0[4] = {*cnt[0], *cnt[1], *cnt[2], *cnt[3]};
      const int l0 = c->launches, b0 = c->lib_calls;
      cudaGraph_t pg = nullptr;
      CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeRelaxed));
      prelude();
      const cudaError_t ec = cudaStreamEndCapture(c->st, &pg);
      CK(ec);
      CK(cudaGraphInstantiate(&c->pre_exec, pg, 0));
      CK(cudaGraphDestroy(pg));
      for (int q = 0; q < 4; ++q) {
        c->pre_dcnt[q] = *cnt[q] - c0[q];
        c->pre_dsnap[q] = snap0[q] - c0[q];
        *cnt[q] = c0[q];
      }
      c->pre_dl = c->launches - l0;
      c->pre_db = c->lib_calls - b0;
      c->launches = l0;
      c->lib_calls = b0;
      c->pre_epoch = c->buf_epoch;
    }
    for (int q = 0; q < 4; ++q) {
      snap0[q] = *cnt[q] + c->pre_dsnap[q];
      *cnt[q] += c->pre_dcnt[q];
    }
    c->launches += c->pre_dl;
    c->lib_calls += c->pre_db;
    CK(cudaGraphLaunch(c->pre_exec, c->st));
  } else {
    prelude();
  }
  read_scalars(c);
  const double fnorm = c->hres[3];
  const double scale = fnorm > 0.0 ? fnorm : 1.0;

  SolveOut res;
  auto monitor = [&](const double2* xv) {
    op_apply(c, OP_RESNORM, opA(c), xv, c->f, nullptr, 0.0, c->dres + 0, scale);
  };
  const double r0 = c->hres[0];
  if (r0 <= opt.tolerance) {  // src/linalg.cpp:17-22
    c->matvecs = snap0[0];
    c->coarse_solves = snap0[1];
    c->shift_solves = snap0[2];
    c->vcycles = snap0[3];
    res.converged = true;
    res.residuals.push_back(r0);
    CK(cudaMemcpyAsync(xout, c->x0, N * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
    return res;
  }
  const double beta = c->hres[2];
  if (beta == 0.0) {  // the reference monitors x0 again: the same r0 > tol
    res.converged = false;
    CK(cudaMemcpyAsync(xout, c->x0, N * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
    return res;
  }
  CK(cudaMemsetAsync(c->H, 0, sizeof(double2) * (maxit + 1) * maxit, c->st));
  CK(cudaMemsetAsync(c->g + 1, 0, sizeof(double2) * maxit, c->st));
  HD_LAUNCH(HD_K_VEC, 2 * P, k_scale_inv<<<grid_for(N), 256, 0, c->st>>>(c->V, c->w, c->dres + 2, N));
  const int ldh = maxit + 1;
  if (c->arn_mode == 1 && maxit + 1 <= kLsaMaxJ) {
    // u_0 = r (unnormalised), sigma_0 = 1 / beta
    CK(cudaMemcpyAsync(c->V, c->w, N * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
    HD_LAUNCH(HD_K_VEC, 0.0, k_inv_scalar<<<1, 1, 0, c->st>>>(c->lsa_sig, c->dres + 2));
    const int G = c->lsa_G;
    if (c->graph_enabled && !c->prof_on) {
      if (c->loop_maxit != maxit || c->loop_tol != opt.tolerance || c->loop_epoch != c->buf_epoch)
        build_loop_graph(c, maxit, opt.tolerance);
      NvtxRange nvtx_loop("GMRES loop (device-resident graph)");
      k_loop_init<<<1, 1, 0, c->st>>>(c->loop_state);
      CK(cudaGraphLaunch(c->loop_exec, c->st));
      CK(cudaMemcpyAsync(c->loop_host, c->loop_state, sizeof(LoopState), cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(c->res_host, c->res_hist, maxit * sizeof(double), cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      const LoopState ls = *c->loop_host;
      if (ls.nonfinite)
        throw Error(HD_ERR_NONFINITE, "non-finite residual or Arnoldi norm at GMRES iteration " + std::to_string(ls.iters));
      // per-iteration launches of the body (op + 7) for the report
      int it = ls.iters;
      res.iterations = it;
      res.converged = ls.conv != 0;
      const int lag = c->mon_side ? 2 : 1;  // monitors recorded by the graph trail the iterate by lag - 1
      const int recorded = ls.conv ? it : ls.need_tail ? std::max(0, maxit - lag) : it - (lag - 1);
      for (int q = 0; q < recorded; ++q) res.residuals.push_back(c->res_host[q]);
      bool tail = ls.need_tail != 0;
      if (c->mon_side && ((ls.need_tail && maxit >= 2) || ls.breakdown)) {
        // x_{it-1} (breakdown) or x_{maxit-2} (budget) is formed but its monitor is not recorded yet
        monitor(c->x);
        read_scalars(c);
        res.residuals.push_back(c->hres[0]);
        if (c->hres[0] <= opt.tolerance) {
          res.converged = true;
          if (tail) it = res.iterations = maxit - 1;
          tail = false;
        }
      }
      if (tail) {  // x_{maxit-1}: its Givens, an iterate-only pass + monitor
        LsaArgs b = lsa_args(c, c->x, maxit - 1, 1, maxit);
        HD_LAUNCH(HD_K_GIVENS, 0.0, k_lsa_givens<<<1, kLsaBD, c->lsa_givens_smem, c->st>>>(b, G));
        HD_LAUNCH(HD_K_ITERATE, (maxit + 2.0) * P, k_lsa_update<<<G, kLsaBD, 0, c->st>>>(b));
        monitor(c->x);
        read_scalars(c);
        res.residuals.push_back(c->hres[0]);
        res.converged = c->hres[0] <= opt.tolerance;
      }
      c->matvecs += it;
      if (c->spec.shift) {
        c->shift_solves += it;
        c->vcycles += static_cast<long>(it) * c->spec.cycles;
      }
      if (c->spec.deflate) c->coarse_solves += it;
      c->launches += (it + 1) * (c->graph_body_kernels);
      if (xout != c->x) CK(cudaMemcpyAsync(xout, c->x, N * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
      return res;
    }
    bool stop = false;
    double hnew_prev = 1.0;
    for (int j = 0; j < maxit && !stop; ++j) {
      // the op of iteration j is speculative until x_{j-1} is known not to
      // have converged; its counts are rolled back if GMRES stops at j-1
      const long snap[4] = {c->matvecs, c->coarse_solves, c->shift_solves, c->vcycles};
      auto rollback = [&]() {
        c->matvecs = snap[0];
        c->coarse_solves = snap[1];
        c->shift_solves = snap[2];
        c->vcycles = snap[3];
      };
      compose_op(c, c->V + static_cast<size_t>(j) * N, c->w);
      LsaArgs a = lsa_args(c, xout, j, 0, maxit);
      // pass 1 reads w, u_j, u_0..u_j; pass 2 reads w, u_0..u_j (+ x0 for j >= 1), writes u_{j+1} (+ x)
      {
        NvtxRange nvtx_a("Arnoldi passes");
        HD_LAUNCH(HD_K_MGS, (j + 3.0) * P, launch_lsa_dots(c, a, G, c->st));
        HD_LAUNCH(HD_K_MGS, (j >= 1 ? j + 5.0 : 3.0) * P, k_lsa_update<<<G, kLsaBD, 0, c->st>>>(a));
      }
      if (j >= 1) {  // x_{j-1} is ready: monitor it (the reference's iteration j-1)
        monitor(xout);
        read_scalars(c);
        const double rr = c->hres[0];
        res.iterations = j;
        res.residuals.push_back(rr);
        if (rr <= opt.tolerance) {
          res.converged = true;
          stop = true;
          rollback();
          break;
        }
        if (hnew_prev < 1e-300) {
          stop = true;
          rollback();
          break;
        }
      }
      HD_LAUNCH(HD_K_GIVENS, 0.0, k_lsa_givens<<<1, kLsaBD, c->lsa_givens_smem, c->st>>>(a, G));
      CK(cudaMemcpyAsync(c->hres + 1, c->dres + 1, sizeof(double), cudaMemcpyDeviceToHost, c->st));
      // hnew of this iteration is needed one iteration later (read with the next sync)
      if (j + 1 == maxit) {
        // budget exhausted: x_{maxit-1} by an iterate-only pass, then its monitor
        LsaArgs b = lsa_args(c, xout, j, 1, maxit);
        HD_LAUNCH(HD_K_ITERATE, (j + 3.0) * P, k_lsa_update<<<G, kLsaBD, 0, c->st>>>(b));
        monitor(xout);
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
    return res;
  }
  for (int j = 0; j < maxit; ++j) {
    double2* Vj = c->V + static_cast<size_t>(j) * N;
    compose_op(c, Vj, c->w);
    double2* Hj = c->H + static_cast<size_t>(j) * ldh;
    // modified Gram-Schmidt (src/linalg.cpp:42-47)
    HD_LAUNCH(HD_K_MGS, 2 * P, k_dot<<<nb, 256, 0, c->st>>>(c->V, c->w, N, red_of(c), Hj + 0));
    for (int i = 0; i < j; ++i)
      HD_LAUNCH(HD_K_MGS, 4 * P,
                k_axpy_dot<<<nb, 256, 0, c->st>>>(c->w, c->V + static_cast<size_t>(i) * N, Hj + i,
                                                  c->V + static_cast<size_t>(i + 1) * N, N, red_of(c), Hj + i + 1));
    HD_LAUNCH(HD_K_MGS, 3 * P,
              k_axpy_norm<<<nb, 256, 0, c->st>>>(c->w, Vj, Hj + j, N, red_of(c, c->dres + 1), Hj + j + 1));
    HD_LAUNCH(HD_K_GIVENS, 0.0, k_givens<<<1, 32, 0, c->st>>>(c->H, ldh, c->g, c->cs, c->sn, c->y, j));
    HD_LAUNCH(HD_K_ITERATE, (j + 3) * P,
              k_iterate<<<grid_for(N), 256, 0, c->st>>>(xout, c->x0, c->V, c->y, j + 1, N));
    res.iterations = j + 1;
    monitor(xout);
    read_scalars(c);
    const double rr = c->hres[0];
    const double hnew = c->hres[1];
    res.residuals.push_back(rr);
    if (rr <= opt.tolerance) {
      res.converged = true;
      break;
    }
    if (hnew < 1e-300) break;
    if (j + 1 < maxit) {
      HD_LAUNCH(HD_K_VEC, 2 * P,
                k_scale_inv<<<grid_for(N), 256, 0, c->st>>>(c->V + static_cast<size_t>(j + 1) * N, c->w, c->dres + 1,
                                                            N));
    }
  }
  return res;
}


}  // namespace hd
