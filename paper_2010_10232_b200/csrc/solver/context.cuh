// Device context: error handling, exact-solver types, hd_ctx, setup of the exact solvers (FD, folded FD, partial FD, banded LU).
// (part of solver.cu, a single translation unit: included in order)
#pragma once

namespace hd {

static thread_local std::string g_last_error;

struct Error : std::runtime_error {
  hd_status code;
  Error(hd_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(x)                                                                                     \
  do {                                                                                            \
    cudaError_t e_ = (x);                                                                         \
    if (e_ != cudaSuccess)                                                                        \
      throw Error(HD_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_) + " @" + __FILE__ + \
                                   ":" + std::to_string(__LINE__));                               \
  } while (0)
#define CKB(x)                                                                                    \
  do {                                                                                            \
    cublasStatus_t e_ = (x);                                                                      \
    if (e_ != CUBLAS_STATUS_SUCCESS) throw Error(HD_ERR_CUDA, std::string(#x) + " failed: " + std::to_string(e_)); \
  } while (0)
#define CKS(x)                                                                                    \
  do {                                                                                            \
    cusolverStatus_t e_ = (x);                                                                    \
    if (e_ != CUSOLVER_STATUS_SUCCESS) throw Error(HD_ERR_CUDA, std::string(#x) + " failed: " + std::to_string(e_)); \
  } while (0)

// Device allocations.  HD_POISON=1 (read once per process) is this build's
// stand-in for compute-sanitizer initcheck / memcheck, which the GPU pool does
// not allow: every allocation is filled with 0xFF bytes (a NaN in every double
// lane), so a result that depends on memory never written turns NaN (and the
// solve stops with HD_ERR_NONFINITE); each allocation also gets kGuard
// poisoned bytes on both sides, verified by hd_debug_check_guards(), so an
// out-of-bounds store shows up as a changed guard and an out-of-bounds load
// of a guard as a NaN.
constexpr size_t kGuard = 512;
struct PoisonReg {
  std::mutex mu;
  std::map<void*, std::pair<void*, size_t>> live;  // user pointer -> (base, user bytes)
};
static PoisonReg& poison_reg() {
  static PoisonReg r;
  return r;
}
static bool poison_on() {
  static const bool on = std::getenv("HD_POISON") && std::atoi(std::getenv("HD_POISON")) == 1;
  return on;
}

template <class T>
static T* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  const size_t bytes = n * sizeof(T);
  if (!poison_on()) {
    CK(cudaMalloc(&p, bytes));
    return static_cast<T*>(p);
  }
  CK(cudaMalloc(&p, bytes + 2 * kGuard));
  CK(cudaMemset(p, 0xFF, bytes + 2 * kGuard));
  void* user = static_cast<char*>(p) + kGuard;
  PoisonReg& r = poison_reg();
  std::lock_guard<std::mutex> lk(r.mu);
  r.live[user] = {p, bytes};
  return static_cast<T*>(user);
}

static void dfree(const void* q) {
  void* p = const_cast<void*>(q);
  if (!p) return;
  if (poison_on()) {
    PoisonReg& r = poison_reg();
    std::lock_guard<std::mutex> lk(r.mu);
    auto it = r.live.find(p);
    if (it != r.live.end()) {
      p = it->second.first;
      r.live.erase(it);
    }
  }
  cudaFree(p);
}

// number of poisoned allocations whose guard bytes changed (HD_POISON=1; else 0)
static long check_guards() {
  if (!poison_on()) return 0;
  CK(cudaDeviceSynchronize());
  PoisonReg& r = poison_reg();
  std::lock_guard<std::mutex> lk(r.mu);
  std::vector<unsigned char> g(kGuard);
  long bad = 0;
  for (const auto& [user, rec] : r.live) {
    const char* base = static_cast<const char*>(rec.first);
    for (const char* at : {base, base + kGuard + rec.second}) {
      CK(cudaMemcpy(g.data(), at, kGuard, cudaMemcpyDeviceToHost));
      for (unsigned char b : g)
        if (b != 0xFF) {
          ++bad;
          std::fprintf(stderr, "[hd poison] guard changed around allocation %p (%zu bytes)\n", user, rec.second);
          break;
        }
    }
  }
  return bad;
}

// NVTX range of a host-side phase (setup phases, the prelude, the GMRES loop and, in the
// host-driven loop, the operator's parts and the Arnoldi passes): visible in nsys / ncu timelines.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Opt-in to `bytes` of dynamic shared memory for kernel `f` on the CURRENT
// device.  cudaFuncSetAttribute applies per device, so the cache is keyed by
// (device, function) and guarded: contexts on other GPUs or other host
// threads each get their own opt-in.
static void smem_optin(const void* f, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> done;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{dev, f}];
  if (bytes <= have) return;
  CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  have = bytes;
}

struct DevBand {
  double* S = nullptr;
  double* M = nullptr;
  int n = 0, b = 0;
  // layered field: the level as a G-term Kronecker sum (layered.cuh), with the
  // unshifted (A) and shifted coefficients; band tables owned by `gen_mem`
  GenLevel* genA = nullptr;
  GenLevel* genM = nullptr;
  double* gen_mem = nullptr;
};

// Exact solver of one Kronecker-sum (2D) or banded (1D) operator.
struct ExactSolver {
  int dim = 0, n = 0;
  // 2D fast diagonalisation
  double* V = nullptr;       // n x n column-major eigenvectors, V^T M V = I
  double2* Dinv = nullptr;   // n x n, 1 / (lam_y + lam_x - c)
  double* T1 = nullptr;      // planar work, 2 n^2
  double* T2 = nullptr;
  // 1D banded LU
  int kl = 0, ku = 0;
  double2* L = nullptr;
  double2* U = nullptr;
  int* piv = nullptr;
  double2* work = nullptr;
  double2* Uinv = nullptr;   // 1 / U(k, k)
  // segmented sweeps (segsolve.cuh); seg.P == 0: single-lane staged kernel
  SegArgs seg{};
  bool seg_seqscan = false;  // P-step single-warp boundary scans instead of k_seg_scan2 (HD_SEG_SEQSCAN at setup)
  // reflection-folded fast diagonalisation (centro-symmetric E, even n):
  // Vt = [Vs_top | Va_top] (2 x n2 x n2), Dinvf in [y parity][x parity][ky][kx]
  bool folded = false;
  int n2 = 0;
  double* Vt = nullptr;
  double2* Dinvf = nullptr;
  double *F = nullptr, *Hh = nullptr, *R = nullptr;  // folded blocks (8 n2^2 each)
  // pointer arrays of the two 8-entry batched x transforms (device): A, B, C of
  // the forward (Vt_xb^T Q -> Hh blocks) and of the inverse (Vt_xb S -> F blocks)
  const double** xf_ptr = nullptr;
  const double** xi_ptr = nullptr;
  // partial diagonalisation (pfd.cuh): x modes by V, banded LU along y per mode
  bool pfd = false;
  int pfd_kl = 0;
  int np = 0;                 // modes padded to kPG (leading dimension of T1)
  double* pfdF = nullptr;     // forward tables
  double* pfdB = nullptr;     // backward tables
  // dense inverse (layered field: E and the coarsest level are not Kronecker sums)
  bool dense = false;
  size_t NN = 0;
  double2* Ainv = nullptr;   // NN x NN column-major
  double2 *dx = nullptr, *dy = nullptr;
  // block tridiagonal (btri.cuh): real non-Kronecker operators too large for a dense inverse
  bool btri = false;
  bool bt_cplx = false;  // complex operator (C_ex on a non-separable field)
  BtriArgs bt{};
  int bt_kr = 0;
};

}  // namespace hd

using namespace hd;

struct hd_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  cublasHandle_t cb = nullptr;
  int dim = 1, p = 1, n = 0;
  size_t N = 0;
  double k = 0.0;
  hd_precond spec{};
  double2 corner = cmk(0.0, 0.0);
  // operators
  DevBand fine;                 // reduced S1, M1 (b = p)
  double2 cA = cmk(0.0, 0.0);   // A = ... - k^2 M(x)M
  double2 cM = cmk(0.0, 0.0);   // shifted: - k^2 (1 - i beta2) M(x)M
  std::vector<DevBand> lev;     // multigrid levels (lev[0] = fine)
  ExactSolver coarsest;
  ExactSolver shift_exact;      // C_ex: exact inverse of the shifted operator (cycles == 0)
  double* sx_plan = nullptr;    // planar scratch for the 2D exact shifted solve
  std::vector<double2*> mg_b, mg_x, mg_y, mg_r;
  // prolongation inside the first post-smoothing sweep (K4, OP_JACOBIP; HD_K4FUSE=1 at create).  Off by
  // default: equal results, but the sweep's extra registers (170 at B = 3: two CTAs per SM instead of
  // three) and per-row interpolation cost more than the saved launch and fine-vector round trip
  // (C5 89.9 vs 88.6 ms, C3 2.58 vs 2.49 ms)
  bool k4_fuse = false;
  bool j0_fuse = true;          // first Jacobi sweeps ride with their producers (HD_NOJ0FUSE=1 at create: off)
  int tail_l = -1;              // 1D: first level of the single-CTA tail V-cycle (tail1d.cuh), -1: none
  TailArgs tail{};
  size_t tail_smem_bytes = 0;
  bool small_ok = false;        // 1D, N <= kSmallMax: the whole solve in one single-CTA kernel (small1d.cuh)
  SmallArgs small{};
  double* small_res = nullptr;  // device residual history
  int* small_state = nullptr;
  // deflation
  int nc = 0;
  ExactSolver E;
  double* ep = nullptr;         // planar coarse buffers (2 nc^dim)
  double* ep2 = nullptr;
  // vectors
  double2 *f = nullptr, *rhsp = nullptr, *x0 = nullptr, *x = nullptr, *w = nullptr, *t1 = nullptr,
          *t2 = nullptr, *t3 = nullptr;
  double2* V = nullptr;
  int v_cap = 0;
  // GMRES scalars
  int maxit_cap = 0;
  double2 *H = nullptr, *g = nullptr, *cs = nullptr, *sn = nullptr, *y = nullptr;
  double2* scal = nullptr;      // [0] hnew, [1] beta, [2] scratch dot
  double* dres = nullptr;       // [0] rr, [1] hnew, [2] beta, [3] fnorm
  double* hres = nullptr;       // pinned mirror
  double2* partials = nullptr;
  unsigned* counter = nullptr;
  int red_blocks = 0;
  int* dj = nullptr;
  // Arnoldi engine: 1 = one-reduction ICWY-MGS streaming passes (default),
  // 0 = exact-order MGS, one kernel per MGS step (budgets above kLsaMaxJ, HD_ARNOLDI=0)
  int arn_mode = 1;
  // one-reduction engine state (arnoldi_lowsync.cuh)
  double* lsa_sig = nullptr;
  double2 *lsa_L = nullptr, *lsa_ch = nullptr, *lsa_cx = nullptr, *lsa_partials = nullptr;
  unsigned* lsa_counter = nullptr;
  int lsa_G = 0, lsa_maxit = -1;
  // tensor-copy stencil (stencil_tma.cuh) for whole-grid 2D level operators of at least
  // tma_min_n rows: HD_STENCIL_TMA=0 at create keeps the cp.async stencil everywhere
  bool stencil_tma = true;
  bool restrict_stream = true;  // streaming linear restriction on levels of >= tma_min_n rows (HD_RESTRICT_STREAM=0: tiled)
  int tma_min_n = 512;
  std::map<std::pair<const double*, const double*>, double2*> tma_ct;  // (S, M) tables -> CT of the level
  struct TmaKey {
    const void* base; int n, nvec, cols;
    bool operator<(const TmaKey& o) const {
      return std::tie(base, n, nvec, cols) < std::tie(o.base, o.n, o.nvec, o.cols);
    }
  };
  std::map<TmaKey, CUtensorMap> tma_maps;
  bool lsa_rev = true;          // HD_LSA_REV=0 at create: pass 2 walks the vectors front to back (A/B of the L2 reuse)
  bool lsa_mma = false;         // HD_LSA_MMA=1 at create: pass 1 as an FP64 tensor-core GEMM (k_lsa_dots_mma)
  bool lsa_tma = false;         // HD_LSA_TMA=1 at create: pass 1 on the bulk-copy ring (k_lsa_dots_tma)
  size_t lsa_givens_smem = 0;
  // graph-resident GMRES loop (WHILE conditional node), rebuilt when (maxit, tol) change
  cudaGraph_t loop_graph = nullptr;
  cudaGraphExec_t loop_exec = nullptr;
  bool pre_graph = true;               // HD_PRE_GRAPH=0: eager prelude launches
  cudaGraphExec_t pre_exec = nullptr;  // GMRES prelude (rhs', start, monitor(x0), op(x0), beta)
  long pre_dcnt[4] = {0, 0, 0, 0}, pre_dsnap[4] = {0, 0, 0, 0};
  int pre_dl = 0, pre_db = 0;
  int loop_maxit = -1;
  double loop_tol = -1.0;
  // bumped whenever a buffer a captured graph points at is reallocated
  // (ensure_gmres, the slab basis); graphs record the epoch they captured
  unsigned buf_epoch = 0;
  unsigned loop_epoch = ~0u, pre_epoch = ~0u;
  LoopState* loop_state = nullptr;
  LoopState* loop_host = nullptr;   // pinned
  double* res_hist = nullptr;       // device, maxit
  double* res_host = nullptr;       // pinned
  void* cublas_ws = nullptr;
  bool graph_enabled = true;        // HD_GRAPH=0: host-driven loop
  bool mon_side = false;            // HD_MON_SIDE=1: monitor of x_{j-2} on the graph body's side branch (measured neutral, opt-in)
  double2* mon_partials = nullptr;  // side-branch monitor's own grid-reduction scratch
  unsigned* mon_counter = nullptr;
  int graph_body_kernels = 0;       // own kernels per body execution
  int n_sms = 148;
  // counters
  long matvecs = 0, coarse_solves = 0, shift_solves = 0, vcycles = 0;
  int launches = 0;             // own kernels launched in the last solve
  int lib_calls = 0;            // cuBLAS calls in the last solve
  double t_setup = 0.0;
  // per-launch event timing (hd_profile)
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_ev;
  size_t prof_used = 0;
  struct ProfRec { int kind; size_t ev; double bytes; };
  std::vector<ProfRec> prof_recs;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaStream_t own_st = nullptr;  // the context's own stream while an external one is set
  cudaStream_t st2 = nullptr;     // side branch of the graph body (Givens of the previous iteration)
  void* slabs = nullptr;          // row-slab state (hd_create_slabs), or null
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

namespace hd {

static DevBand upload_band(const Band& B) {
  DevBand d;
  d.n = B.n;
  d.b = B.b;
  d.S = dalloc<double>(B.a.size());
  CK(cudaMemcpy(d.S, B.a.data(), B.a.size() * sizeof(double), cudaMemcpyHostToDevice));
  return d;
}

static DevBand upload_pair(const Band& S, const Band& M) {
  const int b = std::max(S.b, M.b);
  Band s2(S.n, b), m2(M.n, b);
  for (int i = 0; i < S.n; ++i)
    for (int d = -b; d <= b; ++d) {
      const int j = i + d;
      if (j < 0 || j >= S.n) continue;
      s2.ref(i, j) = S.at(i, j);
      m2.ref(i, j) = M.at(i, j);
    }
  DevBand d;
  d.n = S.n;
  d.b = b;
  d.S = dalloc<double>(s2.a.size());
  d.M = dalloc<double>(m2.a.size());
  CK(cudaMemcpy(d.S, s2.a.data(), s2.a.size() * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d.M, m2.a.data(), m2.a.size() * sizeof(double), cudaMemcpyHostToDevice));
  return d;
}

static Band band_from_host(const double* a, int n, int b) {
  Band B(n, b);
  std::memcpy(B.a.data(), a, B.a.size() * sizeof(double));
  return B;
}

static LevelDev level_dev(const DevBand& d, double2 c, double2 corner, const GenLevel* gen = nullptr) {
  LevelDev L;
  L.gen = gen;
  L.S = d.S;
  L.M = d.M;
  L.n = d.n;
  L.b = d.b;
  L.c = c;
  L.corner = corner;
  return L;
}

static std::vector<double> dense_of(const Band& B) {
  std::vector<double> D(static_cast<size_t>(B.n) * B.n, 0.0);
  for (int i = 0; i < B.n; ++i)
    for (int j = std::max(0, i - B.b); j <= std::min(B.n - 1, i + B.b); ++j) D[i + static_cast<size_t>(j) * B.n] = B.at(i, j);
  return D;
}

// Dense generalized symmetric-definite eigenproblem A v = lam B v (cuSOLVER
// sygvd), eigenvectors returned column-major on the device, V^T B V = I.
// HD_SETUP_TRACE=1 prints the B-orthogonality and the eigen-residuals (at C5's
// n = 800: 3e-15 and 1.7e-13 ||A||, LAPACK's dsygvd on the same pencil: 3e-15
// and 1.1e-13).
static void sygvd_device(cudaStream_t st, const std::vector<double>& A, const std::vector<double>& Bm, int n,
                         double* dV, std::vector<double>& lam) {
  double *dB = dalloc<double>(Bm.size()), *dW = dalloc<double>(n);
  int* dinfo = dalloc<int>(1);
  CK(cudaMemcpy(dV, A.data(), A.size() * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Bm.data(), Bm.size() * sizeof(double), cudaMemcpyHostToDevice));
  cusolverDnHandle_t h;
  CKS(cusolverDnCreate(&h));
  CKS(cusolverDnSetStream(h, st));
  int lwork = 0;
  CKS(cusolverDnDsygvd_bufferSize(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dV, n,
                                  dB, n, dW, &lwork));
  double* dwork = dalloc<double>(std::max(lwork, 1));
  CKS(cusolverDnDsygvd(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dV, n, dB, n, dW,
                       dwork, lwork, dinfo));
  int info = 0;
  CK(cudaMemcpyAsync(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cusolverDnDestroy(h);
  if (info != 0) throw Error(HD_ERR_FACTOR, "coarse operator factorization failed (sygvd info " + std::to_string(info) + ")");
  lam.resize(n);
  CK(cudaMemcpy(lam.data(), dW, n * sizeof(double), cudaMemcpyDeviceToHost));
  dfree(dB);
  dfree(dW);
  dfree(dinfo);
  dfree(dwork);
  if (std::getenv("HD_SETUP_TRACE") && std::atoi(std::getenv("HD_SETUP_TRACE")) == 1) {
    // max |(V^T B V - I)_ij| (sampled columns) and max_j ||A v_j - lam_j B v_j|| / ||A||_inf
    std::vector<double> V(static_cast<size_t>(n) * n);
    CK(cudaMemcpy(V.data(), dV, V.size() * sizeof(double), cudaMemcpyDeviceToHost));
    std::vector<double> BV(V.size(), 0.0), AV(V.size(), 0.0);
    for (int c2 = 0; c2 < n; ++c2)
      for (int r = 0; r < n; ++r) {
        double sb = 0.0, sa = 0.0;
        for (int q = std::max(0, r - 8); q < std::min(n, r + 9); ++q) {
          sb += Bm[r + static_cast<size_t>(q) * n] * V[q + static_cast<size_t>(c2) * n];
          sa += A[r + static_cast<size_t>(q) * n] * V[q + static_cast<size_t>(c2) * n];
        }
        BV[r + static_cast<size_t>(c2) * n] = sb;
        AV[r + static_cast<size_t>(c2) * n] = sa;
      }
    double orth = 0.0, res = 0.0, an = 0.0;
    for (int r = 0; r < n; ++r) {
      double rs = 0.0;
      for (int q = 0; q < n; ++q) rs += std::abs(A[r + static_cast<size_t>(q) * n]);
      an = std::max(an, rs);
    }
    for (int a = 0; a < n; a += std::max(1, n / 64))
      for (int b = 0; b < n; ++b) {
        double d = 0.0;
        for (int r = 0; r < n; ++r) d += V[r + static_cast<size_t>(a) * n] * BV[r + static_cast<size_t>(b) * n];
        orth = std::max(orth, std::abs(d - (a == b ? 1.0 : 0.0)));
      }
    for (int c2 = 0; c2 < n; ++c2) {
      double s2 = 0.0;
      for (int r = 0; r < n; ++r) {
        const double e = AV[r + static_cast<size_t>(c2) * n] - lam[c2] * BV[r + static_cast<size_t>(c2) * n];
        s2 += e * e;
      }
      res = std::max(res, std::sqrt(s2) / an);
    }
    std::fprintf(stderr, "[hd setup] sygvd n=%d: max|V^T B V - I| %.2e, max residual %.2e\n", n, orth, res);
  }
}

// True when the banded matrix is centro-symmetric, X(i,j) = X(n-1-i, n-1-j),
// to rounding (the reflected B-spline basis and an odd fine size make the
// Bezier-coarsened E so).
static bool centro_symmetric(const Band& X) {
  double mx = 0.0, dev = 0.0;
  for (int i = 0; i < X.n; ++i)
    for (int d = -X.b; d <= X.b; ++d) {
      const int j = i + d;
      if (j < 0 || j >= X.n) continue;
      mx = std::max(mx, std::abs(X.at(i, j)));
      dev = std::max(dev, std::abs(X.at(i, j) - X.at(X.n - 1 - i, X.n - 1 - j)));
    }
  // symmetric to 1e-12 relative: the symmetrised E' is within the backward error
  // the fast diagonalisation carries anyway (eigen-residuals ~1e-13 ||E_S|| from
  // cuSOLVER or LAPACK), and C5's history stays inside the envelope of exact
  // implementations; HD_CENTRO_TOL=0 / HD_ESOLVE=fd: unfolded
  const double tol = std::getenv("HD_CENTRO_TOL") ? std::atof(std::getenv("HD_CENTRO_TOL")) : 1e-12;
  return dev <= tol * mx;
}

// Reflection-folded fast diagonalisation: for even n and centro-symmetric
// S, M the eigenvectors are symmetric [a; Ja]/sqrt2 or antisymmetric
// [a; -Ja]/sqrt2 with a from the half-size problems (X_tt +- X_tb J).  Every
// transform then costs two half-size GEMMs instead of one full one.
static ExactSolver make_fd_folded(cudaStream_t st, const Band& S, const Band& M, double2 c) {
  ExactSolver X;
  X.dim = 2;
  X.folded = true;
  X.n = S.n;
  const int n = S.n, n2 = n / 2;
  X.n2 = n2;
  X.Vt = dalloc<double>(2 * static_cast<size_t>(n2) * n2);
  std::vector<double> lam[2];
  for (int par = 0; par < 2; ++par) {
    const double sg = par == 0 ? 1.0 : -1.0;
    std::vector<double> As(static_cast<size_t>(n2) * n2), Bs(As.size());
    for (int i = 0; i < n2; ++i)
      for (int j = 0; j < n2; ++j) {
        // (X_tt +- X_tb J)(i, j) = X(i, j) +- X(i, n-1-j), column-major
        As[i + static_cast<size_t>(j) * n2] = S.at(i, j) + sg * S.at(i, n - 1 - j);
        Bs[i + static_cast<size_t>(j) * n2] = M.at(i, j) + sg * M.at(i, n - 1 - j);
      }
    double* dV = X.Vt + static_cast<size_t>(par) * n2 * n2;
    sygvd_device(st, As, Bs, n2, dV, lam[par]);
  }
  // scale the half-vectors by 1/sqrt2 (full vectors [a; +-Ja]/sqrt2 are M-orthonormal)
  {
    std::vector<double> hv(2 * static_cast<size_t>(n2) * n2);
    CK(cudaMemcpy(hv.data(), X.Vt, hv.size() * sizeof(double), cudaMemcpyDeviceToHost));
    for (double& v : hv) v *= std::sqrt(0.5);
    CK(cudaMemcpy(X.Vt, hv.data(), hv.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  std::vector<double2> D(4 * static_cast<size_t>(n2) * n2);
  for (int yb = 0; yb < 2; ++yb)
    for (int xb = 0; xb < 2; ++xb)
      for (int ky = 0; ky < n2; ++ky)
        for (int kx = 0; kx < n2; ++kx) {
          const std::complex<double> d(lam[yb][ky] + lam[xb][kx] - c.x, -c.y);
          if (d == std::complex<double>(0.0, 0.0))
            throw Error(HD_ERR_FACTOR, "coarse operator factorization failed (singular)");
          const std::complex<double> r = 1.0 / d;
          D[((static_cast<size_t>(yb) * 2 + xb) * n2 + ky) * n2 + kx] = cmk(r.real(), r.imag());
        }
  X.Dinvf = dalloc<double2>(D.size());
  CK(cudaMemcpy(X.Dinvf, D.data(), D.size() * sizeof(double2), cudaMemcpyHostToDevice));
  const size_t half = 2 * static_cast<size_t>(n2) * 2 * n;  // 2 parities x n2 x 2n
  X.F = dalloc<double>(half);
  X.Hh = dalloc<double>(8 * static_cast<size_t>(n2) * n2);
  X.R = dalloc<double>(8 * static_cast<size_t>(n2) * n2);
  // x transforms as 8-entry pointer-batched GEMMs over (x parity, y parity, plane):
  // forward Vt_xb^T Q[xb][yb][p] (Q blocks n2 x n2 in F) into Hh[yb] rows (2 xb + p) n2,
  // inverse Vt_xb Hh[yb] rows (2 xb + p) n2 into F blocks
  {
    const size_t nn = static_cast<size_t>(n2) * n2;
    std::vector<const double*> hp(48);
    for (int xb = 0; xb < 2; ++xb)
      for (int yb = 0; yb < 2; ++yb)
        for (int p = 0; p < 2; ++p) {
          const int e = (xb * 2 + yb) * 2 + p;
          const double* vt = X.Vt + xb * nn;
          const double* fb = X.F + e * nn;
          const double* hb = X.Hh + yb * 4 * nn + (2 * xb + p) * n2;
          hp[e] = vt; hp[8 + e] = fb; hp[16 + e] = hb;        // forward: A, B, C
          hp[24 + e] = vt; hp[32 + e] = hb; hp[40 + e] = fb;  // inverse: A, B, C
        }
    const double** d = dalloc<const double*>(48);
    CK(cudaMemcpy(d, hp.data(), 48 * sizeof(const double*), cudaMemcpyHostToDevice));
    X.xf_ptr = d;
    X.xi_ptr = d + 24;
  }
  return X;
}

// Fast diagonalisation of W = M(x)S + S(x)M - c M(x)M: S V = M V diag(lam),
// V^T M V = I (cuSOLVER sygvd at setup), Dinv = 1/(lam_i + lam_j - c).
static ExactSolver make_fd(cudaStream_t st, const Band& S, const Band& M, double2 c) {
  ExactSolver X;
  X.dim = 2;
  X.n = S.n;
  const int n = S.n;
  double* dA = dalloc<double>(static_cast<size_t>(n) * n);
  std::vector<double> lam;
  sygvd_device(st, dense_of(S), dense_of(M), n, dA, lam);
  std::vector<double2> Dinv(static_cast<size_t>(n) * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const std::complex<double> d(lam[i] + lam[j] - c.x, -c.y);
      if (d == std::complex<double>(0.0, 0.0)) throw Error(HD_ERR_FACTOR, "coarse operator factorization failed (singular)");
      const std::complex<double> r = 1.0 / d;
      Dinv[static_cast<size_t>(i) * n + j] = cmk(r.real(), r.imag());
    }
  X.V = dA;
  X.Dinv = dalloc<double2>(Dinv.size());
  CK(cudaMemcpy(X.Dinv, Dinv.data(), Dinv.size() * sizeof(double2), cudaMemcpyHostToDevice));
  X.T1 = dalloc<double>(2 * static_cast<size_t>(n) * n);
  X.T2 = dalloc<double>(2 * static_cast<size_t>(n) * n);
  return X;
}

// Partial diagonalisation of a real Kronecker sum W = M(x)S + S(x)M - c M(x)M
// (pfd.cuh): V from the x eigenproblem S V = M V diag(lam) (sygvd, as make_fd),
// then for every x mode m the real banded LU with partial pivoting of
// S - (c - lam_m) M along y, packed as the kernel's per-group row tables.
static ExactSolver make_pfd(cudaStream_t st, const Band& S, const Band& M, double c) {
  ExactSolver X;
  X.dim = 2;
  X.pfd = true;
  const int n = S.n, kl = std::max(S.b, M.b), ku = 2 * kl;
  if (kl < 1 || kl > 4) throw Error(HD_ERR_INVALID, "partial diagonalisation: band half-width outside 1..4");
  X.n = n;
  X.pfd_kl = kl;
  const int np = (n + kPG - 1) / kPG * kPG, ng = np / kPG;
  X.np = np;
  X.V = dalloc<double>(static_cast<size_t>(n) * n);
  std::vector<double> lam;
  sygvd_device(st, dense_of(S), dense_of(M), n, X.V, lam);
  const int FW = (kl + 1) * kPG, BW = (ku + 1) * kPG;
  std::vector<double> F(static_cast<size_t>(ng) * n * FW, 0.0), B(static_cast<size_t>(ng) * n * BW, 0.0);
  for (int m = 0; m < np; ++m) {
    const int g = m / kPG, mm = m % kPG;
    double* fg = F.data() + static_cast<size_t>(g) * n * FW;
    double* bg = B.data() + static_cast<size_t>(g) * n * BW;
    if (m >= n) {  // padding modes: identity rows
      for (int k = 0; k < n; ++k) bg[static_cast<size_t>(k) * BW + mm] = 1.0;
      continue;
    }
    const BandLUr f = band_lu_real(S, M, c - lam[m]);
    if (f.kl != kl || f.ku != ku) throw Error(HD_ERR_INVALID, "unexpected band LU shape");
    for (int k = 0; k < n; ++k) {
      double* fr = fg + static_cast<size_t>(k) * FW;
      for (int q = 0; q < kl; ++q) fr[q * kPG + mm] = f.L[static_cast<size_t>(k) * kl + q];
      fr[kl * kPG + mm] = static_cast<double>(f.piv[k] - k);
      double* br = bg + static_cast<size_t>(k) * BW;
      const double ukk = f.U[static_cast<size_t>(k) * (ku + 1)];
      if (ukk == 0.0) throw Error(HD_ERR_FACTOR, "deflation matrix E is singular");
      br[mm] = 1.0 / ukk;
      for (int d = 1; d <= ku; ++d) br[d * kPG + mm] = f.U[static_cast<size_t>(k) * (ku + 1) + d];
    }
  }
  X.pfdF = dalloc<double>(F.size());
  X.pfdB = dalloc<double>(B.size());
  CK(cudaMemcpy(X.pfdF, F.data(), F.size() * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(X.pfdB, B.data(), B.size() * sizeof(double), cudaMemcpyHostToDevice));
  X.T1 = dalloc<double>(2 * static_cast<size_t>(n) * np);
  CK(cudaMemset(X.T1, 0, 2 * static_cast<size_t>(n) * np * sizeof(double)));
  return X;
}

// Influence rows and window transfers of the segmented sweeps (segsolve.cuh),
// by running each segment's recurrences on unit boundary values; all per-row
// tables in the [row-in-segment][field][segment] layout, rows past n = identity.
static void make_segments(ExactSolver& X, const BandLU& f) {
  const int n = f.n, kl = f.kl, ku = f.ku, W = kl + 1, Ls = kSegL;
  const int P = (n + Ls - 1) / Ls;
  if (P < 4 || ku != 2 * kl) return;
  const int NP = P * Ls;
  // padded row access
  auto Lm = [&](int k, int q) { return k < n ? f.L[static_cast<size_t>(k) * kl + q] : cplx(0.0, 0.0); };
  auto Uu = [&](int k, int d) { return k < n ? f.U[static_cast<size_t>(k) * (ku + 1) + d] : (d == 0 ? cplx(1.0, 0.0) : cplx(0.0, 0.0)); };
  auto pv = [&](int k) { return k < n ? f.piv[k] - k : 0; };
  auto at = [&](int k, int fld, int nf) { return (static_cast<size_t>(k % Ls) * nf + fld) * P + k / Ls; };
  std::vector<cplx> Lt(static_cast<size_t>(NP) * kl), hf(static_cast<size_t>(NP) * W), Ut(static_cast<size_t>(NP) * ku),
      Ui(NP), hb(static_cast<size_t>(NP) * ku), Ff(static_cast<size_t>(P) * W * W), Hb(static_cast<size_t>(P) * ku * ku);
  std::vector<int> pt(NP);
  for (int k = 0; k < NP; ++k) {
    for (int q = 0; q < kl; ++q) Lt[at(k, q, kl)] = Lm(k, q);
    pt[at(k, 0, 1)] = pv(k);
    for (int d = 1; d <= ku; ++d) Ut[at(k, d - 1, ku)] = Uu(k, d);
    Ui[at(k, 0, 1)] = 1.0 / Uu(k, 0);
  }
  for (int i = 0; i < P; ++i) {
    const int s = i * Ls, e = s + Ls;
    for (int q = 0; q < W; ++q) {  // forward from window e_q, no rhs
      std::vector<cplx> w(W, cplx(0.0, 0.0));
      w[q] = 1.0;
      for (int k = s; k < e; ++k) {
        const int p = pv(k);
        if (p != 0) std::swap(w[0], w[p]);
        const cplx yk = w[0];
        hf[at(k, q, W)] = yk;
        for (int r = 1; r <= kl; ++r) w[r] -= Lm(k, r - 1) * yk;
        for (int r = 0; r < kl; ++r) w[r] = w[r + 1];
        w[kl] = 0.0;
      }
      for (int r = 0; r < W; ++r) Ff[(static_cast<size_t>(i) * W + r) * W + q] = w[r];
    }
    for (int r = 0; r < ku; ++r) {  // backward from future x_{e+r} = 1, no rhs
      std::vector<cplx> xw(ku, cplx(0.0, 0.0));  // x_{k+1} .. x_{k+ku}
      xw[r] = 1.0;
      for (int k = e - 1; k >= s; --k) {
        cplx acc(0.0, 0.0);
        for (int d = ku; d >= 1; --d) acc -= Uu(k, d) * xw[d - 1];
        const cplx xk = acc / Uu(k, 0);
        for (int d = ku - 1; d >= 1; --d) xw[d] = xw[d - 1];
        xw[0] = xk;
        hb[at(k, r, ku)] = xk;
        if (k - s < ku) Hb[(static_cast<size_t>(i) * ku + (k - s)) * ku + r] = xk;
      }
    }
  }
  auto up = [](const auto& v) {
    using T = typename std::decay_t<decltype(v)>::value_type;
    T* d = dalloc<T>(v.size());
    CK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
  };
  X.seg_seqscan = std::getenv("HD_SEG_SEQSCAN") != nullptr;
  SegArgs& a = X.seg;
  a.n = n;
  a.P = P;
  a.L = reinterpret_cast<const double2*>(up(Lt));
  a.pv = up(pt);
  a.hf = reinterpret_cast<const double2*>(up(hf));
  a.U = reinterpret_cast<const double2*>(up(Ut));
  a.Ui = reinterpret_cast<const double2*>(up(Ui));
  a.hb = reinterpret_cast<const double2*>(up(hb));
  a.Ff = reinterpret_cast<const double2*>(up(Ff));
  a.Hb = reinterpret_cast<const double2*>(up(Hb));
  a.y = dalloc<double2>(NP);
  a.x0 = dalloc<double2>(NP);
  a.D = dalloc<double2>(static_cast<size_t>(P) * W);
  a.Dl = dalloc<double2>(static_cast<size_t>(P) * W);
  a.X0 = dalloc<double2>(static_cast<size_t>(P) * ku);
  a.Xb = dalloc<double2>(static_cast<size_t>(P + 1) * ku);
  a.AgF = dalloc<double2>(static_cast<size_t>(kScanWarps) * W * W);
  a.AgB = dalloc<double2>(static_cast<size_t>(kScanWarps) * ku * ku);
}

// Setup pass of the two-level scans: the matrix parts of their group maps (k_seg_scan2 PRE = 1)
template <int KL>
static void seg_precompute_t(ExactSolver& X) {
  constexpr int W = KL + 1, KU = 2 * KL;
  if (seg_scan2_smem<KU>() > 227u * 1024u) return;  // that size uses the sequential scans
  SegArgs& a = X.seg;
  smem_optin(reinterpret_cast<const void*>(k_seg_scan2<W, 0, 1>), seg_scan2_smem<W>());
  smem_optin(reinterpret_cast<const void*>(k_seg_scan2<KU, 1, 1>), seg_scan2_smem<KU>());
  CK(cudaMemset(a.D, 0, static_cast<size_t>(a.P) * W * sizeof(double2)));
  CK(cudaMemset(a.X0, 0, static_cast<size_t>(a.P) * KU * sizeof(double2)));
  k_seg_scan2<W, 0, 1><<<1, kScanWarps * 32, seg_scan2_smem<W>()>>>(a.Ff, a.D, nullptr, a.P, a.AgF);
  k_seg_scan2<KU, 1, 1><<<1, kScanWarps * 32, seg_scan2_smem<KU>()>>>(a.Hb, a.X0, nullptr, a.P, a.AgB);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
}

static void seg_precompute(ExactSolver& X) {
  switch (X.kl) {
    case 1: seg_precompute_t<1>(X); break;
    case 2: seg_precompute_t<2>(X); break;
    case 3: seg_precompute_t<3>(X); break;
    case 4: seg_precompute_t<4>(X); break;
    case 5: seg_precompute_t<5>(X); break;
    default: seg_precompute_t<6>(X); break;
  }
}

static ExactSolver make_bandlu(const Band& S, const Band& M, double2 c, double2 corner) {
  BandLU f = band_lu(S, M, cplx(c.x, c.y), cplx(corner.x, corner.y));
  ExactSolver X;
  X.dim = 1;
  X.n = f.n;
  X.kl = f.kl;
  X.ku = f.ku;
  X.L = dalloc<double2>(f.L.size());
  X.U = dalloc<double2>(f.U.size());
  X.piv = dalloc<int>(f.piv.size());
  X.work = dalloc<double2>(f.n);
  std::vector<cplx> uinv(f.n);
  for (int k = 0; k < f.n; ++k) uinv[k] = 1.0 / f.U[static_cast<size_t>(k) * (f.ku + 1)];
  X.Uinv = dalloc<double2>(f.n);
  CK(cudaMemcpy(X.Uinv, uinv.data(), uinv.size() * sizeof(double2), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(X.L, f.L.data(), f.L.size() * sizeof(double2), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(X.U, f.U.data(), f.U.size() * sizeof(double2), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(X.piv, f.piv.data(), f.piv.size() * sizeof(int), cudaMemcpyHostToDevice));
  const char* e = std::getenv("HD_SEG");
  if (!(e && std::atoi(e) == 0) && f.kl >= 1 && f.kl <= 6) make_segments(X, f);
  if (X.seg.P && !X.seg_seqscan) seg_precompute(X);
  return X;
}

static void free_exact(ExactSolver& X) {
  dfree(X.V); dfree(X.Dinv); dfree(X.T1); dfree(X.T2);
  dfree(X.Vt); dfree(X.Dinvf); dfree(X.F); dfree(X.Hh); dfree(X.R);
    dfree(const_cast<double**>(X.xf_ptr));
  dfree(X.L); dfree(X.U); dfree(X.piv); dfree(X.work); dfree(X.Uinv);
  if (X.seg.P) {
    for (const void* p : {static_cast<const void*>(X.seg.L), static_cast<const void*>(X.seg.pv),
                          static_cast<const void*>(X.seg.hf), static_cast<const void*>(X.seg.U),
                          static_cast<const void*>(X.seg.Ui), static_cast<const void*>(X.seg.hb),
                          static_cast<const void*>(X.seg.Ff), static_cast<const void*>(X.seg.Hb)})
      dfree(const_cast<void*>(p));
    dfree(X.seg.y); dfree(X.seg.x0); dfree(X.seg.D);
    dfree(X.seg.Dl); dfree(X.seg.X0); dfree(X.seg.Xb); dfree(X.seg.AgF); dfree(X.seg.AgB);
  }
  dfree(X.Ainv); dfree(X.dx); dfree(X.dy);
  dfree(X.pfdF); dfree(X.pfdB);
  if (X.btri) {
    dfree(const_cast<void*>(X.bt.GT)); dfree(const_cast<void*>(X.bt.SinvT));
    dfree(const_cast<void*>(X.bt.HT)); dfree(const_cast<void*>(X.bt.G2)); dfree(X.bt.y); dfree(X.bt.bar); dfree(const_cast<void*>(X.bt.steps));
  }
  X = ExactSolver{};
}

template <int KL>
static void bandlu_launch_t(cudaStream_t st, const ExactSolver& X, const double2* b, const double* bp, double2* x,
                            double* xp) {
  constexpr size_t sm = bandlu_smem<KL>();
  smem_optin(reinterpret_cast<const void*>(k_bandlu_staged<KL>), sm);
  k_bandlu_staged<KL><<<1, 256, sm, st>>>(X.L, X.U, X.Uinv, X.piv, X.n, b, bp, X.work, x, xp);
}

template <int KL>
static void seg_launch_t(cudaStream_t st, const ExactSolver& X, const double2* b, const double* bp, double2* x,
                         double* xp) {
  const SegArgs& a = X.seg;
  const int blocks = (a.P + 31) / 32;
  smem_optin(reinterpret_cast<const void*>(k_seg_fwd<KL>), seg_fwd_smem<KL>());
  smem_optin(reinterpret_cast<const void*>(k_seg_bwd<KL>), seg_bwd_smem<KL>());
  constexpr int W = KL + 1, KU = 2 * KL;
  // the P-step single-warp scans: HD_SEG_SEQSCAN, or maps too large for the staged two-level scan (KL = 6)
  const bool seq = X.seg_seqscan || seg_scan2_smem<KU>() > 227u * 1024u;
  if (!seq) {
    smem_optin(reinterpret_cast<const void*>(k_seg_scan2<W, 0>), seg_scan2_smem<W>());
    smem_optin(reinterpret_cast<const void*>(k_seg_scan2<KU, 1>), seg_scan2_smem<KU>());
  }
  k_seg_fwd<KL><<<blocks, 32, seg_fwd_smem<KL>(), st>>>(a, b, bp);
  if (seq) k_seg_scan_fwd<KL><<<1, 32, 0, st>>>(a);
  else k_seg_scan2<W, 0><<<1, kScanWarps * 32, seg_scan2_smem<W>(), st>>>(a.Ff, a.D, a.Dl, a.P, a.AgF);
  k_seg_bwd<KL><<<blocks, 32, seg_bwd_smem<KL>(), st>>>(a);
  if (seq) k_seg_scan_bwd<KL><<<1, 32, 0, st>>>(a);
  else k_seg_scan2<KU, 1><<<1, kScanWarps * 32, seg_scan2_smem<KU>(), st>>>(a.Hb, a.X0, a.Xb, a.P, a.AgB);
  k_seg_out<KL><<<std::min((a.n + 255) / 256, 148 * 4), 256, 0, st>>>(a, x, xp);
}

// 1D exact solve (kl = 1..6), in/out interleaved or planar: segmented sweeps,
// or the single-lane staged kernel for short systems
static void bandlu_launch(cudaStream_t st, const ExactSolver& X, const double2* b, const double* bp, double2* x,
                          double* xp) {
  if (X.ku != 2 * X.kl) throw Error(HD_ERR_INVALID, "banded LU layout mismatch");
  if (X.seg.P) {
    switch (X.kl) {
      case 1: seg_launch_t<1>(st, X, b, bp, x, xp); break;
      case 2: seg_launch_t<2>(st, X, b, bp, x, xp); break;
      case 3: seg_launch_t<3>(st, X, b, bp, x, xp); break;
      case 4: seg_launch_t<4>(st, X, b, bp, x, xp); break;
      case 5: seg_launch_t<5>(st, X, b, bp, x, xp); break;
      default: seg_launch_t<6>(st, X, b, bp, x, xp); break;
    }
    return;
  }
  switch (X.kl) {
    case 1: bandlu_launch_t<1>(st, X, b, bp, x, xp); break;
    case 2: bandlu_launch_t<2>(st, X, b, bp, x, xp); break;
    case 3: bandlu_launch_t<3>(st, X, b, bp, x, xp); break;
    case 4: bandlu_launch_t<4>(st, X, b, bp, x, xp); break;
    case 5: bandlu_launch_t<5>(st, X, b, bp, x, xp); break;
    case 6: bandlu_launch_t<6>(st, X, b, bp, x, xp); break;
    default: throw Error(HD_ERR_INVALID, "banded LU bandwidth " + std::to_string(X.kl) + " unsupported");
  }
}


}  // namespace hd
