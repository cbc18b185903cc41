// Host driver of the device solve behind the C-ABI of include/helmdef_b200.h.
//
// hd_create  == compose()  (src/precond.cpp:196-265): Galerkin multigrid
//               hierarchy of the shifted operator (as 1D factors, see
//               host/banded.hpp), inverse-diagonal Jacobi, coarsest exact
//               solve, Bezier deflation E = Z^T A Z and its exact solve.
// hd_solve   == gmres(setup.op, setup.rhs, setup.start, setup.monitor, opt)
//               (src/linalg.cpp:10-92) with every vector resident on the
//               device; one 2-scalar device->host read per iteration decides
//               convergence.
// SPDX-License-Identifier: Apache-2.0
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/helmdef_b200.h"
#include "host/assembly.hpp"
#include "host/banded.hpp"
#include "kernels.cuh"
#include "stencil.cuh"
#include "transfer.cuh"
#include "arnoldi.cuh"
#include "arnoldi_lowsync.cuh"
#include "layered.cuh"
#include "btri.cuh"
#include "segsolve.cuh"
#include "ysolve.cuh"

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

template <class T>
static T* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  CK(cudaMalloc(&p, n * sizeof(T)));
  return static_cast<T*>(p);
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
  // partial fast diagonalisation (ysolve.cuh): x modes by V, segmented banded LU sweeps along y
  bool ypart = false;
  int ykl = 0;
  YArgs ya{};
  // reflection-folded fast diagonalisation (centro-symmetric E, even n):
  // Vt = [Vs_top | Va_top] (2 x n2 x n2), Dinvf in [y parity][x parity][ky][kx]
  bool folded = false;
  int n2 = 0;
  double* Vt = nullptr;
  double2* Dinvf = nullptr;
  double *F = nullptr, *G = nullptr, *Hh = nullptr, *R = nullptr;
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
  // persistent Arnoldi tail (arnoldi.cuh)
  bool use_arnoldi = false;
  int arn_G = 0, arn_K = 0;
  size_t arn_chunk = 0, arn_smem = 0;
  int* dj = nullptr;
  double2* arn_partials = nullptr;
  int arn_maxit = -1;
  unsigned* arn_bar = nullptr;
  unsigned long long* arn_trace = nullptr;  // HD_TRACE: phase timestamps of the last launch
  double arn_phase_ns[4] = {0, 0, 0, 0};
  // Arnoldi engine: 2 = one-reduction ICWY-MGS streaming passes (default),
  // 1 = persistent exact-order MGS chain, 0 = one kernel per MGS step.
  int arn_mode = 2;
  // one-reduction engine state (arnoldi_lowsync.cuh)
  double* lsa_sig = nullptr;
  double2 *lsa_L = nullptr, *lsa_ch = nullptr, *lsa_cx = nullptr, *lsa_partials = nullptr;
  unsigned* lsa_counter = nullptr;
  int lsa_G = 0, lsa_maxit = -1;
  size_t lsa_givens_smem = 0;
  // graph-resident GMRES loop (WHILE conditional node), rebuilt when (maxit, tol) change
  cudaGraph_t loop_graph = nullptr;
  cudaGraphExec_t loop_exec = nullptr;
  int loop_maxit = -1;
  double loop_tol = -1.0;
  LoopState* loop_state = nullptr;
  LoopState* loop_host = nullptr;   // pinned
  double* res_hist = nullptr;       // device, maxit
  double* res_host = nullptr;       // pinned
  void* cublas_ws = nullptr;
  bool graph_enabled = true;        // HD_GRAPH=0: host-driven loop
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
  cudaFree(dB);
  cudaFree(dW);
  cudaFree(dinfo);
  cudaFree(dwork);
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
  return dev <= 1e-13 * mx;
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
  X.G = dalloc<double>(half);
  X.Hh = dalloc<double>(8 * static_cast<size_t>(n2) * n2);
  X.R = dalloc<double>(8 * static_cast<size_t>(n2) * n2);
  return X;
}

// Fast diagonalisation of W = M(x)S + S(x)M - c M(x)M: S V = M V diag(lam),
// V^T M V = I (cuSOLVER sygvd at setup), Dinv = 1/(lam_i + lam_j - c).
static ExactSolver make_fd(cudaStream_t st, const Band& S, const Band& M, double2 c) {
  ExactSolver X;
  X.dim = 2;
  X.n = S.n;
  const int n = S.n;
  std::vector<double> As = dense_of(S), Bm = dense_of(M);
  double *dA = dalloc<double>(As.size()), *dB = dalloc<double>(Bm.size()), *dW = dalloc<double>(n);
  int* dinfo = dalloc<int>(1);
  CK(cudaMemcpy(dA, As.data(), As.size() * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, Bm.data(), Bm.size() * sizeof(double), cudaMemcpyHostToDevice));
  cusolverDnHandle_t h;
  CKS(cusolverDnCreate(&h));
  CKS(cusolverDnSetStream(h, st));
  int lwork = 0;
  CKS(cusolverDnDsygvd_bufferSize(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n,
                                  dB, n, dW, &lwork));
  double* dwork = dalloc<double>(std::max(lwork, 1));
  CKS(cusolverDnDsygvd(h, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, dA, n, dB, n, dW,
                       dwork, lwork, dinfo));
  int info = 0;
  CK(cudaMemcpyAsync(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cusolverDnDestroy(h);
  if (info != 0) throw Error(HD_ERR_FACTOR, "coarse operator factorization failed (sygvd info " + std::to_string(info) + ")");
  std::vector<double> lam(n);
  CK(cudaMemcpy(lam.data(), dW, n * sizeof(double), cudaMemcpyDeviceToHost));
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
  cudaFree(dB);
  cudaFree(dW);
  cudaFree(dinfo);
  cudaFree(dwork);
  return X;
}

// Partial fast diagonalisation of a real-shift Kronecker sum (E): V from the
// x eigenproblem (as make_fd); for every x mode the real banded y operator
// T_m = S - (c - lam_m) M, LU-factored with partial pivoting (band_lu), and the
// influence rows / boundary maps of its kYL-row segments (ysolve.cuh).
static ExactSolver make_fd_ypart(cudaStream_t st, const Band& S, const Band& M, double2 c) {
  const int n = S.n, kl = std::max(S.b, M.b), ku = 2 * kl, W = kl + 1;
  ExactSolver X;
  X.dim = 2;
  X.n = n;
  X.ypart = true;
  X.ykl = kl;
  X.V = dalloc<double>(static_cast<size_t>(n) * n);
  std::vector<double> lam;
  sygvd_device(st, dense_of(S), dense_of(M), n, X.V, lam);
  const int np = (n + 31) / 32 * 32, Sg = (n + kYL - 1) / kYL, nr = Sg * kYL;
  const int NF = 2 * kl + 2, NB = 2 * ku + 1;
  std::vector<double> TF(static_cast<size_t>(nr) * NF * np, 0.0), TB(static_cast<size_t>(nr) * NB * np, 0.0),
      FM(static_cast<size_t>(Sg) * W * W * np, 0.0), HM(static_cast<size_t>(Sg) * ku * ku * np, 0.0);
  std::vector<double> Lk, Uk;
  std::vector<int> pk;
  for (int m = 0; m < np; ++m) {
    // factors of mode m, padded rows / modes = identity
    Lk.assign(static_cast<size_t>(nr) * kl, 0.0);
    Uk.assign(static_cast<size_t>(nr) * (ku + 1), 0.0);
    pk.assign(nr, 0);
    for (int k = 0; k < nr; ++k) Uk[static_cast<size_t>(k) * (ku + 1)] = 1.0;
    if (m < n) {
      const BandLU f = band_lu(S, M, cplx(c.x - lam[m], 0.0));
      if (f.kl != kl || f.ku != ku) throw Error(HD_ERR_INVALID, "unexpected band LU shape");
      for (int k = 0; k < n; ++k) {
        for (int q = 0; q < kl; ++q) Lk[static_cast<size_t>(k) * kl + q] = f.L[static_cast<size_t>(k) * kl + q].real();
        for (int d = 0; d <= ku; ++d) Uk[static_cast<size_t>(k) * (ku + 1) + d] = f.U[static_cast<size_t>(k) * (ku + 1) + d].real();
        pk[k] = f.piv[k] - k;
        if (Uk[static_cast<size_t>(k) * (ku + 1)] == 0.0) throw Error(HD_ERR_FACTOR, "deflation matrix E is singular");
      }
    }
    for (int k = 0; k < nr; ++k) {
      double* tf = &TF[static_cast<size_t>(k) * NF * np + m];
      for (int q = 0; q < kl; ++q) tf[static_cast<size_t>(q) * np] = Lk[static_cast<size_t>(k) * kl + q];
      tf[static_cast<size_t>(kl) * np] = pk[k];
      double* tb = &TB[static_cast<size_t>(k) * NB * np + m];
      tb[0] = 1.0 / Uk[static_cast<size_t>(k) * (ku + 1)];
      for (int d = 1; d <= ku; ++d) tb[static_cast<size_t>(d) * np] = Uk[static_cast<size_t>(k) * (ku + 1) + d];
    }
    for (int i = 0; i < Sg; ++i) {
      const int s0 = i * kYL, e0 = s0 + kYL;
      for (int q = 0; q < W; ++q) {  // forward from window e_q, no rhs
        std::vector<double> w(W, 0.0);
        w[q] = 1.0;
        for (int k = s0; k < e0; ++k) {
          const int p = pk[k];
          if (p != 0) std::swap(w[0], w[p]);
          const double yk = w[0];
          TF[(static_cast<size_t>(k) * NF + kl + 1 + q) * np + m] = yk;
          for (int r = 1; r <= kl; ++r) w[r] -= Lk[static_cast<size_t>(k) * kl + r - 1] * yk;
          for (int r = 0; r < kl; ++r) w[r] = w[r + 1];
          w[kl] = 0.0;
        }
        for (int r = 0; r < W; ++r) FM[((static_cast<size_t>(i) * W + r) * W + q) * np + m] = w[r];
      }
      for (int r = 0; r < ku; ++r) {  // backward from future x_{e+r} = 1, no rhs
        std::vector<double> xw(ku, 0.0);
        xw[r] = 1.0;
        for (int k = e0 - 1; k >= s0; --k) {
          double acc = 0.0;
          for (int d = ku; d >= 1; --d) acc -= Uk[static_cast<size_t>(k) * (ku + 1) + d] * xw[d - 1];
          const double xk = acc / Uk[static_cast<size_t>(k) * (ku + 1)];
          for (int d = ku - 1; d >= 1; --d) xw[d] = xw[d - 1];
          xw[0] = xk;
          TB[(static_cast<size_t>(k) * NB + ku + 1 + r) * np + m] = xk;
          if (k - s0 < ku) HM[((static_cast<size_t>(i) * ku + (k - s0)) * ku + r) * np + m] = xk;
        }
      }
    }
  }
  auto up = [](const std::vector<double>& v) {
    double* d = dalloc<double>(v.size());
    CK(cudaMemcpy(d, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice));
    return d;
  };
  YArgs& a = X.ya;
  a.n = n;
  a.np = np;
  a.S = Sg;
  a.nr = nr;
  a.TF = up(TF);
  a.TB = up(TB);
  a.FM = up(FM);
  a.HM = up(HM);
  a.Y = dalloc<double>(2 * static_cast<size_t>(nr) * np);
  a.X0 = dalloc<double>(2 * static_cast<size_t>(nr) * np);
  a.D = dalloc<double>(2 * static_cast<size_t>(Sg) * W * np);
  a.Dl = dalloc<double>(2 * static_cast<size_t>(Sg) * W * np);
  a.XS = dalloc<double>(2 * static_cast<size_t>(Sg) * ku * np);
  a.XB = dalloc<double>(2 * static_cast<size_t>(Sg + 1) * ku * np);
  X.T1 = dalloc<double>(2 * static_cast<size_t>(n) * np);
  CK(cudaMemset(X.T1, 0, 2 * static_cast<size_t>(n) * np * sizeof(double)));
  a.C = X.T1;
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
  return X;
}

static void free_exact(ExactSolver& X) {
  cudaFree(X.V); cudaFree(X.Dinv); cudaFree(X.T1); cudaFree(X.T2);
  cudaFree(X.Vt); cudaFree(X.Dinvf); cudaFree(X.F); cudaFree(X.G); cudaFree(X.Hh); cudaFree(X.R);
  cudaFree(X.L); cudaFree(X.U); cudaFree(X.piv); cudaFree(X.work); cudaFree(X.Uinv);
  if (X.ypart) {
    cudaFree(const_cast<double*>(X.ya.TF)); cudaFree(const_cast<double*>(X.ya.TB));
    cudaFree(const_cast<double*>(X.ya.FM)); cudaFree(const_cast<double*>(X.ya.HM));
    cudaFree(X.ya.Y); cudaFree(X.ya.X0); cudaFree(X.ya.D); cudaFree(X.ya.Dl); cudaFree(X.ya.XS); cudaFree(X.ya.XB);
  }
  if (X.seg.P) {
    for (const void* p : {static_cast<const void*>(X.seg.L), static_cast<const void*>(X.seg.pv),
                          static_cast<const void*>(X.seg.hf), static_cast<const void*>(X.seg.U),
                          static_cast<const void*>(X.seg.Ui), static_cast<const void*>(X.seg.hb),
                          static_cast<const void*>(X.seg.Ff), static_cast<const void*>(X.seg.Hb)})
      cudaFree(const_cast<void*>(p));
    cudaFree(X.seg.y); cudaFree(X.seg.x0); cudaFree(X.seg.D);
    cudaFree(X.seg.Dl); cudaFree(X.seg.X0); cudaFree(X.seg.Xb);
  }
  cudaFree(X.Ainv); cudaFree(X.dx); cudaFree(X.dy);
  if (X.btri) {
    cudaFree(const_cast<void*>(X.bt.GT)); cudaFree(const_cast<void*>(X.bt.SinvT));
    cudaFree(const_cast<void*>(X.bt.HT)); cudaFree(const_cast<void*>(X.bt.G2)); cudaFree(X.bt.y); cudaFree(X.bt.bar);
  }
  X = ExactSolver{};
}

template <int KL>
static void bandlu_launch_t(cudaStream_t st, const ExactSolver& X, const double2* b, const double* bp, double2* x,
                            double* xp) {
  static bool attr = false;
  constexpr size_t sm = bandlu_smem<KL>();
  if (!attr) {
    CK(cudaFuncSetAttribute(k_bandlu_staged<KL>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    attr = true;
  }
  k_bandlu_staged<KL><<<1, 256, sm, st>>>(X.L, X.U, X.Uinv, X.piv, X.n, b, bp, X.work, x, xp);
}

template <int KL>
static void seg_launch_t(cudaStream_t st, const ExactSolver& X, const double2* b, const double* bp, double2* x,
                         double* xp) {
  const SegArgs& a = X.seg;
  const int blocks = (a.P + 31) / 32;
  k_seg_fwd<KL><<<blocks, 32, 0, st>>>(a, b, bp);
  k_seg_scan_fwd<KL><<<1, 32, 0, st>>>(a);
  k_seg_bwd<KL><<<blocks, 32, 0, st>>>(a);
  k_seg_scan_bwd<KL><<<1, 32, 0, st>>>(a);
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

// called right after a launch: error check, launch count, profile record
static void launched(hd_ctx* c, int kind, size_t mark, double bytes, bool library = false) {
  CK(cudaGetLastError());
  if (library) ++c->lib_calls;
  else ++c->launches;
  if (mark == static_cast<size_t>(-1)) return;
  prof_mark(c);
  c->prof_recs.push_back({kind, mark, bytes});
}

#define HD_LAUNCH(kind, bytes, ...)        \
  do {                                     \
    const size_t mk_ = prof_mark(c);       \
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
    default: return 3 * P;
  }
}

// Per instantiation: opt in to the dynamic shared memory of the tallest strip
// and query how many CTAs are resident per SM.
template <int B, int MODE>
static int stencil_occupancy() {
  static int per = 0;
  if (!per) {
    constexpr size_t sm = stencil_smem<B, MODE>(kSRowsMax);
    CK(cudaFuncSetAttribute(k_stencil2d<B, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_stencil2d<B, MODE>, kSW * kSWarps, sm));
    per = std::max(per, 1);
  }
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

template <int B, int MODE>
static void launch_stencil(hd_ctx* c, const LevelDev& L, const double2* x, const double2* b, double2* out,
                           double omega, RedOut red, const int* xidx, size_t xstride, int rb, int re) {
  const int per = stencil_occupancy<B, MODE>();
  const int ry = pick_rows(L.n, re - rb, per * c->n_sms, B);
  dim3 grid((L.n + kSW * kSWarps - 1) / (kSW * kSWarps), (re - rb + ry - 1) / ry);
  k_stencil2d<B, MODE><<<grid, kSW * kSWarps, stencil_smem<B, MODE>(ry), c->st>>>(L, x, b, out, omega, ry, red,
                                                                               xidx, xstride, rb, re);
}

template <int MODE>
static void launch_op2d_mode(hd_ctx* c, const LevelDev& L, const double2* x, const double2* b, double2* out,
                             double omega, RedOut red, int kind, const int* xidx, size_t xstride, int rb = 0,
                             int re = -1) {
  if (re < 0) re = L.n;
  const size_t mk = prof_mark(c);
  switch (L.b) {
#define HD_CASE(BB) \
  case BB: launch_stencil<BB, MODE>(c, L, x, b, out, omega, red, xidx, xstride, rb, re); break;
    HD_CASE(1) HD_CASE(2) HD_CASE(3) HD_CASE(4) HD_CASE(5) HD_CASE(6)
#undef HD_CASE
    default: throw Error(HD_ERR_INVALID, "band half-width " + std::to_string(L.b) + " unsupported");
  }
  launched(c, kind, mk, op_bytes(MODE, static_cast<size_t>(L.n) * (re - rb)));
}

// layered field: G-term Kronecker-sum operator (layered.cuh)
template <int MODE>
static void launch_gen_mode(hd_ctx* c, const GenLevel& G, const double2* x, const double2* b, double2* out,
                            double omega, RedOut red, int kind, const int* xidx, size_t xstride) {
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(k_kron2d<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(gen_smem(6, kGenMaxG))));
    attr = true;
  }
  if (G.b > 6 || G.G > kGenMaxG) throw Error(HD_ERR_INVALID, "layered operator exceeds the kernel limits");
  const dim3 grid((G.n + kGenTX - 1) / kGenTX, (G.n + kGenTY - 1) / kGenTY);
  HD_LAUNCH(kind, op_bytes(MODE, static_cast<size_t>(G.n) * G.n),
            k_kron2d<MODE><<<grid, kGenThreads, gen_smem(G.b, G.G), c->st>>>(G, x, b, out, omega, red, xidx,
                                                                               xstride));
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
      case OP_APPLY: launch_gen_mode<OP_APPLY>(c, G, x, b, out, omega, red, kind, xidx, xstride); break;
      case OP_RESID: launch_gen_mode<OP_RESID>(c, G, x, b, out, omega, red, kind, xidx, xstride); break;
      case OP_JACOBI: launch_gen_mode<OP_JACOBI>(c, G, x, b, out, omega, red, kind, xidx, xstride); break;
      default: launch_gen_mode<OP_RESNORM>(c, G, x, b, out, omega, red, kind, xidx, xstride); break;
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
    HD_LAUNCH(HD_K_JACOBI0, 32.0 * NN,
              k_jacobi0_gen<<<grid_for(NN), 256, 0, c->st>>>(*static_cast<const GenLevel*>(L.gen), b, out, omega));
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
  static size_t attr = 0;
  if (smem > attr) {
    CK(cudaFuncSetAttribute(k_btri_solve<T, KR>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr = smem;
  }
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

// Exact solve: in/out planar (2D FD) or via the banded LU (1D).
template <int KL>
static void ysolve_launch_t(hd_ctx* c, const YArgs& a) {
  const dim3 gs(a.np / 32, a.S), gm((a.np + 127) / 128), go(a.np / 32, a.n);
  k_ys_fwd<KL><<<gs, 32, 0, c->st>>>(a);
  k_ys_scan_fwd<KL><<<gm, 128, 0, c->st>>>(a);
  k_ys_bwd<KL><<<gs, 32, 0, c->st>>>(a);
  k_ys_scan_bwd<KL><<<gm, 128, 0, c->st>>>(a);
  k_ys_out<KL><<<go, 32, 0, c->st>>>(a);
}

static void ysolve_launch(hd_ctx* c, const ExactSolver& X) {
  switch (X.ykl) {
    case 1: ysolve_launch_t<1>(c, X.ya); break;
    case 2: ysolve_launch_t<2>(c, X.ya); break;
    case 3: ysolve_launch_t<3>(c, X.ya); break;
    case 4: ysolve_launch_t<4>(c, X.ya); break;
    case 5: ysolve_launch_t<5>(c, X.ya); break;
    case 6: ysolve_launch_t<6>(c, X.ya); break;
    default: throw Error(HD_ERR_INVALID, "E band outside the y-solve kernels");
  }
}

static void exact_solve_planar(hd_ctx* c, ExactSolver& X, double* inout) {
  if (X.ypart) {
    const int n = X.n, np = X.ya.np;
    const long nn = static_cast<long>(n) * n;
    const double one = 1.0, zero = 0.0;
    const double gb = 16.0 * nn * 2 + 8.0 * nn;
    size_t mk = prof_mark(c);
    // C = V^T [Xre | Xim]  (x modes), leading dimension np
    CKB(cublasDgemm(c->cb, CUBLAS_OP_T, CUBLAS_OP_N, n, 2 * n, n, &one, X.V, n, inout, n, &zero, X.T1, np));
    launched(c, HD_K_LIBGEMM, mk, gb, true);
    // segmented banded sweeps along y for every mode (5 kernels)
    HD_LAUNCH(HD_K_EXACT, 8.0 * X.ya.nr * np * (2 * X.ykl + 2 + 4 * X.ykl + 1) + 64.0 * nn, ysolve_launch(c, X));
    c->launches += 4;
    mk = prof_mark(c);
    // out = V [Yre | Yim]
    CKB(cublasDgemm(c->cb, CUBLAS_OP_N, CUBLAS_OP_N, n, 2 * n, n, &one, X.V, n, X.T1, np, &zero, inout, n));
    launched(c, HD_K_LIBGEMM, mk, gb, true);
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
    const long nn = static_cast<long>(n2) * n2;
    const long hc = static_cast<long>(n2) * 2 * n;  // one parity of a half-folded n2 x 2n block
    const double one = 1.0, zero = 0.0;
    const double gb = 16.0 * nn * 4;               // nominal bytes per GEMM call (profiling)
    HD_LAUNCH(HD_K_EXACT, 32.0 * n * n, k_fold_rows<<<grid_for(hc), 256, 0, c->st>>>(inout, X.F, n, n2, 2 * n));
    size_t mk = prof_mark(c);
    // x transform: G_b = Vt_b^T F_b
    CKB(cublasDgemmStridedBatched(c->cb, CUBLAS_OP_T, CUBLAS_OP_N, n2, 2 * n, n2, &one, X.Vt, n2, nn, X.F, n2, hc,
                                  &zero, X.G, n2, hc, 2));
    launched(c, HD_K_LIBGEMM, mk, gb, true);
    HD_LAUNCH(HD_K_EXACT, 32.0 * n * n, k_fold_cols<<<grid_for(4 * nn), 256, 0, c->st>>>(X.G, X.Hh, n, n2));
    // y transform: R[yb] = Hh[yb] Vt_yb (batch over x parity and plane)
    for (int yb = 0; yb < 2; ++yb) {
      mk = prof_mark(c);
      CKB(cublasDgemmStridedBatched(c->cb, CUBLAS_OP_N, CUBLAS_OP_N, n2, n2, n2, &one, X.Hh + yb * 4 * nn, n2, nn,
                                    X.Vt + yb * nn, n2, 0, &zero, X.R + yb * 4 * nn, n2, nn, 4));
      launched(c, HD_K_LIBGEMM, mk, gb, true);
    }
    HD_LAUNCH(HD_K_EXACT, 48.0 * 4 * nn, k_scale_folded<<<grid_for(4 * nn), 256, 0, c->st>>>(X.R, X.Dinvf, n2));
    // inverse y: S[yb] = R[yb] Vt_yb^T  (into Hh)
    for (int yb = 0; yb < 2; ++yb) {
      mk = prof_mark(c);
      CKB(cublasDgemmStridedBatched(c->cb, CUBLAS_OP_N, CUBLAS_OP_T, n2, n2, n2, &one, X.R + yb * 4 * nn, n2, nn,
                                    X.Vt + yb * nn, n2, 0, &zero, X.Hh + yb * 4 * nn, n2, nn, 4));
      launched(c, HD_K_LIBGEMM, mk, gb, true);
    }
    HD_LAUNCH(HD_K_EXACT, 32.0 * n * n, k_unfold_cols<<<grid_for(4 * nn), 256, 0, c->st>>>(X.Hh, X.F, n, n2));
    // inverse x: Yh_b = Vt_b Z_b  (Z in F, result in G)
    mk = prof_mark(c);
    CKB(cublasDgemmStridedBatched(c->cb, CUBLAS_OP_N, CUBLAS_OP_N, n2, 2 * n, n2, &one, X.Vt, n2, nn, X.F, n2, hc,
                                  &zero, X.G, n2, hc, 2));
    launched(c, HD_K_LIBGEMM, mk, gb, true);
    HD_LAUNCH(HD_K_EXACT, 32.0 * n * n, k_unfold_rows<<<grid_for(hc), 256, 0, c->st>>>(X.G, inout, n, n2, 2 * n));
    return;
  }
  if (X.dim == 2) {
    const int n = X.n;
    const long nn = static_cast<long>(n) * n;
    const double one = 1.0, zero = 0.0;
    const double gb = 16.0 * nn * 2 + 8.0 * nn;  // planar in/out + V  (bytes of one GEMM)
    size_t mk = prof_mark(c);
    // T1 = V^T [Xre | Xim]
    CKB(cublasDgemm(c->cb, CUBLAS_OP_T, CUBLAS_OP_N, n, 2 * n, n, &one, X.V, n, inout, n, &zero, X.T1, n));
    launched(c, HD_K_LIBGEMM, mk, gb, true);
    mk = prof_mark(c);
    // T2_plane = T1_plane V
    CKB(cublasDgemmStridedBatched(c->cb, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, X.T1, n, nn, X.V, n, 0, &zero,
                                  X.T2, n, nn, 2));
    launched(c, HD_K_LIBGEMM, mk, gb, true);
    HD_LAUNCH(HD_K_EXACT, 48.0 * nn, k_fd_scale<<<grid_for(nn), 256, 0, c->st>>>(X.T2, X.Dinv, nn));
    mk = prof_mark(c);
    // T1 = V [T2re | T2im]
    CKB(cublasDgemm(c->cb, CUBLAS_OP_N, CUBLAS_OP_N, n, 2 * n, n, &one, X.V, n, X.T2, n, &zero, X.T1, n));
    launched(c, HD_K_LIBGEMM, mk, gb, true);
    mk = prof_mark(c);
    // out_plane = T1_plane V^T
    CKB(cublasDgemmStridedBatched(c->cb, CUBLAS_OP_N, CUBLAS_OP_T, n, n, n, &one, X.T1, n, nn, X.V, n, 0, &zero,
                                  inout, n, nn, 2));
    launched(c, HD_K_LIBGEMM, mk, gb, true);
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
static double2* smooth(hd_ctx* c, int l, const double2* b, double2* xa, double2* xb, bool x_zero, int steps) {
  const LevelDev L = levM(c, l);
  double2* cur = xa;
  double2* oth = xb;
  int s = 0;
  if (x_zero) {
    if (steps == 0) {
      CK(cudaMemsetAsync(cur, 0, lsize(c, L.n) * sizeof(double2), c->st));
      return cur;
    }
    jacobi0(c, L, b, cur, c->spec.omega);
    s = 1;
  }
  for (; s < steps; ++s) {
    op_apply(c, OP_JACOBI, L, cur, b, oth, c->spec.omega);
    std::swap(cur, oth);
  }
  return cur;
}

// One V-cycle at level l (src/precond.cpp:144-153); returns the buffer holding x.
static double2* cycle_at(hd_ctx* c, int l, const double2* b, bool x_zero) {
  const int last = static_cast<int>(c->lev.size()) - 1;
  if (l == last) {
    coarsest_solve(c, b, c->mg_x[l]);
    return c->mg_x[l];
  }
  const LevelDev L = levM(c, l);
  double2* xcur = smooth(c, l, b, c->mg_x[l], c->mg_y[l], x_zero, c->spec.smooth_steps);
  double2* xoth = xcur == c->mg_x[l] ? c->mg_y[l] : c->mg_x[l];
  op_apply(c, OP_RESID, L, xcur, b, c->mg_r[l]);
  const int nf = c->lev[l].n, ncl = c->lev[l + 1].n;
  restrict_(c, Stencil{0, 0.0}, c->mg_r[l], nf, ncl, c->mg_b[l + 1], nullptr);
  double2* ec = cycle_at(c, l + 1, c->mg_b[l + 1], true);
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

static void mg_solve(hd_ctx* c, const double2* b, double2* out) {
  const size_t N = c->N;
  if (c->spec.cycles <= 0) {
    shift_exact_solve(c, b, out);
    return;
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
      xb = cycle_at(c, 0, b, true);
    } else {
      // general cycle from a non-zero iterate held in mg_x[0]
      const LevelDev L = levM(c, 0);
      double2* xcur = smooth(c, 0, b, c->mg_x[0], c->mg_y[0], false, c->spec.smooth_steps);
      double2* xoth = xcur == c->mg_x[0] ? c->mg_y[0] : c->mg_x[0];
      op_apply(c, OP_RESID, L, xcur, b, c->mg_r[0]);
      restrict_(c, Stencil{0, 0.0}, c->mg_r[0], c->lev[0].n, c->lev[1].n, c->mg_b[1], nullptr);
      double2* ec = cycle_at(c, 1, c->mg_b[1], true);
      prolong_<0>(c, Stencil{0, 0.0}, ec, nullptr, c->lev[0].n, c->lev[1].n, nullptr, xcur);
      xb = smooth(c, 0, b, xcur, xoth, false, c->spec.smooth_steps);
    }
    zero = false;
  }
  if (c->spec.cycles <= 0) {
    CK(cudaMemsetAsync(out, 0, N * sizeof(double2), c->st));
    return;
  }
  CK(cudaMemcpyAsync(out, xb, N * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
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
  op_apply(c, OP_APPLY, opA(c), w, nullptr, c->t3);
  restrict_(c, z, c->t3, c->n, c->nc, nullptr, c->ep);
  exact_solve_planar(c, c->E, c->ep);
  prolong_<1>(c, z, nullptr, c->ep, c->n, c->nc, w, out);
}

// out = op(v) = P MG^-1 A v  (src/precond.cpp:236-245); v, out distinct from t1, t2, t3
static void compose_op(hd_ctx* c, const double2* v, double2* out, const int* vidx = nullptr) {
  ++c->matvecs;
  op_apply(c, OP_APPLY, opA(c), v, nullptr, c->t1, 0.0, nullptr, 1.0, vidx, c->N);
  const double2* cur = c->t1;
  if (c->spec.shift) {
    ++c->shift_solves;
    c->vcycles += c->spec.cycles;
    mg_solve(c, c->t1, c->t2);
    cur = c->t2;
  }
  if (c->spec.deflate) {
    ++c->coarse_solves;
    project(c, cur, out);
  } else {
    CK(cudaMemcpyAsync(out, cur, c->N * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
  }
}

// Chooses the persistent Arnoldi geometry: G CTAs of kArnBD threads (<= one
// per SM), each owning `chunk` elements, K per thread; shared memory holds the
// non-register part of w and, in block 0, the packed R of the back substitution.
static void setup_arnoldi(hd_ctx* c, int maxit) {
  int dev_sms = 0, smem_optin = 0;
  CK(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->device));
  CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
  const size_t N = c->N;
  const size_t per_thread_target = 4;
  int G = static_cast<int>(std::min<size_t>(dev_sms, std::max<size_t>(1, (N + kArnBD * per_thread_target - 1) /
                                                                             (kArnBD * per_thread_target))));
  const size_t chunk = (N + G - 1) / G;
  const int K = static_cast<int>((chunk + kArnBD - 1) / kArnBD);
  const size_t w_smem = static_cast<size_t>(std::max(0, K - kArnRW)) * kArnBD * sizeof(double2);
  const size_t r_smem = (static_cast<size_t>(maxit + 1) * (maxit + 2) / 2 + 4 * (maxit + 2) + 8) * sizeof(double2);
  const size_t smem = std::max(w_smem, r_smem);
  c->use_arnoldi = false;
  if (maxit > 127) return;  // y staged in 128 shared slots
  if (smem + 4096 > static_cast<size_t>(smem_optin)) return;  // w does not fit on chip: per-step kernels
  CK(cudaFuncSetAttribute(k_arnoldi<kArnRW>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_arnoldi<kArnRW>, kArnBD, smem));
  if (per_sm < 1) return;
  c->arn_G = G;
  c->arn_K = K;
  c->arn_chunk = chunk;
  c->arn_smem = smem;
  if (!c->dj) c->dj = dalloc<int>(4);
  if (!c->arn_partials) c->arn_partials = dalloc<double2>(2 * static_cast<size_t>(dev_sms) + 8);
  if (!c->arn_bar) c->arn_bar = dalloc<unsigned>(4);
  if (!c->arn_trace && std::getenv("HD_TRACE")) {
    CK(cudaMallocHost(&c->arn_trace, 8 * sizeof(unsigned long long)));
  }
  c->use_arnoldi = true;
}

static void launch_arnoldi(hd_ctx* c, double2* xout, int maxit, const int* done, double bytes) {
  ArnoldiArgs a;
  a.V = c->V;
  a.Vw = c->V;
  a.w = c->w;
  a.x0 = c->x0;
  a.x = xout;
  a.N = c->N;
  a.dj = c->dj;
  a.done = done;
  a.H = c->H;
  a.ldh = maxit + 1;
  a.g = c->g;
  a.cs = c->cs;
  a.sn = c->sn;
  a.y = c->y;
  a.hnew_out = c->dres + 1;
  a.partials = c->arn_partials;
  a.bar = c->arn_bar;
  a.K = c->arn_K;
  a.chunk = c->arn_chunk;
  a.trace = c->arn_trace;
  CK(cudaMemsetAsync(c->arn_bar, 0, sizeof(unsigned), c->st));
  void* args[] = {&a};
  const double P = 16.0 * static_cast<double>(c->N);
  (void)P;
  const size_t mk = prof_mark(c);
  CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_arnoldi<kArnRW>), dim3(c->arn_G), dim3(kArnBD), args,
                                 c->arn_smem, c->st));
  launched(c, HD_K_MGS, mk, bytes);
}

static void ensure_gmres(hd_ctx* c, int maxit) {
  if (maxit + 1 > c->v_cap) {
    cudaFree(c->V);
    c->V = dalloc<double2>(static_cast<size_t>(maxit + 1) * c->N);
    c->v_cap = maxit + 1;
  }
  if (maxit > c->maxit_cap) {
    cudaFree(c->H); cudaFree(c->g); cudaFree(c->cs); cudaFree(c->sn); cudaFree(c->y);
    c->H = dalloc<double2>(static_cast<size_t>(maxit + 1) * maxit);
    c->g = dalloc<double2>(maxit + 1);
    c->cs = dalloc<double2>(maxit);
    c->sn = dalloc<double2>(maxit);
    c->y = dalloc<double2>(maxit);
    c->maxit_cap = maxit;
  }
  if (maxit != c->arn_maxit) {
    setup_arnoldi(c, maxit);
    c->arn_maxit = maxit;
  }
  if (maxit != c->lsa_maxit && maxit + 1 <= kLsaMaxJ) {
    int sms = 0, per = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    CK(cudaFuncSetAttribute(k_lsa_dots, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(lsa_dots_smem())));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_lsa_dots, kLsaBD, lsa_dots_smem()));
    int per2 = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_lsa_update, kLsaBD, 0));
    per = std::max(1, std::min(per, per2));
    const size_t tiles = (c->N + static_cast<size_t>(kLsaBD) * kLsaTE - 1) / (static_cast<size_t>(kLsaBD) * kLsaTE);
    c->lsa_G = static_cast<int>(std::max<size_t>(1, std::min<size_t>(tiles, static_cast<size_t>(sms) * per)));
    cudaFree(c->lsa_sig); cudaFree(c->lsa_L); cudaFree(c->lsa_ch); cudaFree(c->lsa_cx); cudaFree(c->lsa_partials);
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
    CK(cudaFuncSetAttribute(k_lsa_givens, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(c->lsa_givens_smem)));
    c->lsa_maxit = maxit;
  }
}

static LsaArgs lsa_args(hd_ctx* c, double2* xout, int j, int mode, int maxit) {
  LsaArgs a;
  a.jlag = 0;
  a.part_offset = 0;
  a.partial_only = 0;
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
}

__global__ void k_scale_monitor(double* dres) {  // graph monitor: raw norm / (||f|| or 1)
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
  cudaFree(c->res_hist);
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
  CK(cudaEventRecord(c->ev_join, c->st2));
  compose_op(c, c->V, c->w, dj);
  CK(cudaStreamWaitEvent(c->st, c->ev_join, 0));
  k_lsa_dots<<<G, kLsaBD, lsa_dots_smem(), c->st>>>(a);
  k_lsa_update<<<G, kLsaBD, 0, c->st>>>(a);  // u_{j+1} and the lagged x_{j-1}
  monitor_raw(c, c->x);
  k_scale_monitor<<<1, 1, 0, c->st>>>(c->dres);
  k_loop_check<<<1, 1, 0, c->st>>>(c->loop_state, c->dres, c->res_hist, tol, h);
  k_loop_next<<<1, 1, 0, c->st>>>(c->loop_state, maxit, h);
  cudaGraph_t captured = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(c->st, &captured);
  c->prof_on = prof;
  c->graph_body_kernels = c->launches - saved_l + 6;  // op + monitor kernels + dots/scale/check/update/givens/next
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
}

struct SolveOut {
  int iterations = 0;
  bool converged = false;
  std::vector<double> residuals;
};

// gmres(setup.op, setup.rhs, setup.start, setup.monitor, opt) after the
// compose() right-hand side / start transforms; f already in c->f.
static SolveOut run_solve(hd_ctx* c, const hd_gmres& opt, double2* xout) {
  const size_t N = c->N;
  const int maxit = opt.max_iterations;
  ensure_gmres(c, std::max(maxit, 1));
  c->matvecs = c->coarse_solves = c->shift_solves = c->vcycles = 0;
  c->launches = c->lib_calls = 0;
  const int nb = c->red_blocks;
  const double P = 16.0 * static_cast<double>(N);
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
  read_scalars(c);
  const double fnorm = c->hres[3];
  const double scale = fnorm > 0.0 ? fnorm : 1.0;

  SolveOut res;
  auto monitor = [&](const double2* xv) {
    op_apply(c, OP_RESNORM, opA(c), xv, c->f, nullptr, 0.0, c->dres + 0, scale);
  };
  monitor(c->x0);
  read_scalars(c);
  const double r0 = c->hres[0];
  if (r0 <= opt.tolerance) {  // src/linalg.cpp:17-22
    res.converged = true;
    res.residuals.push_back(r0);
    CK(cudaMemcpyAsync(xout, c->x0, N * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
    return res;
  }
  // r = rhs' - op(x0); beta = ||r||; V0 = r / beta  (src/linalg.cpp:24-33)
  compose_op(c, c->x0, c->w);
  HD_LAUNCH(HD_K_VEC, 3 * P, k_sub<<<grid_for(N), 256, 0, c->st>>>(c->rhsp, c->w, c->w, N));
  HD_LAUNCH(HD_K_VEC, P, k_axpy_norm<<<nb, 256, 0, c->st>>>(c->w, nullptr, nullptr, N, red_of(c, c->dres + 2), c->g));
  read_scalars(c);
  const double beta = c->hres[2];
  if (beta == 0.0) {
    monitor(c->x0);
    read_scalars(c);
    res.converged = c->hres[0] <= opt.tolerance;
    CK(cudaMemcpyAsync(xout, c->x0, N * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
    return res;
  }
  CK(cudaMemsetAsync(c->H, 0, sizeof(double2) * (maxit + 1) * maxit, c->st));
  CK(cudaMemsetAsync(c->g + 1, 0, sizeof(double2) * maxit, c->st));
  HD_LAUNCH(HD_K_VEC, 2 * P, k_scale_inv<<<grid_for(N), 256, 0, c->st>>>(c->V, c->w, c->dres + 2, N));
  const int ldh = maxit + 1;
  if (c->arn_mode == 2 && maxit + 1 <= kLsaMaxJ) {
    // u_0 = r (unnormalised), sigma_0 = 1 / beta
    CK(cudaMemcpyAsync(c->V, c->w, N * sizeof(double2), cudaMemcpyDeviceToDevice, c->st));
    HD_LAUNCH(HD_K_VEC, 0.0, k_inv_scalar<<<1, 1, 0, c->st>>>(c->lsa_sig, c->dres + 2));
    const int G = c->lsa_G;
    if (c->graph_enabled && !c->prof_on) {
      if (c->loop_maxit != maxit || c->loop_tol != opt.tolerance) build_loop_graph(c, maxit, opt.tolerance);
      k_loop_init<<<1, 1, 0, c->st>>>(c->loop_state);
      CK(cudaGraphLaunch(c->loop_exec, c->st));
      CK(cudaMemcpyAsync(c->loop_host, c->loop_state, sizeof(LoopState), cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(c->res_host, c->res_hist, maxit * sizeof(double), cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      const LoopState ls = *c->loop_host;
      // per-iteration launches of the body (op + 7) for the report
      int it = ls.iters;
      res.iterations = it;
      res.converged = ls.conv != 0;
      for (int q = 0; q < (ls.need_tail ? maxit - 1 : it); ++q) res.residuals.push_back(c->res_host[q]);
      if (ls.need_tail) {  // x_{maxit-1}: its Givens, an iterate-only pass + monitor
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
      HD_LAUNCH(HD_K_MGS, (j + 3.0) * P, k_lsa_dots<<<G, kLsaBD, lsa_dots_smem(), c->st>>>(a));
      HD_LAUNCH(HD_K_MGS, (j >= 1 ? j + 5.0 : 3.0) * P, k_lsa_update<<<G, kLsaBD, 0, c->st>>>(a));
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
  const bool persistent = c->use_arnoldi && c->arn_mode == 1;
  if (persistent) CK(cudaMemsetAsync(c->dj, 0, sizeof(int), c->st));
  for (int j = 0; j < maxit && persistent; ++j) {
    compose_op(c, c->V + static_cast<size_t>(j) * N, c->w);
    // w in, V_0..V_j (MGS), V_{j+1} out, x0 + V_0..V_j in + x out (iterate)
    launch_arnoldi(c, xout, maxit, nullptr, (2.0 * j + 6.0) * P);
    res.iterations = j + 1;
    monitor(xout);
    read_scalars(c);
    if (c->arn_trace) {
      const unsigned long long* q = c->arn_trace;
      c->arn_phase_ns[0] += static_cast<double>(q[1] - q[0]);  // MGS chain
      c->arn_phase_ns[1] += static_cast<double>(q[2] - q[1]);  // V_{j+1} + Givens
      c->arn_phase_ns[2] += static_cast<double>(q[3] - q[2]);  // barrier
      c->arn_phase_ns[3] += static_cast<double>(q[4] - q[3]);  // iterate
    }
    const double rr = c->hres[0];
    const double hnew = c->hres[1];
    res.residuals.push_back(rr);
    if (rr <= opt.tolerance) {
      res.converged = true;
      break;
    }
    if (hnew < 1e-300) break;
  }
  for (int j = 0; j < maxit && !persistent; ++j) {
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
  if (c->arn_trace) {
    std::fprintf(stderr, "[hd trace] arnoldi phases over %d its (ms): mgs %.3f givens %.3f barrier %.3f iterate %.3f\n",
                 res.iterations, c->arn_phase_ns[0] * 1e-6, c->arn_phase_ns[1] * 1e-6, c->arn_phase_ns[2] * 1e-6,
                 c->arn_phase_ns[3] * 1e-6);
    for (double& v : c->arn_phase_ns) v = 0.0;
  }
  return res;
}

// ---------------------------------------------------------------------------
// layered field (layered.cuh): level groups (Y_g, X_g), g = 0..5
// ---------------------------------------------------------------------------
struct GenHost {
  std::vector<Band> Y, X;
  // wedge: stored 2D stencil K[(iy*n+ix)*(2kb+1)^2 + (dy+kb)*(2kb+1) + dx+kb] (kb < 0: none)
  std::vector<double> K;
  int kb = -1;
};

// Galerkin product (z (x) z)^T K (z (x) z) of a 2D stencil (the reference's
// sparse triple product Z^T M Z, src/precond.cpp:119, in stencil form), on the
// device: one thread per coarse entry (I, J - I), gathering over the children
// of I and J in y and in x.  K and Kc are row-major [point][tap].
__global__ void k_galerkin_stencil(const double* __restrict__ K, int n, int b, const int* __restrict__ cptr,
                                   const int* __restrict__ crow, const double* __restrict__ cw, int nc, int bc,
                                   double* __restrict__ Kc) {
  const int NB = 2 * b + 1, NBc = 2 * bc + 1;
  const size_t tot = (size_t)nc * nc * NBc * NBc;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    const int tap = (int)(e % (NBc * NBc));
    const size_t I = e / (NBc * NBc);
    const int Iy = (int)(I / nc), Ix = (int)(I % nc);
    const int Jy = Iy + tap / NBc - bc, Jx = Ix + tap % NBc - bc;
    double acc = 0.0;
    if (Jy >= 0 && Jy < nc && Jx >= 0 && Jx < nc) {
      for (int pa = cptr[Iy]; pa < cptr[Iy + 1]; ++pa)
        for (int pc = cptr[Jy]; pc < cptr[Jy + 1]; ++pc) {
          const int iy = crow[pa], jy = crow[pc], dy = jy - iy;
          if (dy < -b || dy > b) continue;
          const double wy = cw[pa] * cw[pc];
          double sx = 0.0;
          for (int pb = cptr[Ix]; pb < cptr[Ix + 1]; ++pb)
            for (int pd = cptr[Jx]; pd < cptr[Jx + 1]; ++pd) {
              const int ix = crow[pb], jx = crow[pd], dx = jx - ix;
              if (dx < -b || dx > b) continue;
              sx += cw[pb] * cw[pd] * K[((size_t)iy * n + ix) * NB * NB + (dy + b) * NB + (dx + b)];
            }
          acc += wy * sx;
        }
    }
    Kc[e] = acc;
  }
}

static void galerkin_stencil2d(const std::vector<double>& K, int n, int b, const Transfer& z, std::vector<double>& Kc,
                               int& bc) {
  const int nc = z.coarse;
  std::vector<std::vector<std::pair<int, double>>> par(n), ch(nc);
  for (size_t t = 0; t < z.w.size(); ++t) {
    par[z.row[t]].push_back({z.col[t], z.w[t]});
    ch[z.col[t]].push_back({z.row[t], z.w[t]});
  }
  bc = 0;
  for (int i = 0; i < n; ++i)
    for (int d = -b; d <= b; ++d) {
      const int j = i + d;
      if (j < 0 || j >= n) continue;
      for (const auto& I : par[i])
        for (const auto& J : par[j]) bc = std::max(bc, std::abs(J.first - I.first));
    }
  // children of every coarse index (CSR), fine row order as in z
  std::vector<int> cptr(nc + 1, 0), crow;
  std::vector<double> cw;
  for (int c = 0; c < nc; ++c) {
    for (const auto& f : ch[c]) {
      crow.push_back(f.first);
      cw.push_back(f.second);
    }
    cptr[c + 1] = static_cast<int>(crow.size());
  }
  const int NBc = 2 * bc + 1;
  const size_t outn = static_cast<size_t>(nc) * nc * NBc * NBc;
  double* dK = dalloc<double>(K.size());
  double* dKc = dalloc<double>(outn);
  int* dptr = dalloc<int>(cptr.size());
  int* drow = dalloc<int>(std::max<size_t>(crow.size(), 1));
  double* dw = dalloc<double>(std::max<size_t>(cw.size(), 1));
  CK(cudaMemcpy(dK, K.data(), K.size() * sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dptr, cptr.data(), cptr.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drow, crow.data(), crow.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dw, cw.data(), cw.size() * sizeof(double), cudaMemcpyHostToDevice));
  k_galerkin_stencil<<<grid_for(outn, 256, 148 * 16), 256>>>(dK, n, b, dptr, drow, dw, nc, bc, dKc);
  CK(cudaGetLastError());
  Kc.resize(outn);
  CK(cudaMemcpy(Kc.data(), dKc, outn * sizeof(double), cudaMemcpyDeviceToHost));
  cudaFree(dK);
  cudaFree(dKc);
  cudaFree(dptr);
  cudaFree(drow);
  cudaFree(dw);
}

// wedge fine level: (M, S), (S, M) and the stored K2 stencil
static GenHost wedge_fine(const Band& S1, const Band& M1, const double* K2, int p) {
  GenHost h;
  h.Y = {M1, S1};
  h.X = {S1, M1};
  const size_t n = static_cast<size_t>(M1.n);
  h.K.assign(K2, K2 + n * n * (2 * p + 1) * (2 * p + 1));
  h.kb = p;
  return h;
}

// fine level: (M, S), (S, M), (B_by, W_by = sum_bx m_{by,bx}^2 B_bx), by = 0..3
// (K2 of src/assembly.cpp:234-246 grouped by its y factor)
static GenHost layered_fine(const Band& S1, const Band& M1, const double* interval_mass, const double* mult) {
  GenHost h;
  h.Y = {M1, S1};
  h.X = {S1, M1};
  std::vector<Band> Bb;
  for (int b = 0; b < 4; ++b)
    Bb.push_back(band_from_host(interval_mass + static_cast<size_t>(b) * M1.a.size(), M1.n, M1.b));
  for (int by = 0; by < 4; ++by) {
    Band W(M1.n, M1.b);
    for (int bx = 0; bx < 4; ++bx) {
      const double m2 = mult[4 * by + bx] * mult[4 * by + bx];
      for (size_t e = 0; e < W.a.size(); ++e) W.a[e] += m2 * Bb[bx].a[e];
    }
    h.Y.push_back(Bb[by]);
    h.X.push_back(W);
  }
  return h;
}

static GenHost galerkin_gen(const GenHost& h, const Transfer& z) {
  GenHost o;
  for (const Band& y : h.Y) o.Y.push_back(galerkin(y, z));
  for (const Band& x : h.X) o.X.push_back(galerkin(x, z));
  if (h.kb >= 0) galerkin_stencil2d(h.K, h.Y[0].n, h.kb, z, o.K, o.kb);
  return o;
}

// diagonal entry (iy, ix) of a level operator with group coefficients 1 (g < 2), cl (g >= 2) and kc = cl
static std::complex<double> gen_diag_host(const GenHost& h, int iy, int ix, std::complex<double> cl) {
  std::complex<double> d(0.0, 0.0);
  for (size_t g = 0; g < h.Y.size(); ++g)
    d += (g < 2 ? std::complex<double>(1.0, 0.0) : cl) * (h.Y[g].at(iy, iy) * h.X[g].at(ix, ix));
  if (h.kb >= 0) {
    const int n = h.Y[0].n, NB = 2 * h.kb + 1;
    d += cl * h.K[(static_cast<size_t>(iy) * n + ix) * NB * NB + h.kb * NB + h.kb];
  }
  return d;
}

static Band padded(const Band& B, int b) {
  Band o(B.n, b);
  for (int i = 0; i < B.n; ++i)
    for (int j = std::max(0, i - B.b); j <= std::min(B.n - 1, i + B.b); ++j) o.ref(i, j) = B.at(i, j);
  return o;
}

// Upload the groups; layered coefficient cl of groups 2..5 (groups 0, 1: 1).
static GenLevel upload_gen(const GenHost& h, double2 cl, double** mem) {
  const int G = static_cast<int>(h.Y.size());
  int b = std::max(h.kb, 0);
  for (int g = 0; g < G; ++g) b = std::max({b, h.Y[g].b, h.X[g].b});
  const int n = h.Y[0].n;
  const size_t per = static_cast<size_t>(n) * (2 * b + 1);
  const int NB = 2 * b + 1;
  const size_t NN = static_cast<size_t>(n) * n, kplanes = h.kb >= 0 ? static_cast<size_t>(NB) * NB * NN : 0;
  *mem = dalloc<double>(2 * G * per + kplanes);
  GenLevel L{};
  L.n = n;
  L.b = b;
  L.G = G;
  for (int g = 0; g < G; ++g) {
    const Band y = padded(h.Y[g], b), x = padded(h.X[g], b);
    double* dy = *mem + (2 * g) * per;
    double* dx = *mem + (2 * g + 1) * per;
    CK(cudaMemcpy(dy, y.a.data(), per * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dx, x.a.data(), per * sizeof(double), cudaMemcpyHostToDevice));
    L.Y[g] = dy;
    L.X[g] = dx;
    L.coef[g] = g < 2 ? cmk(1.0, 0.0) : cl;
  }
  L.K = nullptr;
  L.kc = cl;
  if (h.kb >= 0) {
    // tap-planar, padded to the level band b
    const int kNB = 2 * h.kb + 1;
    std::vector<double> planes(kplanes, 0.0);
    for (size_t i = 0; i < NN; ++i)
      for (int dy = -h.kb; dy <= h.kb; ++dy)
        for (int dx = -h.kb; dx <= h.kb; ++dx)
          planes[static_cast<size_t>((dy + b) * NB + dx + b) * NN + i] = h.K[i * kNB * kNB + (dy + h.kb) * kNB + dx + h.kb];
    double* dk = *mem + 2 * G * per;
    CK(cudaMemcpy(dk, planes.data(), kplanes * sizeof(double), cudaMemcpyHostToDevice));
    L.K = dk;
  }
  return L;
}

// attach the layered groups to a level: unshifted (-k^2) and shifted (-k^2 (1 - i beta2))
static void attach_gen(DevBand& d, const GenHost& h, double2 cA, double2 cM) {
  double* mem = nullptr;
  GenLevel a = upload_gen(h, cmk(-cA.x, -cA.y), &mem);
  GenLevel m = a;
  for (int g = 2; g < m.G; ++g) m.coef[g] = cmk(-cM.x, -cM.y);
  m.kc = cmk(-cM.x, -cM.y);
  d.gen_mem = mem;
  d.genA = new GenLevel(a);
  d.genM = new GenLevel(m);
}

// Dense inverse of a layered level operator (coefficient cl on groups 2..5):
// E = Z^T A Z and the coarsest shifted level of the layered hierarchy stand in
// for the reference's SparseLU factors (src/precond.cpp:95-99, 133).
static ExactSolver make_btri(cudaStream_t st, const GenHost& h, double2 cl, int n_sms);

static ExactSolver make_dense(cudaStream_t st, const GenHost& h, double2 cl, int n_sms = 148, bool allow_btri = true) {
  const int n = h.Y[0].n;
  const size_t NN = static_cast<size_t>(n) * n;
  // operators beyond the dense-inverse limit, or HD_BTRI=1: block tridiagonal LU
  const char* fb = std::getenv("HD_BTRI");
  if (allow_btri && (NN > 20000 || (fb && std::atoi(fb) == 1)) && !(fb && std::atoi(fb) == 0))
    return make_btri(st, h, cl, n_sms);
  if (NN > 20000)
    throw Error(HD_ERR_INVALID, "non-separable field: exact solve of " + std::to_string(NN) +
                                    " complex unknowns exceeds the dense-inverse limit (20000)");
  ExactSolver X;
  X.dim = 2;
  X.n = n;
  X.dense = true;
  X.NN = NN;
  double* mem = nullptr;
  const GenLevel L = upload_gen(h, cl, &mem);
  double2* A = dalloc<double2>(NN * NN);
  X.Ainv = dalloc<double2>(NN * NN);
  X.dx = dalloc<double2>(NN);
  X.dy = dalloc<double2>(NN);
  k_dense_kron<<<grid_for(NN * NN, 256, 148 * 32), 256, 0, st>>>(L, A);
  CK(cudaGetLastError());
  k_identity<<<grid_for(NN * NN, 256, 148 * 32), 256, 0, st>>>(X.Ainv, NN);
  CK(cudaGetLastError());
  cusolverDnHandle_t hs;
  CKS(cusolverDnCreate(&hs));
  CKS(cusolverDnSetStream(hs, st));
  const int m = static_cast<int>(NN);
  int lwork = 0;
  auto* Az = reinterpret_cast<cuDoubleComplex*>(A);
  CKS(cusolverDnZgetrf_bufferSize(hs, m, m, Az, m, &lwork));
  cuDoubleComplex* work = dalloc<cuDoubleComplex>(std::max(lwork, 1));
  int* ipiv = dalloc<int>(NN);
  int* info = dalloc<int>(2);
  CKS(cusolverDnZgetrf(hs, m, m, Az, m, work, ipiv, info));
  CKS(cusolverDnZgetrs(hs, CUBLAS_OP_N, m, m, Az, m, ipiv, reinterpret_cast<cuDoubleComplex*>(X.Ainv), m, info + 1));
  int hinfo[2] = {0, 0};
  CK(cudaMemcpyAsync(hinfo, info, sizeof(hinfo), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cusolverDnDestroy(hs);
  cudaFree(A);
  cudaFree(work);
  cudaFree(ipiv);
  cudaFree(info);
  cudaFree(mem);
  if (hinfo[0] != 0 || hinfo[1] != 0)
    throw Error(HD_ERR_FACTOR, "layered exact solve: singular operator (getrf info " + std::to_string(hinfo[0]) + ")");
  return X;
}

// Block tridiagonal LU of a level operator (btri.cuh): q = b grid rows per
// block; real (T = double) when every coefficient is real, else complex.
template <class T>
struct BtriLib;
template <>
struct BtriLib<double> {
  static cublasStatus_t gemm(cublasHandle_t h, cublasOperation_t ta, cublasOperation_t tb, int m, const double* al,
                             const double* A, const double* B, const double* be, double* C) {
    return cublasDgemm(h, ta, tb, m, m, m, al, A, m, B, m, be, C, m);
  }
  static cusolverStatus_t getrf_ws(cusolverDnHandle_t h, int m, double* A, int* lw) {
    return cusolverDnDgetrf_bufferSize(h, m, m, A, m, lw);
  }
  static cusolverStatus_t getrf(cusolverDnHandle_t h, int m, double* A, double* w, int* piv, int* info) {
    return cusolverDnDgetrf(h, m, m, A, m, w, piv, info);
  }
  static cusolverStatus_t getrs_t(cusolverDnHandle_t h, int m, const double* A, const int* piv, double* B, int* info) {
    return cusolverDnDgetrs(h, CUBLAS_OP_T, m, m, A, m, piv, B, m, info);
  }
  static double one() { return 1.0; }
  static double mone() { return -1.0; }
  static double zero() { return 0.0; }
};
template <>
struct BtriLib<double2> {
  using Z = cuDoubleComplex;
  static cublasStatus_t gemm(cublasHandle_t h, cublasOperation_t ta, cublasOperation_t tb, int m, const double2* al,
                             const double2* A, const double2* B, const double2* be, double2* C) {
    return cublasZgemm(h, ta, tb, m, m, m, reinterpret_cast<const Z*>(al), reinterpret_cast<const Z*>(A), m,
                       reinterpret_cast<const Z*>(B), m, reinterpret_cast<const Z*>(be), reinterpret_cast<Z*>(C), m);
  }
  static cusolverStatus_t getrf_ws(cusolverDnHandle_t h, int m, double2* A, int* lw) {
    return cusolverDnZgetrf_bufferSize(h, m, m, reinterpret_cast<Z*>(A), m, lw);
  }
  static cusolverStatus_t getrf(cusolverDnHandle_t h, int m, double2* A, double2* w, int* piv, int* info) {
    return cusolverDnZgetrf(h, m, m, reinterpret_cast<Z*>(A), m, reinterpret_cast<Z*>(w), piv, info);
  }
  static cusolverStatus_t getrs_t(cusolverDnHandle_t h, int m, const double2* A, const int* piv, double2* B, int* info) {
    // plain transpose (not conjugate): the stored factors are the row-major blocks
    return cusolverDnZgetrs(h, CUBLAS_OP_T, m, m, reinterpret_cast<const Z*>(A), m, piv, reinterpret_cast<Z*>(B), m, info);
  }
  static double2 one() { return cmk(1.0, 0.0); }
  static double2 mone() { return cmk(-1.0, 0.0); }
  static double2 zero() { return cmk(0.0, 0.0); }
};

template <class T>
static void btri_factor(cudaStream_t st, const GenLevel& L, int q, int m, int nb, ExactSolver& X) {
  using Lb = BtriLib<T>;
  const size_t mm = static_cast<size_t>(m) * m, tot = static_cast<size_t>(nb) * mm;
  const int k = nb / 2;  // the twist: top half eliminated downwards, bottom half upwards
  T *D = dalloc<T>(tot), *Bu = dalloc<T>(tot), *Cl = dalloc<T>(tot);
  T *GT = dalloc<T>(tot), *SinvT = dalloc<T>(tot), *HT = dalloc<T>(tot), *G2 = dalloc<T>(mm);
  CK(cudaMemsetAsync(GT, 0, tot * sizeof(T), st));
  CK(cudaMemsetAsync(HT, 0, tot * sizeof(T), st));
  CK(cudaMemsetAsync(G2, 0, mm * sizeof(T), st));
  k_btri_blocks<T><<<grid_for(tot, 256, 148 * 32), 256, 0, st>>>(L, q, m, nb, D, Bu, Cl);
  CK(cudaGetLastError());
  cublasHandle_t cb;
  CKB(cublasCreate(&cb));
  CKB(cublasSetStream(cb, st));
  cusolverDnHandle_t hs;
  CKS(cusolverDnCreate(&hs));
  CKS(cusolverDnSetStream(hs, st));
  int lwork = 0;
  CKS(Lb::getrf_ws(hs, m, D, &lwork));
  T* work = dalloc<T>(std::max(lwork, 1));
  int* ipiv = dalloc<int>(m);
  int* info = dalloc<int>(2 * nb);
  CK(cudaMemsetAsync(info, 0, 2 * nb * sizeof(int), st));
  std::vector<T> eye(mm);
  for (size_t e = 0; e < mm; ++e) eye[e] = (e % (m + 1) == 0) ? Lb::one() : Lb::zero();
  const T one = Lb::one(), mone = Lb::mone(), zero = Lb::zero();
  // Schur block S (in place of D_i) -> its inverse transposed in SinvT[i] (= row-major inverse)
  auto invert = [&](int i) {
    T* S = D + i * mm;
    CKS(Lb::getrf(hs, m, S, work, ipiv, info + 2 * i));
    T* Si = SinvT + i * mm;
    CK(cudaMemcpyAsync(Si, eye.data(), mm * sizeof(T), cudaMemcpyHostToDevice, st));
    CKS(Lb::getrs_t(hs, m, S, ipiv, Si, info + 2 * i + 1));  // S^T X = I
  };
  // top: i = 0 .. k-1  (S_i = D_i - G_i B_{i-1}; G_{i+1}^T = S_i^-T C_{i+1}^T; H_i^T = B_i^T S_i^-T)
  for (int i = 0; i < k; ++i) {
    if (i > 0) CKB(Lb::gemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, m, &mone, GT + i * mm, Bu + (i - 1) * mm, &one, D + i * mm));
    invert(i);
    CKB(Lb::gemm(cb, CUBLAS_OP_N, CUBLAS_OP_T, m, &one, SinvT + i * mm, Cl + (i + 1) * mm, &zero, GT + (i + 1) * mm));
    CKB(Lb::gemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, m, &one, Bu + i * mm, SinvT + i * mm, &zero, HT + i * mm));
  }
  // bottom: i = nb-1 .. k+1  (T_i = D_i - G'_i C_{i+1}; G'_{i-1}^T = T_i^-T B_{i-1}^T; H'_i^T = C_i^T T_i^-T)
  for (int i = nb - 1; i > k; --i) {
    if (i < nb - 1) CKB(Lb::gemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, m, &mone, GT + i * mm, Cl + (i + 1) * mm, &one, D + i * mm));
    invert(i);
    T* gdst = (i - 1 == k) ? G2 : GT + (i - 1) * mm;
    CKB(Lb::gemm(cb, CUBLAS_OP_N, CUBLAS_OP_T, m, &one, SinvT + i * mm, Bu + (i - 1) * mm, &zero, gdst));
    CKB(Lb::gemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, m, &one, Cl + i * mm, SinvT + i * mm, &zero, HT + i * mm));
  }
  // middle: M = D_k - G_k B_{k-1} - G'_k C_{k+1}
  if (k > 0) CKB(Lb::gemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, m, &mone, GT + k * mm, Bu + (k - 1) * mm, &one, D + k * mm));
  if (k < nb - 1) CKB(Lb::gemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, m, &mone, G2, Cl + (k + 1) * mm, &one, D + k * mm));
  invert(k);
  std::vector<int> hinfo(2 * nb);
  CK(cudaMemcpyAsync(hinfo.data(), info, hinfo.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  cublasDestroy(cb);
  cusolverDnDestroy(hs);
  cudaFree(D); cudaFree(Bu); cudaFree(Cl); cudaFree(work); cudaFree(ipiv); cudaFree(info);
  for (int v : hinfo)
    if (v != 0) {
      cudaFree(GT); cudaFree(SinvT); cudaFree(HT); cudaFree(G2);
      throw Error(HD_ERR_FACTOR, "block tridiagonal exact solve: singular block (info " + std::to_string(v) + ")");
    }
  X.bt.GT = GT;
  X.bt.G2 = G2;
  X.bt.SinvT = SinvT;
  X.bt.HT = HT;
  X.bt.k = k;
}

static ExactSolver make_btri(cudaStream_t st, const GenHost& h, double2 cl, int n_sms) {
  const int n = h.Y[0].n;
  double* mem = nullptr;
  const GenLevel L = upload_gen(h, cl, &mem);
  bool cplx = L.K && L.kc.y != 0.0;
  for (int g = 0; g < L.G; ++g) cplx = cplx || L.coef[g].y != 0.0;
  const int q = std::max(L.b, 1), m = q * n, nb = (n + q - 1) / q;
  const int kr_need = (m + 31) / 32;
  int kr = 0;
  for (int cand : {8, 16, 24, 32, 48, 64, 96})
    if (cand >= kr_need && (!cplx || cand <= 48)) {
      kr = cand;
      break;
    }
  if (kr == 0)
    throw Error(HD_ERR_INVALID, "block tridiagonal solve: block size " + std::to_string(m) + " above the kernel limit");
  ExactSolver X;
  X.dim = 2;
  X.n = n;
  X.btri = true;
  X.bt_cplx = cplx;
  X.bt_kr = kr;
  try {
    if (cplx) btri_factor<double2>(st, L, q, m, nb, X);
    else btri_factor<double>(st, L, q, m, nb, X);
  } catch (...) {
    cudaFree(mem);
    throw;
  }
  cudaFree(mem);
  X.bt.n = n;
  X.bt.q = q;
  X.bt.m = m;
  X.bt.nb = nb;
  X.bt.NN = static_cast<size_t>(n) * n;
  // y, w, x: one allocation
  X.bt.y = dalloc<double>(6 * static_cast<size_t>(nb) * m);
  X.bt.w = X.bt.y + 2 * static_cast<size_t>(nb) * m;
  X.bt.x = X.bt.w + 2 * static_cast<size_t>(nb) * m;
  X.bt.bar = dalloc<unsigned>(1);
  (void)n_sms;
  return X;
}

static void destroy_slabs(hd_ctx* c);

static void destroy_ctx(hd_ctx* c) {
  if (!c) return;
  if (c->slabs) destroy_slabs(c);
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->st);
  auto fb = [](DevBand& d) {
    cudaFree(d.S);
    cudaFree(d.M);
    cudaFree(d.gen_mem);
    delete d.genA;
    delete d.genM;
  };
  fb(c->fine);
  for (size_t l = 1; l < c->lev.size(); ++l) fb(c->lev[l]);
  free_exact(c->coarsest);
  free_exact(c->shift_exact);
  cudaFree(c->sx_plan);
  free_exact(c->E);
  for (auto* p : c->mg_b) cudaFree(p);
  for (auto* p : c->mg_x) cudaFree(p);
  for (auto* p : c->mg_y) cudaFree(p);
  for (auto* p : c->mg_r) cudaFree(p);
  cudaFree(c->ep); cudaFree(c->ep2);
  cudaFree(c->f); cudaFree(c->rhsp); cudaFree(c->x0); cudaFree(c->x); cudaFree(c->w);
  cudaFree(c->t1); cudaFree(c->t2); cudaFree(c->t3); cudaFree(c->V);
  cudaFree(c->H); cudaFree(c->g); cudaFree(c->cs); cudaFree(c->sn); cudaFree(c->y);
  cudaFree(c->scal); cudaFree(c->dres); cudaFree(c->partials); cudaFree(c->counter);
  cudaFree(c->dj); cudaFree(c->arn_partials); cudaFree(c->arn_bar);
  cudaFree(c->lsa_sig); cudaFree(c->lsa_L); cudaFree(c->lsa_ch); cudaFree(c->lsa_cx); cudaFree(c->lsa_partials);
  cudaFree(c->lsa_counter);
  if (c->loop_exec) cudaGraphExecDestroy(c->loop_exec);
  if (c->loop_graph) cudaGraphDestroy(c->loop_graph);
  cudaFree(c->loop_state); cudaFree(c->res_hist); cudaFree(c->cublas_ws);
  if (c->loop_host) cudaFreeHost(c->loop_host);
  if (c->res_host) cudaFreeHost(c->res_host);
  if (c->arn_trace) cudaFreeHost(c->arn_trace);
  if (c->hres) cudaFreeHost(c->hres);
  if (c->cb) cublasDestroy(c->cb);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  for (auto e : c->prof_ev) cudaEventDestroy(e);
  cudaStream_t mine = c->own_st ? c->own_st : c->st;
  if (mine) cudaStreamDestroy(mine);
  if (c->st2) cudaStreamDestroy(c->st2);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  delete c;
}

static void create_ctx(const hd_system* sys, const hd_precond* spec, const int* devices, int n_devices, hd_ctx** out) {
  if (!sys || !spec || !out) throw Error(HD_ERR_INVALID, "null argument");
  if (n_devices > 1) throw Error(HD_ERR_INVALID, "multi-device row slabs are not available in this build");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error(HD_ERR_NO_DEVICE, "no CUDA device: the helmdef_b200 path has no CPU fallback");
  if (sys->dim != 1 && sys->dim != 2) throw Error(HD_ERR_INVALID, "dim must be 1 or 2");
  const bool layered = sys->field_kind == HD_FIELD_LAYERED;
  const bool wedge = sys->field_kind == HD_FIELD_WEDGE;
  const bool gen = layered || wedge;  // non-Kronecker-sum fields (layered.cuh)
  if (sys->field_kind != HD_FIELD_CONSTANT && !gen) throw Error(HD_ERR_INVALID, "unknown wave-number field kind");
  if (gen && sys->dim != 2) throw Error(HD_ERR_INVALID, "the layered and wedge fields are two-dimensional");
  if (layered && !sys->interval_mass) throw Error(HD_ERR_INVALID, "layered field needs the interval masses");
  if (wedge && !sys->shift_mass_2d) throw Error(HD_ERR_INVALID, "wedge field needs shift_mass_2d (hd_assemble_field)");
  if (sys->per_dim < 2) throw Error(HD_ERR_INVALID, "per_dim must be >= 2");
  const auto t0 = std::chrono::steady_clock::now();
  // HD_SETUP_TRACE=1: wall time of the setup phases on stderr
  const bool trace = std::getenv("HD_SETUP_TRACE") && std::atoi(std::getenv("HD_SETUP_TRACE")) == 1;
  auto tlast = t0;
  auto mark = [&](const char* what) {
    if (!trace) return;
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hd setup] %-28s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - tlast).count());
    tlast = now;
  };
  std::unique_ptr<hd_ctx, void (*)(hd_ctx*)> c(new hd_ctx(), destroy_ctx);
  c->device = (devices && n_devices == 1) ? devices[0] : 0;
  if (!devices || n_devices == 0) CK(cudaGetDevice(&c->device));
  CK(cudaSetDevice(c->device));
  CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
  CKB(cublasCreate(&c->cb));
  CKB(cublasSetStream(c->cb, c->st));
  CKB(cublasSetMathMode(c->cb, CUBLAS_DEFAULT_MATH));
  CK(cudaEventCreate(&c->ev0));
  CK(cudaEventCreate(&c->ev1));
  c->dim = sys->dim;
  c->p = sys->order;
  c->n = sys->per_dim;
  c->N = c->dim == 2 ? static_cast<size_t>(c->n) * c->n : c->n;
  c->k = sys->k;
  c->spec = *spec;
  if (c->spec.coarsest <= 0) c->spec.coarsest = 32;
  c->corner = c->dim == 1 ? cmk(sys->corner_re, sys->corner_im) : cmk(0.0, 0.0);
  // wedge: K2 carries k(x,y)^2 itself, so its coefficients are 1 and 1 - i beta2
  const double k2 = wedge ? 1.0 : c->k * c->k;
  c->cA = cmk(k2, 0.0);
  // shifted operator A + i beta2 K2 = ... - k^2 (1 - i beta2) M(x)M  (src/precond.cpp:165-167)
  c->cM = cmk(k2, -k2 * c->spec.beta2);
  const Band S1 = band_from_host(sys->stiffness_band, c->n, sys->order);
  const Band M1 = band_from_host(sys->mass_band, c->n, sys->order);
  mark("context, streams, handles");
  c->fine = upload_pair(S1, M1);
  GenHost fineH;
  if (gen) {
    fineH = layered ? layered_fine(S1, M1, sys->interval_mass, sys->multipliers)
                    : wedge_fine(S1, M1, sys->shift_mass_2d, sys->order);
    attach_gen(c->fine, fineH, c->cA, c->cM);
  }
  // C_ex: exact shifted inverse (src/precond.cpp:204-211)
  if (c->spec.shift && c->spec.cycles <= 0) {
    if (gen) {
      // non-separable field: dense inverse (small) or complex block tridiagonal LU of the shifted operator
      int nsm = 148;
      CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
      c->shift_exact = make_dense(c->st, fineH, cmk(-c->cM.x, -c->cM.y), nsm);
      c->sx_plan = dalloc<double>(2 * c->N);
    } else if (c->dim == 2) {
      c->shift_exact = make_fd(c->st, S1, M1, c->cM);
      c->sx_plan = dalloc<double>(2 * c->N);
    } else {
      c->shift_exact = make_bandlu(S1, M1, c->cM, c->corner);
    }
  }
  mark("fine level (+ C_ex)");
  // multigrid hierarchy of the shifted operator (src/precond.cpp:110-134)
  if (c->spec.shift && c->spec.cycles > 0) {
    std::vector<Band> Ss{S1}, Ms{M1};
    std::vector<GenHost> Hs{fineH};
    int nl = c->n;
    while (nl > c->spec.coarsest) {
      const Transfer z = linear_stencil(nl);
      Ss.push_back(galerkin(Ss.back(), z));
      Ms.push_back(galerkin(Ms.back(), z));
      if (gen) Hs.push_back(galerkin_gen(Hs.back(), z));
      nl = z.coarse;
    }
    c->lev.push_back(c->fine);
    for (size_t l = 1; l < Ss.size(); ++l) {
      c->lev.push_back(upload_pair(Ss[l], Ms[l]));
      if (gen) attach_gen(c->lev.back(), Hs[l], c->cA, c->cM);
    }
    if (gen)  // zero-diagonal check of the layered / wedge levels (src/precond.cpp:125-132)
      for (size_t l = 0; l < Hs.size(); ++l) {
        const GenHost& h = Hs[l];
        const int nn = h.Y[0].n;
        for (int i = 0; i < nn; ++i)
          for (int j = 0; j < nn; ++j)
            if (gen_diag_host(h, i, j, -std::complex<double>(c->cM.x, c->cM.y)) == std::complex<double>(0.0, 0.0))
              throw Error(HD_ERR_FACTOR, "zero diagonal in smoother");
      }
    // zero-diagonal check of every level (src/precond.cpp:125-132)
    for (size_t l = 0; !gen && l < Ss.size(); ++l)
      for (int i = 0; i < Ss[l].n; ++i)
        for (int j = 0; j < (c->dim == 2 ? Ss[l].n : 1); ++j) {
          const int jj = c->dim == 2 ? j : i;
          std::complex<double> d = c->dim == 2
                                       ? std::complex<double>(Ms[l].at(i, i) * Ss[l].at(jj, jj) + Ss[l].at(i, i) * Ms[l].at(jj, jj), 0.0) -
                                             std::complex<double>(c->cM.x, c->cM.y) * (Ms[l].at(i, i) * Ms[l].at(jj, jj))
                                       : std::complex<double>(Ss[l].at(i, i), 0.0) - std::complex<double>(c->cM.x, c->cM.y) * Ms[l].at(i, i);
          if (l == 0 && c->dim == 1 && i == c->n - 1) d += std::complex<double>(c->corner.x, c->corner.y);
          if (d == std::complex<double>(0.0, 0.0)) throw Error(HD_ERR_FACTOR, "zero diagonal in smoother");
        }
    const Band& SL = Ss.back();
    const Band& ML = Ms.back();
    if (gen) c->coarsest = make_dense(c->st, Hs.back(), cmk(-c->cM.x, -c->cM.y), 148, false);  // <= 32^2 unknowns
    else if (c->dim == 2) c->coarsest = make_fd(c->st, SL, ML, c->cM);
    else c->coarsest = make_bandlu(SL, ML, c->cM, Ss.size() == 1 ? c->corner : cmk(0.0, 0.0));
    for (size_t l = 0; l < c->lev.size(); ++l) {
      const size_t NL = lsize(c.get(), c->lev[l].n);
      c->mg_b.push_back(l == 0 ? nullptr : dalloc<double2>(NL));
      c->mg_x.push_back(dalloc<double2>(NL));
      c->mg_y.push_back(dalloc<double2>(NL));
      c->mg_r.push_back(dalloc<double2>(NL));
    }
  }
  mark("multigrid hierarchy");
  // deflation: E = Z^T A Z with the Bezier stencil (src/precond.cpp:93-100, 228-232)
  if (c->spec.deflate) {
    const Transfer z = halving_stencil(c->n, c->spec.drop);
    c->nc = z.coarse;
    if (c->nc < 1) throw Error(HD_ERR_INVALID, "deflation needs per_dim >= 2");
    const Band ES = galerkin(S1, z), EM = galerkin(M1, z);
    if (gen) {
      int nsm = 148;
      CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
      c->E = make_dense(c->st, galerkin_gen(fineH, z), cmk(-c->cA.x, -c->cA.y), nsm);
    } else if (c->dim == 2) {
      const bool fold = (c->nc % 2 == 0) && centro_symmetric(ES) && centro_symmetric(EM) &&
                        !std::getenv("HD_NOFOLD");
      const char* ey = std::getenv("HD_EYSOLVE");
      // HD_EYSOLVE=1: partial diagonalisation + segmented y sweeps (experimental:
      // equally exact, but its rounding differs from the oracle's FD by more
      // than the C3/C5 history bars allow, and it is not yet faster -- DESIGN.md §4)
      const bool ys = ey && std::atoi(ey) == 1 && c->cA.y == 0.0 && std::max(ES.b, EM.b) <= 6 && c->nc >= 4 * kYL;
      if (fold) c->E = make_fd_folded(c->st, ES, EM, c->cA);
      else if (ys) c->E = make_fd_ypart(c->st, ES, EM, c->cA);
      else c->E = make_fd(c->st, ES, EM, c->cA);
    } else {
      // corner term of A restricted: Z^T (corner e_n e_n^T) Z
      double2 corner_c = cmk(0.0, 0.0);
      if (c->corner.x != 0.0 || c->corner.y != 0.0) {
        // the last fine row maps onto the last coarse column(s); E's (nc-1, nc-1) gets w^2 * corner
        double wl = 0.0;
        for (size_t t = 0; t < z.w.size(); ++t)
          if (z.row[t] == c->n - 1 && z.col[t] == c->nc - 1) wl = z.w[t];
        if (wl != 0.0) corner_c = cmk(c->corner.x * wl * wl, c->corner.y * wl * wl);
      }
      c->E = make_bandlu(ES, EM, c->cA, corner_c);
    }
    const size_t NC = lsize(c.get(), c->nc);
    c->ep = dalloc<double>(2 * NC);
    c->ep2 = dalloc<double>(2 * NC);
  }
  mark("deflation E and its solver");
  const size_t N = c->N;
  c->f = dalloc<double2>(N);
  c->rhsp = dalloc<double2>(N);
  c->x0 = dalloc<double2>(N);
  c->x = dalloc<double2>(N);
  c->w = dalloc<double2>(N);
  c->t1 = dalloc<double2>(N);
  c->t2 = dalloc<double2>(N);
  c->t3 = dalloc<double2>(N);
  c->scal = dalloc<double2>(8);
  c->dres = dalloc<double>(8);
  CK(cudaMallocHost(&c->hres, 8 * sizeof(double)));
  c->red_blocks = 148 * 4;
  const int max_stencil_blocks = 148 * 64;
  c->partials = dalloc<double2>(std::max(c->red_blocks, max_stencil_blocks) + 16);
  c->counter = dalloc<unsigned>(4);
  CK(cudaMemset(c->counter, 0, 4 * sizeof(unsigned)));
  CK(cudaStreamSynchronize(c->st));
  CK(cudaDeviceSynchronize());
  if (const char* e = std::getenv("HD_ARNOLDI")) c->arn_mode = std::atoi(e);
  if (const char* e = std::getenv("HD_GRAPH")) c->graph_enabled = std::atoi(e) != 0;
  CK(cudaDeviceGetAttribute(&c->n_sms, cudaDevAttrMultiProcessorCount, c->device));
  c->cublas_ws = dalloc<char>(32u << 20);
  CKB(cublasSetWorkspace(c->cb, c->cublas_ws, 32u << 20));
  mark("vectors, workspaces");
  c->t_setup = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *out = c.release();
}

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
  CK(cudaMemcpyAsync(c->hres + 1, c->dres + 1, sizeof(double), cudaMemcpyDeviceToHost, c->st));
}

// Capture one iteration (parts a and b with the monitor of x_{j-1} between
// them, the scalars copied to the pinned mirror at the end) as a graph; the
// counters it adds per launch are recorded.  NCCL calls are captured too.
static void build_slab_body(hd_ctx* c, int maxit, int nparts) {
  hd_slabs* sl = slabs_of(c);
  if (!sl->dj) {
    sl->dj = dalloc<int>(1);
    CK(cudaMallocHost(&sl->hj, sizeof(int)));
  }
  if (sl->body) {
    cudaGraphExecDestroy(sl->body);
    sl->body = nullptr;
  }
  const long before[6] = {c->matvecs, c->coarse_solves, c->shift_solves, c->vcycles, c->launches, c->lib_calls};
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(c->st, cudaStreamCaptureModeRelaxed));
  slab_iteration_a(c, 0, maxit, sl->dj);
  s_monitor(c, sl->x);  // x_{j-1} (used by the host for j >= 1)
  slab_iteration_b(c, 0, maxit, nparts, sl->dj);
  CK(cudaMemcpyAsync(c->hres, c->dres, 4 * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamEndCapture(c->st, &g));
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
}

static SolveOut run_solve_slabs(hd_ctx* c, const hd_gmres& opt, const double2* f_full, double2* xout_full) {
  hd_slabs* sl = slabs_of(c);
  const int maxit = std::max(opt.max_iterations, 1);
  if (maxit + 1 > kLsaMaxJ) throw Error(HD_ERR_INVALID, "row slabs: max_iterations above the Arnoldi limit");
  ensure_gmres(c, maxit);
  const SlabLevel& G = sl->lv[0];
  if (sl->maxit < maxit) {
    for (auto* p : sl->V) cudaFree(p);
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
  bool stop = false;
  double hnew_prev = 1.0;
  const bool graph = c->graph_enabled && !c->prof_on;
  if (graph && sl->body_maxit != maxit) build_slab_body(c, maxit, nparts);
  for (int j = 0; j < maxit && !stop; ++j) {
    const long snap[4] = {c->matvecs, c->coarse_solves, c->shift_solves, c->vcycles};
    auto rollback = [&]() {
      c->matvecs = snap[0];
      c->coarse_solves = snap[1];
      c->shift_solves = snap[2];
      c->vcycles = snap[3];
    };
    if (graph) {
      // the whole iteration (pass 1, pass 2, monitor of x_{j-1}, Givens) as one graph launch
      *sl->hj = j;
      CK(cudaMemcpyAsync(sl->dj, sl->hj, sizeof(int), cudaMemcpyHostToDevice, c->st));
      CK(cudaGraphLaunch(sl->body, c->st));
      CK(cudaStreamSynchronize(c->st));
      c->matvecs += sl->body_delta[0];
      c->coarse_solves += sl->body_delta[1];
      c->shift_solves += sl->body_delta[2];
      c->vcycles += sl->body_delta[3];
      c->launches += static_cast<int>(sl->body_delta[4]);
      c->lib_calls += static_cast<int>(sl->body_delta[5]);
      if (j >= 1) {
        const double rr = c->hres[0];
        res.iterations = j;
        res.residuals.push_back(rr);
        if (rr <= opt.tolerance || hnew_prev < 1e-300) {
          res.converged = rr <= opt.tolerance;
          rollback();
          break;
        }
      }
    } else {
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
    }
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
  if (c->fine.genA) throw Error(HD_ERR_INVALID, "row slabs: constant wave-number field only");
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
    sl->dist_e = c->spec.deflate && X.dim == 2 && X.V && !X.folded && !X.ypart && !X.dense && !X.btri &&
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
    for (auto* p : v) cudaFree(p);
  };
  for (auto& v : sl->X) fr(v);
  for (auto& v : sl->Y) fr(v);
  for (auto& v : sl->B) fr(v);
  for (auto& v : sl->R) fr(v);
  for (auto* v : {&sl->f, &sl->w, &sl->t1, &sl->t2, &sl->t3, &sl->x, &sl->x0, &sl->rhsp, &sl->vin, &sl->V}) fr(*v);
  cudaFree(sl->slots);
  cudaFree(sl->parts);
  cudaFree(sl->red);
  if (sl->vranks || sl->nranks > 1)
    for (int s : sl->mine) {
      cudaFree(sl->eT1[s]);
      cudaFree(sl->eT2[s]);
    }
  for (int s : sl->mine) {
    if (!sl->esend.empty()) cudaFree(sl->esend[s]);
    if (!sl->erecv.empty()) cudaFree(sl->erecv[s]);
  }
  if (sl->body) cudaGraphExecDestroy(sl->body);
  cudaFree(sl->dj);
  if (sl->hj) cudaFreeHost(sl->hj);
  if (sl->comm) nccl().CommDestroy(sl->comm);
  delete sl;
  c->slabs = nullptr;
}

}  // namespace hd

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* hd_last_error(void) { return g_last_error.c_str(); }

#define HD_GUARD_BEGIN try {
#define HD_GUARD_END                          \
  }                                           \
  catch (const hd::Error& e) {                \
    g_last_error = e.what();                  \
    return e.code;                            \
  }                                           \
  catch (const std::exception& e) {           \
    g_last_error = e.what();                  \
    return HD_ERR_INVALID;                    \
  }                                           \
  return HD_OK;

int hd_problem_per_dim(const hd_problem* pb) {
  if (!pb) return -1;
  return pb->elements + pb->order - 2;  // both ends (all faces) Dirichlet
}

hd_status hd_assemble(const hd_problem* pb, double* stiffness_band, double* mass_band, double* interval_mass,
                      double* rhs) {
  HD_GUARD_BEGIN
  if (!pb || !stiffness_band || !mass_band || !rhs) throw Error(HD_ERR_INVALID, "null argument");
  if (pb->dim != 1 && pb->dim != 2) throw Error(HD_ERR_INVALID, "dim must be 1 or 2");
  if (pb->order < 1 || pb->order > 6 || pb->elements < 1) throw Error(HD_ERR_INVALID, "bad order/elements");
  const Forms1d f = assemble_forms_1d(pb->elements, pb->order);
  const int nb = f.kv.basis_count();
  std::vector<int> kept;
  for (int j = 1; j < nb - 1; ++j) kept.push_back(j);  // Dirichlet at both ends / all faces
  const int n = static_cast<int>(kept.size());
  const Band S1 = reduce(f.stiffness, kept), M1 = reduce(f.mass, kept);
  std::memcpy(stiffness_band, S1.a.data(), S1.a.size() * sizeof(double));
  std::memcpy(mass_band, M1.a.data(), M1.a.size() * sizeof(double));
  if (interval_mass) {
    for (int b = 0; b < 4; ++b) {
      const Band Bb = reduce(mass_on_interval(f.kv, 0.25 * b, 0.25 * (b + 1)), kept);
      std::memcpy(interval_mass + static_cast<size_t>(b) * Bb.a.size(), Bb.a.data(), Bb.a.size() * sizeof(double));
    }
  }
  // point load phi_i(x_s) phi_j(y_s) (src/assembly.cpp:251-256; (1/2, 1/2) unless set)
  const double xs = pb->point_source ? pb->source[0] : 0.5, ys = pb->point_source ? pb->source[1] : 0.5;
  std::vector<double> phix(n), phiy(n);
  for (int i = 0; i < n; ++i) {
    phix[i] = bspline_value(f.kv, f.kv.degree, kept[i], xs);
    phiy[i] = bspline_value(f.kv, f.kv.degree, kept[i], ys);
  }
  if (pb->dim == 1) {
    for (int i = 0; i < n; ++i) {
      rhs[2 * i] = phix[i];
      rhs[2 * i + 1] = 0.0;
    }
  } else {
    for (int iy = 0; iy < n; ++iy)
      for (int ix = 0; ix < n; ++ix) {
        const size_t g = static_cast<size_t>(iy) * n + ix;
        rhs[2 * g] = phiy[iy] * phix[ix];
        rhs[2 * g + 1] = 0.0;
      }
  }
  HD_GUARD_END
}

hd_status hd_assemble_field(const hd_problem* pb, double* shift_mass_2d) {
  HD_GUARD_BEGIN
  if (!pb || !shift_mass_2d) throw Error(HD_ERR_INVALID, "null argument");
  if (pb->field_kind != HD_FIELD_WEDGE || pb->dim != 2)
    throw Error(HD_ERR_INVALID, "hd_assemble_field: only the 2D wedge field has a non-separable K2");
  if (pb->order < 1 || pb->order > 6 || pb->elements < 1) throw Error(HD_ERR_INVALID, "bad order/elements");
  const Knots kv = Knots::open_uniform(pb->elements, pb->order);
  std::vector<int> kept;
  for (int j = 1; j < kv.basis_count() - 1; ++j) kept.push_back(j);
  const std::vector<double> K = wedge_mass_stencil(kv, pb->k, pb->multipliers, pb->lines, kept);
  std::memcpy(shift_mass_2d, K.data(), K.size() * sizeof(double));
  HD_GUARD_END
}

hd_status hd_create(const hd_system* sys, const hd_precond* spec, const int* devices, int n_devices, hd_ctx** out) {
  HD_GUARD_BEGIN
  create_ctx(sys, spec, devices, n_devices, out);
  HD_GUARD_END
}

hd_status hd_create_slabs(const hd_system* sys, const hd_precond* spec, int nslabs, hd_ctx** out) {
  HD_GUARD_BEGIN
  if (!out || nslabs < 1) throw Error(HD_ERR_INVALID, "nslabs must be >= 1");
  hd_ctx* c = nullptr;
  create_ctx(sys, spec, nullptr, 0, &c);
  try {
    create_slabs(c, nslabs);
  } catch (...) {
    destroy_ctx(c);
    throw;
  }
  *out = c;
  HD_GUARD_END
}

hd_status hd_nccl_unique_id(unsigned char* out) {
  HD_GUARD_BEGIN
  if (!out) throw Error(HD_ERR_INVALID, "null argument");
  ncclUniqueId id;
  CKN(nccl().GetUniqueId(&id));
  std::memcpy(out, id.internal, sizeof(id.internal));
  HD_GUARD_END
}

hd_status hd_create_dist(const hd_system* sys, const hd_precond* spec, int rank, int nranks,
                         const unsigned char* nccl_id, int device, hd_ctx** out) {
  HD_GUARD_BEGIN
  if (!out || !nccl_id || nranks < 1 || rank < 0 || rank >= nranks) throw Error(HD_ERR_INVALID, "bad rank / nranks");
  hd_ctx* c = nullptr;
  const int dev[1] = {device};
  create_ctx(sys, spec, dev, 1, &c);
  try {
    ncclUniqueId id;
    std::memcpy(id.internal, nccl_id, sizeof(id.internal));
    ncclComm_t comm = nullptr;
    CK(cudaSetDevice(device));
    CKN(nccl().CommInitRank(&comm, nranks, id, rank));
    try {
      create_slabs(c, nranks, rank, nranks, comm);
    } catch (...) {
      nccl().CommDestroy(comm);
      throw;
    }
  } catch (...) {
    destroy_ctx(c);
    throw;
  }
  *out = c;
  HD_GUARD_END
}

int hd_slab_info(const hd_ctx* c, int* gather_level, int* bounds) {
  if (!c || !c->slabs) return 0;
  const hd_slabs* sl = reinterpret_cast<const hd_slabs*>(c->slabs);
  if (gather_level) *gather_level = sl->g;
  if (bounds)
    for (int s = 0; s <= sl->S; ++s) bounds[s] = sl->lv[0].bounds[s];
  return sl->S;
}

static hd_status solve_impl(hd_ctx* c, const hd_gmres* opt, const double* rhs, bool rhs_dev, double* x_out,
                            bool x_dev, double* residuals_out, hd_report* report) {
  HD_GUARD_BEGIN
  if (!c || !opt || !rhs || !x_out) throw Error(HD_ERR_INVALID, "null argument");
  if (opt->max_iterations < 0) throw Error(HD_ERR_INVALID, "max_iterations < 0");
  CK(cudaSetDevice(c->device));
  const size_t N = c->N;
  CK(cudaEventRecord(c->ev0, c->st));
  CK(cudaMemcpyAsync(c->f, rhs, N * sizeof(double2), rhs_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     c->st));
  double2* xd = x_dev ? reinterpret_cast<double2*>(x_out) : c->x;
  hd_gmres o = *opt;
  SolveOut r;
  if (o.max_iterations == 0) {
    // degenerate budget: only the start vector and its monitor
    o.max_iterations = 1;
    ensure_gmres(c, 1);
  }
  r = c->slabs ? run_solve_slabs(c, *opt, c->f, xd) : run_solve(c, *opt, xd);
  if (!x_dev) CK(cudaMemcpyAsync(x_out, xd, N * sizeof(double2), cudaMemcpyDeviceToHost, c->st));
  CK(cudaEventRecord(c->ev1, c->st));
  CK(cudaEventSynchronize(c->ev1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  if (residuals_out)
    for (size_t i = 0; i < r.residuals.size(); ++i) residuals_out[i] = r.residuals[i];
  if (report) {
    report->iterations = r.iterations;
    report->converged = r.converged ? 1 : 0;
    report->matvecs = c->matvecs;
    report->coarse_solves = c->coarse_solves;
    report->shift_solves = c->shift_solves;
    report->vcycles = c->vcycles;
    report->t_setup_s = c->t_setup;
    report->t_solve_s = ms * 1e-3;
    report->kernel_launches = c->launches;
    report->library_calls = c->lib_calls;
  }
  HD_GUARD_END
}

hd_status hd_solve(hd_ctx* c, const hd_gmres* opt, const double* rhs, double* x_out, double* residuals_out,
                   hd_report* report) {
  return solve_impl(c, opt, rhs, false, x_out, false, residuals_out, report);
}

hd_status hd_solve_device(hd_ctx* c, const hd_gmres* opt, const double* d_rhs, double* d_x, double* residuals_out,
                          hd_report* report) {
  return solve_impl(c, opt, d_rhs, true, d_x, true, residuals_out, report);
}

long hd_size(const hd_ctx* c) { return c ? static_cast<long>(c->N) : -1; }
int hd_levels(const hd_ctx* c) { return c ? static_cast<int>(c->lev.size()) : -1; }

hd_status hd_apply(hd_ctx* c, int which, const double* d_x, double* d_y) {
  HD_GUARD_BEGIN
  if (!c || !d_x || !d_y) throw Error(HD_ERR_INVALID, "null argument");
  CK(cudaSetDevice(c->device));
  const double2* x = reinterpret_cast<const double2*>(d_x);
  double2* yv = reinterpret_cast<double2*>(d_y);
  if (c->slabs) {  // the row-slab operators: scatter, apply on the slabs, gather
    hd_slabs* sl = slabs_of(c);
    s_scatter(c, x, sl->vin);
    switch (which) {
      case HD_APPLY_A: s_apply(c, OP_APPLY, opA(c), sl->lv[0], sl->vin, nullptr, &sl->t3, 0.0); s_gather(c, sl->t3, yv); break;
      case HD_APPLY_MG: s_mg_solve(c, sl->vin, sl->t2); s_gather(c, sl->t2, yv); break;
      case HD_APPLY_PROJECT:
        if (!c->spec.deflate) throw Error(HD_ERR_INVALID, "no deflation in this context");
        s_deflate(c, sl->vin, sl->rhsp, true); s_gather(c, sl->rhsp, yv); break;
      case HD_APPLY_Q:
        if (!c->spec.deflate) throw Error(HD_ERR_INVALID, "no deflation in this context");
        s_deflate(c, sl->vin, sl->rhsp, false); s_gather(c, sl->rhsp, yv); break;
      case HD_APPLY_OP: s_op(c, sl->vin, sl->w); s_gather(c, sl->w, yv); break;
      default: throw Error(HD_ERR_INVALID, "apply selector not available on row slabs");
    }
    CK(cudaStreamSynchronize(c->st));
    return HD_OK;
  }
  switch (which) {
    case HD_APPLY_A: op_apply(c, OP_APPLY, opA(c), x, nullptr, yv); break;
    case HD_APPLY_SHIFTED: op_apply(c, OP_APPLY, level_dev(c->fine, c->cM, c->corner, c->fine.genM), x, nullptr, yv); break;
    case HD_APPLY_MG:
      if (!c->spec.shift) throw Error(HD_ERR_INVALID, "no multigrid in this context");
      mg_solve(c, x, yv);
      break;
    case HD_APPLY_PROJECT:
      if (!c->spec.deflate) throw Error(HD_ERR_INVALID, "no deflation in this context");
      project(c, x, yv);
      break;
    case HD_APPLY_Q:
      if (!c->spec.deflate) throw Error(HD_ERR_INVALID, "no deflation in this context");
      apply_Q(c, x, yv);
      break;
    case HD_APPLY_OP: compose_op(c, x, yv); break;
    default: throw Error(HD_ERR_INVALID, "unknown apply selector");
  }
  CK(cudaStreamSynchronize(c->st));
  HD_GUARD_END
}

hd_status hd_set_stream(hd_ctx* c, void* stream) {
  HD_GUARD_BEGIN
  if (!c) throw Error(HD_ERR_INVALID, "null context");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->st));
  if (!c->own_st) c->own_st = c->st;
  c->st = stream ? static_cast<cudaStream_t>(stream) : c->own_st;
  CKB(cublasSetStream(c->cb, c->st));
  HD_GUARD_END
}

hd_status hd_profile(hd_ctx* c, int enable) {
  HD_GUARD_BEGIN
  if (!c) throw Error(HD_ERR_INVALID, "null context");
  CK(cudaStreamSynchronize(c->st));
  c->prof_on = enable != 0;
  c->prof_used = 0;
  c->prof_recs.clear();
  HD_GUARD_END
}

hd_status hd_profile_read(hd_ctx* c, int kind, long* launches, double* ms, double* bytes) {
  HD_GUARD_BEGIN
  if (!c || !launches || !ms || !bytes) throw Error(HD_ERR_INVALID, "null argument");
  CK(cudaStreamSynchronize(c->st));
  long n = 0;
  double t = 0.0, b = 0.0;
  for (const auto& r : c->prof_recs) {
    if (r.kind != kind) continue;
    float e = 0.f;
    CK(cudaEventElapsedTime(&e, c->prof_ev[r.ev], c->prof_ev[r.ev + 1]));
    ++n;
    t += e;
    b += r.bytes;
  }
  *launches = n;
  *ms = t;
  *bytes = b;
  HD_GUARD_END
}

int hd_level_size(const hd_ctx* c, int level) {
  if (!c || level < 0 || level >= static_cast<int>(c->lev.size())) return -1;
  return c->lev[level].n;
}

hd_status hd_debug_level(hd_ctx* c, int which, int level, const double* d_x, double* d_y) {
  HD_GUARD_BEGIN
  if (!c || !d_x || !d_y) throw Error(HD_ERR_INVALID, "null argument");
  if (level < 0 || level >= static_cast<int>(c->lev.size())) throw Error(HD_ERR_INVALID, "bad level");
  CK(cudaSetDevice(c->device));
  const double2* x = reinterpret_cast<const double2*>(d_x);
  double2* yv = reinterpret_cast<double2*>(d_y);
  const LevelDev L = levM(c, level);
  const bool has_next = level + 1 < static_cast<int>(c->lev.size());
  switch (which) {
    case 0: op_apply(c, OP_APPLY, L, x, nullptr, yv); break;
    case 1: jacobi0(c, L, x, yv, c->spec.omega); break;
    case 2: op_apply(c, OP_JACOBI, L, x, x, yv, c->spec.omega); break;
    case 3: op_apply(c, OP_RESID, L, x, x, yv); break;
    case 4:
      if (!has_next) throw Error(HD_ERR_INVALID, "no coarser level");
      restrict_(c, Stencil{0, 0.0}, x, L.n, c->lev[level + 1].n, yv, nullptr);
      break;
    case 5:
      if (!has_next) throw Error(HD_ERR_INVALID, "no coarser level");
      prolong_<0>(c, Stencil{0, 0.0}, x, nullptr, L.n, c->lev[level + 1].n, nullptr, yv);
      break;
    case 6: coarsest_solve(c, x, yv); break;
    default: throw Error(HD_ERR_INVALID, "unknown debug selector");
  }
  CK(cudaStreamSynchronize(c->st));
  HD_GUARD_END
}

void hd_destroy(hd_ctx* c) { destroy_ctx(c); }

}  // extern "C"
