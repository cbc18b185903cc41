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
#include <nvtx3/nvToolsExt.h>  // header-only: ranges cost nothing unless a profiler is attached

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/helmdef_b200.h"
#include "host/assembly.hpp"
#include "host/banded.hpp"
#include "kernels.cuh"
#include "stencil.cuh"
#include "transfer.cuh"
#include "stencil_restrict.cuh"
#include "stencil_tma.cuh"
#include "arnoldi_lowsync.cuh"
#include "layered.cuh"
#include "btri.cuh"
#include "pfd.cuh"
#include "dgemm.cuh"
#include "segsolve.cuh"
#include "tail1d.cuh"
#include "small1d.cuh"


#include "solver/context.cuh"
#include "solver/launch.cuh"
#include "solver/setup.cuh"
#include "solver/slabs.cuh"


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
  NvtxRange nvtx_solve("hd_solve");
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
  for (size_t i = 0; i < r.residuals.size(); ++i)
    if (!std::isfinite(r.residuals[i]))
      throw Error(HD_ERR_NONFINITE, "non-finite residual at GMRES iteration " + std::to_string(i + 1));
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

hd_status hd_direct_solve(const hd_system* sys, const double* rhs, double* x_out) {
  HD_GUARD_BEGIN
  if (!sys || !rhs || !x_out) throw Error(HD_ERR_INVALID, "null argument");
  // A itself is the "shifted" operator with beta2 = 0; cycles = 0 selects its exact inverse
  hd_precond p{};
  p.shift = 1;
  p.beta2 = 0.0;
  p.cycles = 0;
  p.smooth_steps = 1;
  p.omega = 0.6;
  p.coarsest = 32;
  hd_ctx* c = nullptr;
  create_ctx(sys, &p, nullptr, 0, &c);
  std::unique_ptr<hd_ctx, void (*)(hd_ctx*)> guard(c, destroy_ctx);
  const size_t N = c->N;
  CK(cudaMemcpyAsync(c->f, rhs, N * sizeof(double2), cudaMemcpyHostToDevice, c->st));
  shift_exact_solve(c, c->f, c->x);
  CK(cudaMemcpyAsync(x_out, c->x, N * sizeof(double2), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  HD_GUARD_END
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

long hd_debug_check_guards(void) {
  try {
    return check_guards();
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return -1;
  }
}

void hd_destroy(hd_ctx* c) { destroy_ctx(c); }

}  // extern "C"
