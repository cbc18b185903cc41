// helmdef_b200.hpp -- C++17 host mirror of the reference's solve API over the
// C-ABI of helmdef_b200.h (header-only; link libhelmdef_b200.so).
//
// Same names, fields and error behaviour as the reference (helmdef, C++20):
//   Problem factories           include/helmdef/problems.hpp, src/problems.cpp:34-74
//   DiscreteSystem / assemble   include/helmdef/assembly.hpp:43-52, src/assembly.cpp:163-258
//                               (factored form: the 1D bands the device consumes)
//   PrecondSpec, OperationCounts, SolverSetup, compose
//                               include/helmdef/precond.hpp:114-149, src/precond.cpp:196-265
//   GmresOptions, GmresResult, gmres
//                               include/helmdef/linalg.hpp:24-42, src/linalg.cpp:10-92
//   to_spec, derived_elements, RunRecord, run_cell
//                               include/helmdef/harness.hpp:75-98, src/harness.cpp:149-243
// Differences forced by the device boundary: the SolverSetup owns a device
// context instead of host closures, and gmres() takes the setup (its op, rhs,
// start and monitor live on the GPU).  Errors are std::runtime_error (the
// reference's convention for LU failure, zero smoother diagonal and bad
// configurations); non-convergence is converged = false, as in the reference.
#pragma once

#include <array>
#include <chrono>
#include <cmath>
#include <complex>
#include <limits>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "helmdef_b200.h"

namespace helmdef_b200 {

using cplx = std::complex<double>;
using Vec = std::vector<cplx>;

class Error : public std::runtime_error {
 public:
  Error(hd_status s, const std::string& what) : std::runtime_error(what), status(s) {}
  hd_status status;
};

inline void check(hd_status s) {
  if (s != HD_OK) throw Error(s, hd_last_error());
}

// src/problems.cpp:25-32: the pinned 4x4 multiplier table of layered_medium_2d
inline const std::array<double, 16>& layered_multipliers() {
  static const std::array<double, 16> m = {1.00, 0.50, 1.25, 0.75, 1.50, 1.00, 0.50, 1.25,
                                           0.75, 1.50, 1.00, 0.50, 1.25, 0.75, 1.50, 1.00};
  return m;
}

struct Problem {
  std::string name = "point_source_1d";
  int dim = 1;
  int order = 1;
  int elements = 8;
  double k = 1.0;
  bool layered = false;
  std::array<double, 16> multipliers{};
  // BASELINE config-4 wedge (an extension: the reference's WaveField cannot express it)
  bool wedge = false;
  std::array<double, 4> lines{{0.6, -0.2, 0.3, 0.1}};  // top iff y > l0 + l1 x; middle iff y > l2 + l3 x
  bool point_source = false;                           // load at `source` instead of (1/2, 1/2)
  std::array<double, 2> source{{0.5, 0.5}};
};

inline Problem point_source_1d(int elements, int order, double k) {
  Problem p;
  p.name = "point_source_1d";
  p.dim = 1;
  p.order = order;
  p.elements = elements;
  p.k = k;
  p.multipliers.fill(1.0);
  return p;
}
inline Problem point_source_2d(int elements, int order, double k) {
  Problem p = point_source_1d(elements, order, k);
  p.name = "point_source_2d";
  p.dim = 2;
  return p;
}
inline Problem layered_medium_2d(int elements, int order, double k,
                                 const std::array<double, 16>& m = layered_multipliers()) {
  Problem p = point_source_2d(elements, order, k);
  p.name = "layered_medium_2d";
  p.layered = true;
  p.multipliers = m;
  return p;
}

// The three-layer wedge k = k0 (1.2, 1.5, 1.0) with the load at (1/2, 1 - h):
// BASELINE config 4 (oracle/helmdef_oracle.py wedge_2d freezes the same rule).
inline Problem wedge_2d(int elements, int order, double k0) {
  Problem p;
  p.name = "wedge_2d";
  p.dim = 2;
  p.order = order;
  p.elements = elements;
  p.k = k0;
  p.wedge = true;
  p.multipliers.fill(0.0);
  p.multipliers[0] = 1.2;
  p.multipliers[1] = 1.5;
  p.multipliers[2] = 1.0;
  p.point_source = true;
  p.source = {{0.5, 1.0 - 1.0 / elements}};
  return p;
}

struct DiscreteSystem {
  int dim = 1, order = 1, elements = 1, per_dim = 0;
  double k = 0.0;
  bool layered = false;
  bool wedge = false;
  std::vector<double> shift_mass_2d;  // wedge: K2 as a 2D stencil, N x (2p+1)^2
  std::array<double, 16> multipliers{};
  std::vector<double> stiffness_band, mass_band, interval_mass;  // per_dim x (2p+1) (x4 for interval_mass)
  Vec rhs;
  long size() const { return static_cast<long>(rhs.size()); }
};

inline hd_problem to_hd(const Problem& pb) {
  hd_problem h{};
  h.dim = pb.dim;
  h.order = pb.order;
  h.elements = pb.elements;
  h.k = pb.k;
  h.field_kind = pb.wedge ? HD_FIELD_WEDGE : (pb.layered ? HD_FIELD_LAYERED : HD_FIELD_CONSTANT);
  for (int i = 0; i < 16; ++i) h.multipliers[i] = pb.multipliers[i];
  for (int i = 0; i < 4; ++i) h.lines[i] = pb.lines[i];
  h.point_source = pb.point_source ? 1 : 0;
  h.source[0] = pb.source[0];
  h.source[1] = pb.source[1];
  return h;
}

inline DiscreteSystem assemble(const Problem& pb) {
  const hd_problem h = to_hd(pb);
  DiscreteSystem s;
  s.dim = pb.dim;
  s.order = pb.order;
  s.elements = pb.elements;
  s.k = pb.k;
  s.layered = pb.layered;
  s.multipliers = pb.multipliers;
  s.per_dim = hd_problem_per_dim(&h);
  if (s.per_dim < 1) throw Error(HD_ERR_INVALID, "problem has no unknowns");
  const size_t nb = static_cast<size_t>(s.per_dim) * (2 * pb.order + 1);
  s.stiffness_band.assign(nb, 0.0);
  s.mass_band.assign(nb, 0.0);
  if (pb.layered) s.interval_mass.assign(4 * nb, 0.0);
  const size_t N = pb.dim == 2 ? static_cast<size_t>(s.per_dim) * s.per_dim : static_cast<size_t>(s.per_dim);
  s.rhs.assign(N, cplx(0.0, 0.0));
  check(hd_assemble(&h, s.stiffness_band.data(), s.mass_band.data(),
                    pb.layered ? s.interval_mass.data() : nullptr, reinterpret_cast<double*>(s.rhs.data())));
  s.wedge = pb.wedge;
  if (pb.wedge) {
    s.shift_mass_2d.assign(N * (2 * pb.order + 1) * (2 * pb.order + 1), 0.0);
    check(hd_assemble_field(&h, s.shift_mass_2d.data()));
  }
  return s;
}

struct OperationCounts {
  long matvecs = 0;
  long coarse_solves = 0;
  long shift_solves = 0;
  long vcycles = 0;
};

struct PrecondSpec {
  bool deflate = false;
  double drop = 0.0;
  bool shift = false;
  double beta2 = 1.0;
  int cycles = 0;
  int smooth_steps = 1;
  double omega = 0.6;
};

struct GmresOptions {
  int max_iterations = 100;
  double tolerance = 1e-7;
};

struct GmresResult {
  Vec solution;
  int iterations = 0;
  bool converged = false;
  std::vector<double> residuals;
};

// compose(): the device context (hierarchy, E and its exact solver, buffers)
class SolverSetup {
 public:
  SolverSetup() = default;
  SolverSetup(const SolverSetup&) = delete;
  SolverSetup& operator=(const SolverSetup&) = delete;
  SolverSetup(SolverSetup&& o) noexcept { *this = std::move(o); }
  SolverSetup& operator=(SolverSetup&& o) noexcept {
    if (this != &o) {
      reset();
      ctx_ = o.ctx_;
      o.ctx_ = nullptr;
      rhs = std::move(o.rhs);
      counts = std::move(o.counts);
      t_setup = o.t_setup;
    }
    return *this;
  }
  ~SolverSetup() { reset(); }
  hd_ctx* context() const { return ctx_; }
  Vec rhs;                                    // the system's f (the transformed rhs lives on the device)
  std::shared_ptr<OperationCounts> counts;    // accumulated over the solves of this setup
  double t_setup = 0.0;

 private:
  friend SolverSetup compose(const DiscreteSystem&, const PrecondSpec&);
  void reset() {
    if (ctx_) hd_destroy(ctx_);
    ctx_ = nullptr;
  }
  hd_ctx* ctx_ = nullptr;
};

// the device's view of a DiscreteSystem (plain pointers into sys; sys must outlive the call)
inline hd_system to_hd_system(const DiscreteSystem& sys) {
  hd_system hs{};
  hs.dim = sys.dim;
  hs.order = sys.order;
  hs.elements = sys.elements;
  hs.per_dim = sys.per_dim;
  hs.field_kind = sys.wedge ? HD_FIELD_WEDGE : (sys.layered ? HD_FIELD_LAYERED : HD_FIELD_CONSTANT);
  hs.k = sys.k;
  for (int i = 0; i < 16; ++i) hs.multipliers[i] = sys.multipliers[i];
  hs.stiffness_band = sys.stiffness_band.data();
  hs.mass_band = sys.mass_band.data();
  hs.interval_mass = sys.layered ? sys.interval_mass.data() : nullptr;
  hs.shift_mass_2d = sys.wedge ? sys.shift_mass_2d.data() : nullptr;
  return hs;
}

inline SolverSetup compose(const DiscreteSystem& sys, const PrecondSpec& spec) {
  const hd_system hs = to_hd_system(sys);
  hd_precond hp{};
  hp.deflate = spec.deflate ? 1 : 0;
  hp.drop = spec.drop;
  hp.shift = spec.shift ? 1 : 0;
  hp.beta2 = spec.beta2;
  hp.cycles = spec.cycles;
  hp.smooth_steps = spec.smooth_steps;
  hp.omega = spec.omega;
  hp.coarsest = 32;  // MultigridOptions::coarsest (include/helmdef/precond.hpp:57-61)
  SolverSetup s;
  check(hd_create(&hs, &hp, nullptr, 0, &s.ctx_));
  s.rhs = sys.rhs;
  s.counts = std::make_shared<OperationCounts>();
  return s;
}

// gmres(setup.op, setup.rhs, setup.start, setup.monitor, opt) as one device call
inline GmresResult gmres(SolverSetup& setup, const GmresOptions& opt = {}, const Vec* rhs = nullptr) {
  if (!setup.context()) throw Error(HD_ERR_INVALID, "empty SolverSetup");
  const Vec& f = rhs ? *rhs : setup.rhs;
  GmresResult r;
  r.solution.assign(f.size(), cplx(0.0, 0.0));
  std::vector<double> res(static_cast<size_t>(opt.max_iterations) + 1, 0.0);
  hd_gmres ho{opt.max_iterations, opt.tolerance};
  hd_report rep{};
  check(hd_solve(setup.context(), &ho, reinterpret_cast<const double*>(f.data()),
                 reinterpret_cast<double*>(r.solution.data()), res.data(), &rep));
  r.iterations = rep.iterations;
  r.converged = rep.converged != 0;
  // one entry per iteration; an immediate exit on tolerance carries the start's residual
  // (src/linalg.cpp:17-22), a zero Krylov start none (:26-30)
  if (rep.iterations > 0 || rep.converged)
    r.residuals.assign(res.begin(), res.begin() + (rep.iterations > 0 ? rep.iterations : 1));
  setup.counts->matvecs += rep.matvecs;
  setup.counts->coarse_solves += rep.coarse_solves;
  setup.counts->shift_solves += rep.shift_solves;
  setup.counts->vcycles += rep.vcycles;
  setup.t_setup = rep.t_setup_s;
  return r;
}

// ---- harness (src/harness.cpp) ----------------------------------------------
inline int resolution_for(double k, double kh) { return static_cast<int>(std::ceil(k / kh - 1e-12)); }  // src/problems.cpp:110-114
inline int derived_elements(double k, double kh, int order) {  // src/harness.cpp:149-152
  const int e = resolution_for(k, kh) + 1 - order;
  return e > 4 ? e : 4;
}
inline double resolve_beta2(const std::string& expr, double k) {  // src/harness.cpp:143-147
  if (expr == "1/k") return 1.0 / k;
  if (expr == "1/(3k)") return 1.0 / (3.0 * k);
  return std::stod(expr);
}
// src/harness.cpp:175-205, including the per-degree overrides of :200-203
inline PrecondSpec to_spec(const std::string& tag, int order, double k, double epsilon = 0.1,
                           const std::string& beta2 = "1", int cycles = 1, int smoothing = 1, double omega = 0.6,
                           const std::map<int, int>& smoothing_by_p = {},
                           const std::map<int, double>& omega_by_p = {}) {
  PrecondSpec s;
  if (tag == "D") {
    s.deflate = true;
  } else if (tag == "D_eps") {
    s.deflate = true;
    s.drop = epsilon;
  } else if (tag == "C_ex") {
    s.shift = true;
    s.cycles = 0;
  } else if (tag == "DC_MG") {
    s.deflate = s.shift = true;
    s.cycles = cycles;
  } else if (tag == "Deps_C_MG") {
    s.deflate = s.shift = true;
    s.drop = epsilon;
    s.cycles = cycles;
  } else if (tag != "none") {
    throw Error(HD_ERR_INVALID, "unknown preconditioner tag: " + tag);
  }
  if (s.shift) s.beta2 = resolve_beta2(beta2, k);
  const auto is = smoothing_by_p.find(order);
  s.smooth_steps = is != smoothing_by_p.end() ? is->second : smoothing;
  const auto io = omega_by_p.find(order);
  s.omega = io != omega_by_p.end() ? io->second : omega;
  return s;
}
inline std::string label(const std::string& tag, int cycles) {  // src/harness.cpp:77-82
  return (tag == "DC_MG" || tag == "Deps_C_MG") ? tag + "^" + std::to_string(cycles) : tag;
}

struct RunRecord {  // include/helmdef/harness.hpp:81-98
  std::string problem, tag;
  double k = 0.0;
  int order = 0, elements = 0;
  long dofs = 0;
  int iterations = 0;
  bool converged = false;
  double residual = 0.0;
  double direct_gap = std::numeric_limits<double>::quiet_NaN();  // ||x - A^-1 f|| / ||A^-1 f|| (check_direct)
  long matvecs = 0, shift_solves = 0, vcycles = 0, coarse_solves = 0;
  double seconds = 0.0;
  std::string config_hash;  // FNV-1a of the sweep config (helmdef_b200_harness.hpp)
};

inline RunRecord run_cell(const Problem& pb, const PrecondSpec& spec, const std::string& tag,
                          const GmresOptions& opt, GmresResult* out = nullptr) {  // src/harness.cpp:207-243
  const auto t0 = std::chrono::steady_clock::now();
  const DiscreteSystem sys = assemble(pb);
  SolverSetup setup = compose(sys, spec);
  GmresResult gr = gmres(setup, opt);
  RunRecord r;
  r.problem = pb.name;
  r.tag = tag;
  r.k = pb.k;
  r.order = pb.order;
  r.elements = pb.elements;
  r.dofs = sys.size();
  r.iterations = gr.iterations;
  r.converged = gr.converged;
  r.residual = gr.residuals.empty() ? 0.0 : gr.residuals.back();
  r.matvecs = setup.counts->matvecs;
  r.shift_solves = setup.counts->shift_solves;
  r.vcycles = setup.counts->vcycles;
  r.coarse_solves = setup.counts->coarse_solves;
  r.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (out) *out = std::move(gr);
  return r;
}

}  // namespace helmdef_b200
