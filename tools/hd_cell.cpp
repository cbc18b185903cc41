// hd_cell -- one iteration-study cell through the C++ host mirror
// (include/helmdef_b200.hpp), the B200 counterpart of the reference's
// run_cell (src/harness.cpp:207-243).  Prints the RunRecord and the residual
// history as one JSON line; exit status 0, or 2 with the library's error
// message on stderr (no CUDA device, bad configuration, singular operator).
//
//   hd_cell <problem> <tag> <p> <k> [elements|0] [beta2] [cycles] [smoothing] [omega] [maxit] [tol] [epsilon]
//   hd_cell --assemble <problem> <p> <k> <elements>      (host assembly only: per_dim, |f|, band sums)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "helmdef_b200.hpp"

namespace hb = helmdef_b200;

static hb::Problem make_problem(const std::string& name, int e, int p, double k) {
  if (name == "point_source_1d") return hb::point_source_1d(e, p, k);
  if (name == "point_source_2d") return hb::point_source_2d(e, p, k);
  if (name == "layered_medium_2d") return hb::layered_medium_2d(e, p, k);
  if (name == "wedge_2d") return hb::wedge_2d(e, p, k);
  throw hb::Error(HD_ERR_INVALID, "unknown problem: " + name);
}

int main(int argc, char** argv) {
  try {
    if (argc >= 6 && std::string(argv[1]) == "--assemble") {
      const hb::Problem pb = make_problem(argv[2], std::atoi(argv[5]), std::atoi(argv[3]), std::atof(argv[4]));
      const hb::DiscreteSystem s = hb::assemble(pb);
      double fn = 0.0, ss = 0.0, ms = 0.0;
      for (const auto& v : s.rhs) fn += std::norm(v);
      for (double v : s.stiffness_band) ss += v;
      for (double v : s.mass_band) ms += v;
      double ks = 0.0;
      for (double v : s.shift_mass_2d) ks += v;
      std::printf("{\"per_dim\": %d, \"size\": %ld, \"rhs_norm\": %.17g, \"stiffness_sum\": %.17g, \"mass_sum\": %.17g, "
                  "\"shift_mass_sum\": %.17g}\n",
                  s.per_dim, s.size(), std::sqrt(fn), ss, ms, ks);
      return 0;
    }
    if (argc < 5) {
      std::fprintf(stderr,
                   "usage: hd_cell <problem> <tag> <p> <k> [elements|0] [beta2] [cycles] [smoothing] [omega] "
                   "[maxit] [tol] [epsilon]\n       hd_cell --assemble <problem> <p> <k> <elements>\n");
      return 2;
    }
    const std::string problem = argv[1], tag = argv[2];
    const int p = std::atoi(argv[3]);
    const double k = std::atof(argv[4]);
    int elements = argc > 5 ? std::atoi(argv[5]) : 0;
    if (elements <= 0) elements = hb::derived_elements(k, 0.625, p);
    const std::string beta2 = argc > 6 ? argv[6] : "1";
    const int cycles = argc > 7 ? std::atoi(argv[7]) : 1;
    const int smoothing = argc > 8 ? std::atoi(argv[8]) : 1;
    const double omega = argc > 9 ? std::atof(argv[9]) : 0.6;
    hb::GmresOptions opt;
    if (argc > 10) opt.max_iterations = std::atoi(argv[10]);
    if (argc > 11) opt.tolerance = std::atof(argv[11]);
    const double eps = argc > 12 ? std::atof(argv[12]) : 0.1;
    const hb::PrecondSpec spec = hb::to_spec(tag, p, k, eps, beta2, cycles, smoothing, omega);
    hb::GmresResult gr;
    const hb::RunRecord r = hb::run_cell(make_problem(problem, elements, p, k), spec, hb::label(tag, cycles), opt, &gr);
    double xn = 0.0;
    for (const auto& v : gr.solution) xn += std::norm(v);
    std::printf("{\"problem\": \"%s\", \"tag\": \"%s\", \"k\": %.17g, \"order\": %d, \"elements\": %d, \"dofs\": %ld, "
                "\"iterations\": %d, \"converged\": %s, \"residual\": %.17g, \"matvecs\": %ld, \"shift_solves\": %ld, "
                "\"vcycles\": %ld, \"coarse_solves\": %ld, \"seconds\": %.6f, \"solution_norm\": %.17g, \"residuals\": [",
                r.problem.c_str(), r.tag.c_str(), r.k, r.order, r.elements, r.dofs, r.iterations,
                r.converged ? "true" : "false", r.residual, r.matvecs, r.shift_solves, r.vcycles, r.coarse_solves,
                r.seconds, std::sqrt(xn));
    for (size_t i = 0; i < gr.residuals.size(); ++i) std::printf("%s%.17g", i ? ", " : "", gr.residuals[i]);
    std::printf("]}\n");
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "hd_cell: %s\n", e.what());
    return 2;
  }
}
