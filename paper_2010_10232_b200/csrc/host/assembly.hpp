// Host-side B-spline assembly of the reduced 1D factors the device solver
// consumes.  Mirrors the reference's assembly layer (src/spline.cpp,
// src/assembly.cpp:23-146, 163-258) for the point-source problems: open
// uniform knots, Cox-de Boor evaluation, (p+1)-point Gauss-Legendre rule,
// element stiffness/mass, Dirichlet elimination by dropping end functions.
// The 2D operator is never formed: A = M1(x)S1 + S1(x)M1 - K2 is applied by
// the device from these 1D bands.
#pragma once

#include <vector>

#include "banded.hpp"

namespace hd {

struct Knots {
  int degree = 1, elements = 1;
  std::vector<double> t;
  static Knots open_uniform(int elements, int degree);
  int basis_count() const { return elements + degree; }
  int span_of(double x) const;
};

double bspline_value(const Knots& kv, int degree, int j, double x);
double bspline_derivative(const Knots& kv, int j, double x);
void gauss_legendre(int points, std::vector<double>& nodes, std::vector<double>& weights);

/// Full-basis 1D forms (nb x nb, half-bandwidth p).
struct Forms1d {
  Knots kv;
  Band stiffness, mass;
};
Forms1d assemble_forms_1d(int elements, int order);

/// Mass restricted to [x0, x1] (own Gauss rule per element overlap).
Band mass_on_interval(const Knots& kv, double x0, double x1);

/// Wedge field (BASELINE config 4; an oracle extension, the reference's WaveField
/// cannot express it): top iff y > l[0] + l[1] x, else middle iff y > l[2] + l[3] x,
/// else bottom; k = k0 * mult[layer].
double wedge_k2(double x, double y, double k0, const double* mult, const double* lines);

/// K2 = sum_e sum_(qy,qx) w w k(x_q, y_q)^2 phi phi with the (p+1)-point Gauss rule
/// per direction (src/assembly.cpp:23-43 applied pointwise), on the basis kept in
/// both directions, as a 2D stencil out[(iy*n+ix)*NB*NB + (dy+p)*NB + (dx+p)],
/// NB = 2p+1, n = kept.size().
std::vector<double> wedge_mass_stencil(const Knots& kv, double k0, const double* mult, const double* lines,
                                       const std::vector<int>& kept);

/// Drop rows/cols not in `kept` (Dirichlet elimination).
Band reduce(const Band& full, const std::vector<int>& kept);

}  // namespace hd
