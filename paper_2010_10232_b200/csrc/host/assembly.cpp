// SPDX-License-Identifier: Apache-2.0
#include "assembly.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace hd {

Knots Knots::open_uniform(int elements, int degree) {
  if (elements < 1 || degree < 1) throw std::invalid_argument("knots need elements >= 1 and degree >= 1");
  Knots k;
  k.degree = degree;
  k.elements = elements;
  k.t.assign(degree, 0.0);
  for (int i = 0; i <= elements; ++i) k.t.push_back(static_cast<double>(i) / elements);
  k.t.insert(k.t.end(), degree, 1.0);
  return k;
}

int Knots::span_of(double x) const {
  if (x >= 1.0) return elements - 1;
  if (x <= 0.0) return 0;
  return std::min(static_cast<int>(x * elements), elements - 1);
}

// Degree-0 indicator of [t_j, t_{j+1}); the right end x = 1 belongs to the
// last non-degenerate span (src/spline.cpp:36-40).
static inline double indicator(const std::vector<double>& t, int j, double x) {
  if (t[j] <= x && x < t[j + 1]) return 1.0;
  return (x == t.back() && t[j] < t[j + 1] && t[j + 1] == t.back()) ? 1.0 : 0.0;
}

double bspline_value(const Knots& kv, int degree, int j, double x) {
  const auto& t = kv.t;
  double N[16];
  for (int r = 0; r <= degree; ++r) N[r] = indicator(t, j + r, x);
  for (int d = 1; d <= degree; ++d)
    for (int r = 0; r + d <= degree; ++r) {
      const double dl = t[j + r + d] - t[j + r];
      const double dr = t[j + r + d + 1] - t[j + r + 1];
      const double a = dl > 0.0 ? (x - t[j + r]) / dl * N[r] : 0.0;
      const double b = dr > 0.0 ? (t[j + r + d + 1] - x) / dr * N[r + 1] : 0.0;
      N[r] = a + b;
    }
  return N[0];
}

double bspline_derivative(const Knots& kv, int j, double x) {
  const int p = kv.degree;
  const auto& t = kv.t;
  const double dl = t[j + p] - t[j];
  const double dr = t[j + p + 1] - t[j + 1];
  const double a = dl > 0.0 ? bspline_value(kv, p - 1, j, x) / dl : 0.0;
  const double b = dr > 0.0 ? bspline_value(kv, p - 1, j + 1, x) / dr : 0.0;
  return p * (a - b);
}

void gauss_legendre(int points, std::vector<double>& nodes, std::vector<double>& weights) {
  nodes.assign(points, 0.0);
  weights.assign(points, 0.0);
  const double pi = std::acos(-1.0);
  for (int i = 0; i < points; ++i) {
    double x = std::cos(pi * (i + 0.75) / (points + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      // Legendre three-term recurrence for P_n(x) and P_{n-1}(x)
      double pm = 1.0, pn = x;
      for (int m = 2; m <= points; ++m) {
        const double next = ((2 * m - 1) * x * pn - (m - 1) * pm) / m;
        pm = pn;
        pn = next;
      }
      if (points == 1) pm = 1.0;
      dp = points * (x * pn - pm) / (x * x - 1.0);
      const double step = pn / dp;
      x -= step;
      if (std::abs(step) < 1e-15) break;
    }
    nodes[i] = x;
    weights[i] = 2.0 / ((1.0 - x * x) * dp * dp);
  }
}

namespace {

// Element matrices over [a, a+len] on element e: sum_q w_q f_a(x_q) f_b(x_q).
void element_mats(const Knots& kv, int e, double a, double len, const std::vector<double>& nodes,
                  const std::vector<double>& weights, std::vector<double>& ks, std::vector<double>& km) {
  const int p = kv.degree;
  const int m = p + 1;
  ks.assign(m * m, 0.0);
  km.assign(m * m, 0.0);
  std::vector<double> v(m), d(m);
  for (size_t q = 0; q < nodes.size(); ++q) {
    const double x = a + 0.5 * len * (nodes[q] + 1.0);
    const double wq = 0.5 * len * weights[q];
    for (int l = 0; l < m; ++l) {
      v[l] = bspline_value(kv, p, e + l, x);
      d[l] = bspline_derivative(kv, e + l, x);
    }
    for (int r = 0; r < m; ++r)
      for (int c = 0; c < m; ++c) {
        ks[r * m + c] += d[r] * wq * d[c];
        km[r * m + c] += v[r] * wq * v[c];
      }
  }
}

}  // namespace

Forms1d assemble_forms_1d(int elements, int order) {
  Forms1d f;
  f.kv = Knots::open_uniform(elements, order);
  const int nb = f.kv.basis_count();
  const int p = order;
  std::vector<double> nodes, weights;
  gauss_legendre(p + 1, nodes, weights);
  f.stiffness = Band(nb, p);
  f.mass = Band(nb, p);
  const double h = 1.0 / elements;
  // uniform knots: every interior element (p <= e < elements-p) has the same
  // element matrices (the reference caches them, src/assembly.cpp:47-72)
  std::vector<double> is, im;
  bool have_interior = false;
  std::vector<double> ks, km;
  for (int e = 0; e < elements; ++e) {
    const bool interior = e >= p && e < elements - p;
    const std::vector<double>* S;
    const std::vector<double>* M;
    if (interior) {
      if (!have_interior) {
        const int er = std::min(p, elements - 1);
        element_mats(f.kv, er, er * h, h, nodes, weights, is, im);
        have_interior = true;
      }
      S = &is;
      M = &im;
    } else {
      element_mats(f.kv, e, e * h, h, nodes, weights, ks, km);
      S = &ks;
      M = &km;
    }
    for (int r = 0; r <= p; ++r)
      for (int c = 0; c <= p; ++c) {
        f.stiffness.ref(e + r, e + c) += (*S)[r * (p + 1) + c];
        f.mass.ref(e + r, e + c) += (*M)[r * (p + 1) + c];
      }
  }
  return f;
}

Band mass_on_interval(const Knots& kv, double x0, double x1) {
  const int p = kv.degree;
  std::vector<double> nodes, weights, ks, km;
  gauss_legendre(p + 1, nodes, weights);
  Band out(kv.basis_count(), p);
  const double h = 1.0 / kv.elements;
  for (int e = 0; e < kv.elements; ++e) {
    const double a = std::max(e * h, x0);
    const double b = std::min((e + 1) * h, x1);
    if (b - a < 1e-14) continue;
    element_mats(kv, e, a, b - a, nodes, weights, ks, km);
    for (int r = 0; r <= p; ++r)
      for (int c = 0; c <= p; ++c) out.ref(e + r, e + c) += km[r * (p + 1) + c];
  }
  return out;
}

double wedge_k2(double x, double y, double k0, const double* mult, const double* lines) {
  const double m = y > lines[0] + lines[1] * x ? mult[0] : (y > lines[2] + lines[3] * x ? mult[1] : mult[2]);
  const double kk = k0 * m;
  return kk * kk;
}

std::vector<double> wedge_mass_stencil(const Knots& kv, double k0, const double* mult, const double* lines,
                                       const std::vector<int>& kept) {
  const int p = kv.degree, m = p + 1, ne = kv.elements, nb = kv.basis_count(), NB = 2 * p + 1;
  std::vector<double> nodes, weights;
  gauss_legendre(m, nodes, weights);
  const double h = 1.0 / ne;
  // Gauss points, weights and the p+1 nonzero basis values of every element
  std::vector<double> X(static_cast<size_t>(ne) * m), W(X.size()), B(X.size() * m);
  for (int e = 0; e < ne; ++e)
    for (int q = 0; q < m; ++q) {
      const double x = e * h + 0.5 * h * (nodes[q] + 1.0);
      X[e * m + q] = x;
      W[e * m + q] = 0.5 * h * weights[q];
      for (int l = 0; l < m; ++l) B[(static_cast<size_t>(e) * m + q) * m + l] = bspline_value(kv, p, e + l, x);
    }
  // full-basis band table K[iy][dy][ix][dx]
  const size_t rowsz = static_cast<size_t>(NB) * nb * NB;
  std::vector<double> K(static_cast<size_t>(nb) * rowsz, 0.0);
  std::vector<double> T(static_cast<size_t>(m) * m * m);  // T[qy][lx][mx] of one element
  std::vector<double> KK(static_cast<size_t>(m) * m);      // k^2 at the element's Gauss points [qy][qx]
  for (int ey = 0; ey < ne; ++ey)
    for (int ex = 0; ex < ne; ++ex) {
      for (int qy = 0; qy < m; ++qy)
        for (int qx = 0; qx < m; ++qx) KK[qy * m + qx] = wedge_k2(X[ex * m + qx], X[ey * m + qy], k0, mult, lines);
      // x stage: T[qy][lx][mx] = sum_qx w_qx k^2 B[ex,qx,lx] B[ex,qx,mx]
      for (int qy = 0; qy < m; ++qy)
        for (int lx = 0; lx < m; ++lx)
          for (int mx = 0; mx < m; ++mx) {
            double t = 0.0;
            for (int qx = 0; qx < m; ++qx) {
              const double kk = KK[qy * m + qx];
              t += kk * W[ex * m + qx] * B[(static_cast<size_t>(ex) * m + qx) * m + lx] *
                   B[(static_cast<size_t>(ex) * m + qx) * m + mx];
            }
            T[(qy * m + lx) * m + mx] = t;
          }
      // y stage into the band table
      for (int ly = 0; ly < m; ++ly)
        for (int my = 0; my < m; ++my)
          for (int lx = 0; lx < m; ++lx)
            for (int mx = 0; mx < m; ++mx) {
              double v = 0.0;
              for (int qy = 0; qy < m; ++qy)
                v += W[ey * m + qy] * B[(static_cast<size_t>(ey) * m + qy) * m + ly] *
                     B[(static_cast<size_t>(ey) * m + qy) * m + my] * T[(qy * m + lx) * m + mx];
              K[static_cast<size_t>(ey + ly) * rowsz + (static_cast<size_t>(my - ly + p) * nb + ex + lx) * NB +
                (mx - lx + p)] += v;
            }
    }
  // reduce to the kept basis (contiguous in this build: Dirichlet on all faces)
  const int n = static_cast<int>(kept.size());
  std::vector<double> out(static_cast<size_t>(n) * n * NB * NB, 0.0);
  for (int iy = 0; iy < n; ++iy)
    for (int dy = -p; dy <= p; ++dy) {
      const int jy = iy + dy;
      if (jy < 0 || jy >= n) continue;
      for (int ix = 0; ix < n; ++ix)
        for (int dx = -p; dx <= p; ++dx) {
          const int jx = ix + dx;
          if (jx < 0 || jx >= n) continue;
          const int fy = kept[iy], fx = kept[ix];
          const int gy = kept[jy] - fy, gx = kept[jx] - fx;
          if (gy < -p || gy > p || gx < -p || gx > p) continue;
          out[(static_cast<size_t>(iy) * n + ix) * NB * NB + (dy + p) * NB + (dx + p)] =
              K[static_cast<size_t>(fy) * rowsz + (static_cast<size_t>(gy + p) * nb + fx) * NB + (gx + p)];
        }
    }
  return out;
}

Band reduce(const Band& full, const std::vector<int>& kept) {
  const int n = static_cast<int>(kept.size());
  Band out(n, full.b);
  for (int i = 0; i < n; ++i)
    for (int d = -full.b; d <= full.b; ++d) {
      const int j = i + d;
      if (j < 0 || j >= n) continue;
      out.ref(i, j) = full.at(kept[i], kept[j]);
    }
  return out;
}

}  // namespace hd
