// SPDX-License-Identifier: Apache-2.0
#include "banded.hpp"

#include <algorithm>
#include <cmath>

namespace hd {

Band Band::trimmed() const {
  int bb = 0;
  for (int i = 0; i < n; ++i)
    for (int d = -b; d <= b; ++d)
      if (at(i, i + d) != 0.0) bb = std::max(bb, std::abs(d));
  Band out(n, bb);
  for (int i = 0; i < n; ++i)
    for (int d = -bb; d <= bb; ++d) {
      const int j = i + d;
      if (j >= 0 && j < n) out.ref(i, j) = at(i, j);
    }
  return out;
}

Transfer halving_stencil(int fine, double drop) {
  Transfer z;
  z.fine = fine;
  z.coarse = fine / 2;
  auto push = [&](int j, int c, double w) {
    if (c >= 1 && c <= z.coarse) {
      z.row.push_back(j - 1);
      z.col.push_back(c - 1);
      z.w.push_back(w);
    }
  };
  for (int j = 1; j <= fine; ++j) {
    if (j % 2 == 0) {
      push(j, (j - 2) / 2, 1.0 / 8.0);
      push(j, j / 2, (6.0 - drop) / 8.0);
      push(j, (j + 2) / 2, 1.0 / 8.0);
    } else {
      push(j, (j - 1) / 2, 0.5);
      push(j, (j + 1) / 2, 0.5);
    }
  }
  return z;
}

Transfer linear_stencil(int fine) {
  Transfer z;
  z.fine = fine;
  z.coarse = fine / 2;
  auto push = [&](int j, int c, double w) {
    if (c >= 1 && c <= z.coarse) {
      z.row.push_back(j - 1);
      z.col.push_back(c - 1);
      z.w.push_back(w);
    }
  };
  for (int j = 1; j <= fine; ++j) {
    if (j % 2 == 0) {
      push(j, j / 2, 1.0);
    } else {
      push(j, (j - 1) / 2, 0.5);
      push(j, (j + 1) / 2, 0.5);
    }
  }
  return z;
}

Band galerkin(const Band& A, const Transfer& z) {
  if (A.n != z.fine) throw std::invalid_argument("galerkin: size mismatch");
  // rows of z: fine index -> list of (coarse, w)
  std::vector<std::vector<std::pair<int, double>>> zr(z.fine);
  for (size_t t = 0; t < z.w.size(); ++t) zr[z.row[t]].push_back({z.col[t], z.w[t]});
  // C = z^T (A z); bandwidth bound: (A.b + 4) / 2 + 1 is ample for both stencils
  const int bc = (A.b + 4) / 2 + 1;
  Band C(z.coarse, bc);
  for (int i = 0; i < z.fine; ++i) {
    for (const auto& [q, wq] : zr[i]) {
      for (int d = -A.b; d <= A.b; ++d) {
        const int i2 = i + d;
        if (i2 < 0 || i2 >= A.n) continue;
        const double aij = A.at(i, i2);
        if (aij == 0.0) continue;
        for (const auto& [q2, wq2] : zr[i2]) C.ref(q, q2) += wq * aij * wq2;
      }
    }
  }
  return C.trimmed();
}

namespace {

// Banded LU with partial pivoting of S - c M (+ corner), scalar type T
// (complex for the 1D operators, real for the per-mode systems of the
// partially diagonalised E); the same elimination order for both.
template <class T, class F>
void band_lu_t(const Band& S, const Band& M, T c, T corner, F& f) {
  const int n = S.n;
  const int kl = std::max(S.b, M.b);
  const int ku = kl;
  const int w = 2 * kl + ku + 1;  // window columns [i-kl, i+kl+ku]
  std::vector<T> W(static_cast<size_t>(n) * w, T(0.0));
  auto el = [&](int i, int j) -> T& { return W[static_cast<size_t>(i) * w + (j - i + kl)]; };
  for (int i = 0; i < n; ++i)
    for (int d = -kl; d <= ku; ++d) {
      const int j = i + d;
      if (j < 0 || j >= n) continue;
      el(i, j) = T(S.at(i, j)) - c * M.at(i, j);
    }
  el(n - 1, n - 1) += corner;
  f.n = n;
  f.kl = kl;
  f.ku = kl + ku;
  f.L.assign(static_cast<size_t>(n) * std::max(kl, 1), T(0.0));
  f.U.assign(static_cast<size_t>(n) * (f.ku + 1), T(0.0));
  f.piv.assign(n, 0);
  for (int k = 0; k < n; ++k) {
    const int last = std::min(n - 1, k + kl);
    int p = k;
    double best = std::abs(el(k, k));
    for (int i = k + 1; i <= last; ++i)
      if (std::abs(el(i, k)) > best) {
        best = std::abs(el(i, k));
        p = i;
      }
    if (best == 0.0) throw std::runtime_error("banded LU: singular matrix");
    f.piv[k] = p;
    const int jend = std::min(n - 1, k + kl + ku);
    if (p != k)
      for (int j = k; j <= jend; ++j) std::swap(el(k, j), el(p, j));
    const T piv = el(k, k);
    for (int i = k + 1; i <= last; ++i) {
      const T l = el(i, k) / piv;
      f.L[static_cast<size_t>(k) * kl + (i - k - 1)] = l;
      if (l == T(0.0)) continue;
      for (int j = k + 1; j <= jend; ++j) el(i, j) -= l * el(k, j);
    }
    for (int d = 0; d <= f.ku; ++d) {
      const int j = k + d;
      f.U[static_cast<size_t>(k) * (f.ku + 1) + d] = j < n ? el(k, j) : T(0.0);
    }
  }
}

}  // namespace

BandLU band_lu(const Band& S, const Band& M, cplx c, cplx corner) {
  BandLU f;
  band_lu_t<cplx>(S, M, c, corner, f);
  return f;
}

BandLUr band_lu_real(const Band& S, const Band& M, double c) {
  BandLUr f;
  band_lu_t<double>(S, M, c, 0.0, f);
  return f;
}

std::vector<cplx> band_lu_solve(const BandLU& f, std::vector<cplx> b) {
  const int n = f.n;
  for (int k = 0; k < n; ++k) {
    if (f.piv[k] != k) std::swap(b[k], b[f.piv[k]]);
    for (int r = 1; r <= f.kl && k + r < n; ++r) b[k + r] -= f.L[static_cast<size_t>(k) * f.kl + r - 1] * b[k];
  }
  for (int k = n - 1; k >= 0; --k) {
    cplx s = b[k];
    for (int d = 1; d <= f.ku && k + d < n; ++d) s -= f.U[static_cast<size_t>(k) * (f.ku + 1) + d] * b[k + d];
    b[k] = s / f.U[static_cast<size_t>(k) * (f.ku + 1)];
  }
  return b;
}

}  // namespace hd
