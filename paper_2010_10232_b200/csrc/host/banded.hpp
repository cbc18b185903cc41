// Host-side 1D banded algebra for the solver setup: the Galerkin hierarchy of
// 1D factors, the Bezier/linear transfer stencils and a banded complex LU.
//
// The reference forms every coarse operator as an Eigen sparse triple product
// Z^T M Z on the full (2D) matrix (src/precond.cpp:95, :119).  For the
// Kronecker-sum operators of this path that product factorises exactly:
// (z (x) z)^T (a (x) b) (z (x) z) = (z^T a z) (x) (z^T b z), so only 1D banded
// factors are formed here and the device applies the Kronecker structure.
#pragma once

#include <complex>
#include <stdexcept>
#include <vector>

namespace hd {

using cplx = std::complex<double>;

/// Real banded n x n matrix, half-bandwidth b, row-major band storage:
/// a[i*(2b+1) + (j-i+b)] = A(i,j) for |i-j| <= b, zero elsewhere.
struct Band {
  int n = 0;
  int b = 0;
  std::vector<double> a;
  Band() = default;
  Band(int n_, int b_) : n(n_), b(b_), a(static_cast<size_t>(n_) * (2 * b_ + 1), 0.0) {}
  double at(int i, int j) const {
    const int d = j - i;
    if (d < -b || d > b || i < 0 || i >= n || j < 0 || j >= n) return 0.0;
    return a[static_cast<size_t>(i) * (2 * b + 1) + (d + b)];
  }
  double& ref(int i, int j) { return a[static_cast<size_t>(i) * (2 * b + 1) + (j - i + b)]; }
  /// Smallest half-bandwidth holding every nonzero.
  Band trimmed() const;
};

/// Sparse 1D transfer Z (fine x coarse) in coordinate form.
struct Transfer {
  int fine = 0, coarse = 0;
  std::vector<int> row, col;
  std::vector<double> w;
};

/// Quadratic-Bezier two-level stencil, src/precond.cpp:34-55 (1-based j, c;
/// even j: 1/8 (1, 6-drop, 1) on c = (j-2)/2, j/2, (j+2)/2; odd j: 1/2 (1,1) on
/// c = (j-1)/2, (j+1)/2; out-of-range entries dropped without renormalising).
Transfer halving_stencil(int fine, double drop);

/// Linear-interpolation multigrid stencil, src/precond.cpp:57-76.
Transfer linear_stencil(int fine);

/// Galerkin product z^T A z of a banded matrix with a 1D transfer.
Band galerkin(const Band& A, const Transfer& z);

/// Banded complex LU with partial pivoting (LAPACK gbtrf layout semantics):
/// L has kl subdiagonals (unit, stored as multipliers), U has kl+ku
/// superdiagonals after row interchanges.  Exact direct solve used for the 1D
/// deflation matrix E and the coarsest 1D multigrid level, standing in for the
/// reference's Eigen::SparseLU (src/linalg.cpp:94-102, src/precond.cpp:95-99).
struct BandLU {
  int n = 0, kl = 0, ku = 0;      // ku of the factor U (= kl + ku of the input)
  std::vector<cplx> L;            // n x kl multipliers: L[i*kl + (r-1)] = l(i+r, i)
  std::vector<cplx> U;            // n x (ku+1): U[i*(ku+1) + d] = u(i, i+d)
  std::vector<int> piv;           // row interchanged with i at step i
};

/// Factor the complex banded matrix (S - c M) (+ corner at (n-1,n-1)).
BandLU band_lu(const Band& S, const Band& M, cplx c, cplx corner = cplx(0.0, 0.0));

/// The same factorisation in real arithmetic (real S - c M).
struct BandLUr {
  int n = 0, kl = 0, ku = 0;
  std::vector<double> L, U;
  std::vector<int> piv;
};
BandLUr band_lu_real(const Band& S, const Band& M, double c);

/// Reference host solve (used by the unit test of the factorisation only).
std::vector<cplx> band_lu_solve(const BandLU& f, std::vector<cplx> b);

}  // namespace hd
