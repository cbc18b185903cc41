"""CPU tests of the oracle restatement against the reference's own unit-test
identities (tests/test_precond.cpp, tests/test_linalg.cpp, tests/test_spline.cpp,
tests/test_assembly.cpp of /root/reference/proj).  The oracle is the checker of
the CUDA path, so it is pinned here first."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import helmdef_oracle as O


def rvec(n, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)


# ---- B-splines / assembly (tests/test_spline.cpp, tests/test_assembly.cpp) ----
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_partition_of_unity(p):
    kv = O.KnotVector.open_uniform(7, p)
    for x in np.linspace(0, 1, 23):
        s = sum(O.bspline_value(kv, j, x) for j in range(kv.basis_count()))
        assert abs(s - 1.0) < 1e-13


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_derivative_matches_finite_difference(p):
    kv = O.KnotVector.open_uniform(6, p)
    h = 1e-6
    for j in range(kv.basis_count()):
        for x in [0.13, 0.41, 0.77]:
            fd = (O.bspline_value(kv, j, x + h) - O.bspline_value(kv, j, x - h)) / (2 * h)
            assert abs(fd - O.bspline_derivative(kv, j, x)) < 1e-6 * max(1.0, abs(fd))


def test_gauss_rule_exactness():
    for n in range(1, 7):
        nodes, w = O.gauss_legendre(n)
        for deg in range(2 * n):
            exact = 0.0 if deg % 2 else 2.0 / (deg + 1)
            assert abs(np.sum(w * nodes ** deg) - exact) < 1e-13


def test_forms_symmetric_and_mass_total():
    kv, S, M = O.assemble_forms_1d(12, 3)
    assert np.abs(S - S.T).max() < 1e-13 and np.abs(M - M.T).max() < 1e-15
    assert abs(M.sum() - 1.0) < 1e-13  # partition of unity: sum_ij int phi_i phi_j = 1
    assert np.abs(S.sum(axis=1)).max() < 1e-10  # constants are in the kernel of S


def test_2d_kron_layout():
    s = O.assemble(O.point_source_2d(9, 2, 5.0))
    n = s.per_dim
    S1, M1 = s.S1, s.M1
    A = s.A.toarray()
    iy, ix, jy, jx = 3, 4, 4, 2
    want = M1[iy, jy] * S1[ix, jx] + S1[iy, jy] * M1[ix, jx] - 25.0 * M1[iy, jy] * M1[ix, jx]
    assert abs(A[iy * n + ix, jy * n + jx] - want) < 1e-14


# ---- transfers (tests/test_precond.cpp:51-97) ----
def test_halving_stencil_rows():
    Z = O.halving_stencil(9, 0.1).toarray()
    assert Z.shape == (9, 4)
    assert abs(Z[3, 0] - 1 / 8) < 1e-15 and abs(Z[3, 1] - 5.9 / 8) < 1e-15 and abs(Z[3, 2] - 1 / 8) < 1e-15
    assert abs(Z[2, 0] - 0.5) < 1e-15 and abs(Z[2, 1] - 0.5) < 1e-15
    assert Z[0, 0] == 0.5 and Z[1, 0] == 5.9 / 8 and Z[1, 1] == 1 / 8  # dropped out-of-range entries


def test_linear_stencil_rows():
    Z = O.linear_stencil(9).toarray()
    assert Z.shape == (9, 4)
    assert Z[1, 0] == 1.0 and Z[0, 0] == 0.5 and Z[2, 0] == 0.5 and Z[2, 1] == 0.5 and Z[8, 3] == 0.5


# ---- deflation / multigrid identities (tests/test_precond.cpp:99-218) ----
def test_deflation_projection_identities():
    s = O.assemble(O.point_source_1d(33, 2, 20.0))
    n = s.A.shape[0]
    assert n == 33
    d = O.Deflation(s.A, O.halving_stencil(n, 0.1))
    assert d.coarse_size() == 16
    v = rvec(n, 5)
    qv = d.apply_Q(v)
    assert np.linalg.norm(d.apply_Q(s.A @ qv) - qv) < 1e-10 * np.linalg.norm(qv)
    pw = d.project(v)
    assert np.linalg.norm(d.project(pw) - pw) < 1e-10 * np.linalg.norm(pw)
    zc = d.Z @ rvec(16, 6)
    assert np.linalg.norm(d.project(zc)) < 1e-10 * np.linalg.norm(zc)
    apv = s.A @ d.project(v)
    assert np.linalg.norm(d.ZT @ apv) < 1e-10 * np.linalg.norm(apv)


def test_single_level_multigrid_is_direct_solve():
    s = O.assemble(O.point_source_1d(30, 2, 18.0))
    M = O.shifted_operator(s, 1.0)
    mg = O.Multigrid(M, s.A.shape[0], 1)
    assert mg.levels() == 1
    b = rvec(M.shape[0], 9)
    x = mg.solve(b, 1)
    assert np.linalg.norm(M @ x - b) / np.linalg.norm(b) < 1e-12


def test_two_level_cycle_matches_explicit_propagator():
    s = O.assemble(O.point_source_1d(63, 2, 25.0))
    n = s.A.shape[0]
    M = O.shifted_operator(s, 1.0)
    mg = O.Multigrid(M, n, 1, omega=0.6, smooth_steps=2)
    assert mg.levels() == 2
    Md = M.toarray()
    Z = mg.trans[0].toarray()
    M2 = mg.mats[1].toarray()
    S = np.eye(n) - 0.6 * np.diag(1 / np.diag(Md)) @ Md
    Snu = S @ S
    prop = Snu @ (np.eye(n) - Z @ np.linalg.solve(M2, Z.T @ Md)) @ Snu
    b, x0 = rvec(n, 13), rvec(n, 14)
    exact = np.linalg.solve(Md, b)
    x1 = mg.vcycle(b, x0)
    assert np.linalg.norm(x1 - (exact + prop @ (x0 - exact))) < 1e-11 * np.linalg.norm(x0 - exact)


def test_zero_smoothing_is_identity():
    s = O.assemble(O.point_source_1d(20, 2, 10.0))
    mg = O.Multigrid(O.shifted_operator(s, 1.0), s.A.shape[0], 1)
    x = rvec(s.A.shape[0], 18)
    assert np.array_equal(mg.smooth(0, rvec(s.A.shape[0], 17), x, 0), x)


def test_shift_algebra():
    s = O.assemble(O.point_source_1d(24, 3, 14.0))
    assert abs(O.shifted_operator(s, 0.0) - s.A).max() < 1e-14
    diff = (O.shifted_operator(s, 2.5) - s.A).toarray()
    assert np.abs(diff - 2.5j * s.shift_mass.toarray()).max() < 1e-12


def test_composed_deflated_operator_annihilates_coarse_range():
    s = O.assemble(O.point_source_1d(33, 2, 21.0))
    st = O.compose(s, O.PrecondSpec(deflate=True, drop=0.1))
    w = st.op(rvec(33, 29))
    aw = s.A @ w
    assert np.linalg.norm(st.deflation.ZT @ aw) < 1e-10 * np.linalg.norm(aw)
    assert np.isfinite(st.monitor(st.start))


@pytest.mark.parametrize("cycles", [1, 10])
def test_composed_solve_matches_direct(cycles):
    s = O.assemble(O.point_source_1d(159, 2, 100.0))
    st = O.compose(s, O.PrecondSpec(deflate=True, drop=0.1, shift=True, beta2=1.0, cycles=cycles))
    r = O.gmres(st.op, st.rhs, st.start, st.monitor)
    assert r.converged
    ref = O.DirectSolver(s.A).solve(s.rhs)
    assert np.linalg.norm(r.solution - ref) / np.linalg.norm(ref) < 1e-6
    assert st.counts.vcycles == cycles * st.counts.shift_solves
    # counters: matvecs = it+1, shift_solves = it+2, coarse_solves = it+3
    assert (st.counts.matvecs, st.counts.shift_solves, st.counts.coarse_solves) == \
        (r.iterations + 1, r.iterations + 2, r.iterations + 3)


def test_2d_kronecker_deflation_and_solve():
    s = O.assemble(O.point_source_2d(17, 2, 10.0))
    assert s.per_dim == 17
    st = O.compose(s, O.PrecondSpec(deflate=True, drop=0.1))
    z1 = O.halving_stencil(17, 0.1)
    assert abs(st.deflation.Z - O.kron_real(z1, z1)).max() < 1e-13
    r = O.gmres(st.op, st.rhs, st.start, st.monitor)
    assert r.converged
    ref = O.DirectSolver(s.A).solve(s.rhs)
    assert np.linalg.norm(r.solution - ref) / np.linalg.norm(ref) < 1e-6


# ---- GMRES (tests/test_linalg.cpp:40-108) ----
def test_gmres_random_systems_match_lu():
    for seed in range(101, 106):
        rng = np.random.default_rng(seed)
        n = 40
        A = np.eye(n) * 4 + (rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))) / 4
        b = rvec(n, seed + 50)
        r = O.gmres(lambda v: A @ v, b, np.zeros(n, complex),
                    lambda x: np.linalg.norm(b - A @ x) / np.linalg.norm(b), O.GmresOptions(100, 1e-10))
        assert r.converged and len(r.residuals) == r.iterations
        assert np.linalg.norm(r.solution - np.linalg.solve(A, b)) / np.linalg.norm(b) < 1e-8


def test_gmres_converged_start_takes_zero_iterations():
    A = np.diag(np.arange(1.0, 6.0)).astype(complex)
    b = rvec(5, 3)
    x = np.linalg.solve(A, b)
    r = O.gmres(lambda v: A @ v, b, x, lambda y: np.linalg.norm(b - A @ y) / np.linalg.norm(b))
    assert r.converged and r.iterations == 0 and len(r.residuals) == 1


def test_gmres_budget_and_generator_identity():
    s = O.assemble(O.point_source_1d(80, 2, 50.0))
    st = O.compose(s, O.to_spec("DC_MG", 2, 50.0, beta2="0.5", omega=2 / 3))
    full = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(3, 1e-7))
    assert full.iterations == 3 and not full.converged
    st2 = O.compose(s, O.to_spec("DC_MG", 2, 50.0, beta2="0.5", omega=2 / 3))
    part = O.gmres(st2.op, st2.rhs, st2.start, st2.monitor, O.GmresOptions(100, 1e-7), max_steps=3)
    assert part.residuals == full.residuals


# ---- oracle variants used for large configs ----
def test_kron_galerkin_equals_sparse_galerkin():
    s = O.assemble(O.point_source_2d(80, 3, 30.0))
    spec = O.to_spec("DC_MG", 3, 30.0, beta2="0.5", omega=2 / 3)
    a = O.compose(s, spec, galerkin="sparse")
    b = O.compose(s, spec, galerkin="kron")
    for ma, mb in zip(a.multigrid.mats, b.multigrid.mats):
        assert abs(ma - mb).max() < 1e-12 * abs(ma).max()


def test_fd_coarse_solve_matches_splu():
    s = O.assemble(O.point_source_2d(64, 2, 40.0))
    spec = O.to_spec("DC_MG", 2, 40.0, beta2="0.5", omega=2 / 3)
    a = O.compose(s, spec, e_solver="splu")
    b = O.compose(s, spec, e_solver="fd")
    v = rvec(s.A.shape[0], 3)
    qa, qb = a.deflation.apply_Q(v), b.deflation.apply_Q(v)
    assert np.linalg.norm(qa - qb) < 1e-10 * np.linalg.norm(qa)


def test_c_spmv_bit_identical_to_scipy():
    """oracle/csr_spmv.c (the oracle's threaded product for the live C5 run) must
    round exactly like scipy's csr_matvec, for any thread count."""
    if not O.use_c_spmv(3):
        pytest.skip("oracle/libcsr_spmv.so not built")
    try:
        s = O.assemble(O.point_source_2d(60, 3, 30.0))
        A = sp.csr_matrix(O.shifted_operator(s, 0.5))
        A.sort_indices()
        rng = np.random.default_rng(7)
        x = rng.uniform(-1, 1, A.shape[0]) + 1j * rng.uniform(-1, 1, A.shape[0])
        for t in (1, 3, 8):
            O.use_c_spmv(t)
            assert np.array_equal(O._mv(A, x), A @ x)
        B = sp.random(3000, 2000, density=0.01, format="csr", random_state=3).astype(np.complex128)
        B.data = B.data + 1j * rng.uniform(-1, 1, B.nnz)
        B.sort_indices()
        y = rng.uniform(-1, 1, 2000) + 1j * rng.uniform(-1, 1, 2000)
        assert np.array_equal(O._mv(B, y), B @ y)
    finally:
        O._SPMV["lib"] = None
