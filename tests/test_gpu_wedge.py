"""GPU parity of the wedge field (BASELINE config 4, C4) against the oracle.

The wedge is an oracle extension (oracle/helmdef_oracle.py wedge_2d): the
reference's WaveField cannot express it, so parity is pinned
by the restatement, which runs the reference's own sparse algorithm on the
assembled matrices (Galerkin triple products, SuperLU for E and the coarsest
level).  The device path: Kronecker-sum part + stored K2 stencil planes on
every level (layered.cuh), dense inverse of the coarsest level, and E by the
dense inverse (small) or the block tridiagonal LU (btri.cuh; forced here with
HD_BTRI=1, the default beyond 20000 unknowns as at C4).

Bars as for the other configs: iterations equal, residual
history within 1e-10 on every common step, solution within 1e-8 relative,
identical converged flag and OperationCounts.
"""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2010_10232_b200 as hd
from oracle import helmdef_oracle as O

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
BASE = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)


def _oracle(ne, p, k0, kw):
    so = O.assemble(O.wedge_2d(ne, p, k0))
    return so, O.compose(so, O.to_spec("DC_MG", p, k0, **kw))


@pytest.mark.parametrize("btri", [0, 1])
@pytest.mark.parametrize("p,ne,k0,kw", [(2, 40, 20.0, BASE), (3, 64, 30.0, BASE),
                                        (3, 48, 25.0, dict(BASE, cycles=2, smoothing=2))])
def test_wedge_components_match_oracle(p, ne, k0, kw, btri, monkeypatch):
    import torch
    monkeypatch.setenv("HD_BTRI", str(btri))
    so, st = _oracle(ne, p, k0, kw)
    s = hd.assemble(hd.wedge_2d(ne, p, k0))
    spec = hd.to_spec("DC_MG", p, k0, **kw)
    rng = np.random.default_rng(7)
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


@pytest.mark.parametrize("btri", [0, 1])
@pytest.mark.parametrize("p,ne,k0", [(2, 64, 40.0), (3, 96, 50.0), (4, 80, 40.0)])
def test_wedge_live(p, ne, k0, btri, monkeypatch):
    """Small wedges solved by the oracle (the reference's sparse algorithm) and
    the device: iterations, counts, history <= 1e-10, solution <= 1e-8."""
    monkeypatch.setenv("HD_BTRI", str(btri))
    so, st = _oracle(ne, p, k0, BASE)
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
    s = hd.assemble(hd.wedge_2d(ne, p, k0))
    with hd.Solver(s, hd.to_spec("DC_MG", p, k0, **BASE)) as solver:
        r = solver.solve(hd.GmresOptions(100, 1e-7))
        r2 = solver.solve(hd.GmresOptions(100, 1e-7))
    assert np.array_equal(r.solution, r2.solution), "device solve must be deterministic"
    assert r.converged == g.converged and r.iterations == g.iterations
    d = np.abs(np.array(r.residuals) - np.array(g.residuals))
    assert d.max() <= 1e-10, (d.max(), int(np.argmax(d)))
    rel = np.linalg.norm(r.solution - g.solution) / np.linalg.norm(g.solution)
    assert rel <= 1e-8, rel
    c = st.counts
    assert (r.counts.matvecs, r.counts.coarse_solves, r.counts.shift_solves, r.counts.vcycles) == \
        (c.matvecs, c.coarse_solves, c.shift_solves, c.vcycles)


def _wedge_apply(s, x):
    """A x = (M (x) S + S (x) M) x - K2 x on the host from the assembled bands and
    the K2 stencil (independent of the device)."""
    n, p = s.per_dim, s.problem.order
    NB = 2 * p + 1
    X = x.reshape(n, n)

    def band_apply(B, V):  # rows of B act along axis 0
        out = np.zeros_like(V)
        for d in range(-p, p + 1):
            lo, hi = max(0, -d), min(n, n - d)
            out[lo:hi] += B[lo:hi, d + p][:, None] * V[lo + d:hi + d]
        return out

    S, M = s.stiffness_band, s.mass_band
    lap = band_apply(M, band_apply(S, X.T).T) + band_apply(S, band_apply(M, X.T).T)
    K = s.shift_mass_2d.reshape(n, n, NB, NB)
    Xp = np.zeros((n + 2 * p, n + 2 * p), complex)
    Xp[p:p + n, p:p + n] = X
    kx = np.zeros_like(X)
    for dy in range(NB):
        for dx in range(NB):
            kx += K[:, :, dy, dx] * Xp[dy:dy + n, dx:dx + n]
    return (lap - kx).reshape(-1)


def test_C4_full_size_wedge():
    """C4: the BASELINE config-4 wedge (k0 = 150, p = 3, 480^2 elements, source at
    (0.5, 1 - h); E = 57,600 unknowns by the block tridiagonal LU) against the
    committed oracle run (tests/golden/make_c4.py, the reference's sparse
    algorithm with SuperLU), plus the true residual of the returned x."""
    ref = json.loads((GOLD / "C4_oracle.json").read_text())
    s = hd.assemble(hd.wedge_2d(480, 3, 150.0))
    with hd.Solver(s, hd.to_spec("DC_MG", 3, 150.0, **BASE)) as solver:
        r = solver.solve(hd.GmresOptions(100, 1e-7))
    assert r.converged == ref["converged"] and r.iterations == ref["iterations"]
    d = np.abs(np.array(r.residuals) - np.array(ref["residuals"][:len(r.residuals)]))
    assert d.max() <= 1e-10, (d.max(), int(np.argmax(d)))
    c = ref["counts"]
    assert (r.counts.matvecs, r.counts.coarse_solves, r.counts.shift_solves, r.counts.vcycles) == \
        (c["matvecs"], c["coarse_solves"], c["shift_solves"], c["vcycles"])
    true = np.linalg.norm(s.rhs - _wedge_apply(s, r.solution)) / np.linalg.norm(s.rhs)
    assert abs(true - r.residuals[-1]) <= 1e-12 and true <= 1e-7
    rng = np.random.default_rng(2024)
    for re_, im_ in ref["projections"]:
        w = rng.uniform(-1, 1, r.solution.size) + 1j * rng.uniform(-1, 1, r.solution.size)
        got = np.vdot(w, r.solution)
        assert abs(got - complex(re_, im_)) <= 1e-8 * abs(complex(re_, im_))
    assert abs(np.linalg.norm(r.solution) - ref["solution_norm"]) <= 1e-8 * ref["solution_norm"]


@pytest.mark.parametrize("btri", [0, 1])
def test_wedge_cex_live(btri, monkeypatch):
    """C_ex on the wedge: the exact shifted inverse by the dense inverse or the
    complex block tridiagonal LU, against the oracle (SuperLU)."""
    monkeypatch.setenv("HD_BTRI", str(btri))
    ne, p, k0 = 48, 3, 25.0
    so = O.assemble(O.wedge_2d(ne, p, k0))
    st = O.compose(so, O.to_spec("C_ex", p, k0, beta2="0.5"))
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
    s = hd.assemble(hd.wedge_2d(ne, p, k0))
    with hd.Solver(s, hd.to_spec("C_ex", p, k0, beta2="0.5")) as solver:
        r = solver.solve(hd.GmresOptions(100, 1e-7))
    assert r.converged == g.converged and r.iterations == g.iterations
    assert np.max(np.abs(np.array(r.residuals) - np.array(g.residuals))) <= 1e-10
    assert np.linalg.norm(r.solution - g.solution) <= 1e-8 * np.linalg.norm(g.solution)
