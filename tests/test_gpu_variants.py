"""GPU checks of the round-1 fast paths against the paths they replace (same
library, switched at context creation), so each optimisation is shown not to
move results beyond rounding:

  * the first Jacobi sweep of a V-cycle level taken by the kernel that produces
    its right-hand side (OP_APPLYJ0 / k_restrict2d J0) vs the separate
    k_jacobi0_2d_t launch (HD_NOJ0FUSE=1);
  * the two-level segment scans of the 1D banded solves (k_seg_scan2) vs the
    P-step single-warp scans (HD_SEG_SEQSCAN=1);
  * the reflection-folded E solve at C5, whose factors are centro-symmetric to
    3e-13 only, vs the unfolded fast diagonalisation (HD_NOFOLD=1).

Each pair is also tied to the oracle by tests/test_gpu_parity.py (the default
paths) -- these tests bound the distance between the two device paths.
"""
import numpy as np
import pytest

import paper_2010_10232_b200 as hd

pytestmark = pytest.mark.gpu
BASE = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)


def _apply(solver, which, x):
    import torch
    xd = torch.from_numpy(x).cuda()
    yd = torch.zeros_like(xd)
    solver.apply(which, xd.data_ptr(), yd.data_ptr())
    torch.cuda.synchronize()
    return yd.cpu().numpy()


def _rand(n, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)


def _pair(monkeypatch, var, s, spec):
    """(default solver, solver created with the environment switch `var` set)"""
    monkeypatch.delenv(var, raising=False)
    a = hd.Solver(s, spec)
    monkeypatch.setenv(var, "1")
    b = hd.Solver(s, spec)
    monkeypatch.delenv(var, raising=False)
    return a, b


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _same_solve(ra, rb, sol_tol):
    """Equal iterations and flags, solutions within sol_tol, the last five
    history entries within the spec's 1e-10.  Earlier entries are held to 1e-2
    relative only: some cases pass a transient where the true residual amplifies
    rounding-level differences ~1e3x per step and then recovers (the p = 3,
    ne = 130 case: 1e-13 at step 3, ~5e-6 at steps 6-7, 1e-16 from step 10 on).
    The same path, run after different earlier work in the process, was seen to
    differ there by the same order; it is the phenomenon of C5's stagnation
    phase."""
    assert ra.iterations == rb.iterations and ra.converged == rb.converged
    ha, hb = np.array(ra.residuals), np.array(rb.residuals)
    assert np.all(np.abs(ha - hb) <= 1e-2 * hb)
    assert np.max(np.abs(ha[-5:] - hb[-5:])) <= 1e-10
    assert _rel(ra.solution, rb.solution) <= sol_tol


@pytest.mark.parametrize("ne,p,k", [(96, 2, 60.0), (130, 3, 80.0), (64, 4, 40.0)])
def test_fused_first_sweep_matches_separate_launch(monkeypatch, ne, p, k):
    s = hd.assemble(hd.point_source_2d(ne, p, k))
    a, b = _pair(monkeypatch, "HD_NOJ0FUSE", s, hd.to_spec("DC_MG", p, k, **BASE))
    with a, b:
        x = _rand(s.size, 11)
        for which in (hd.HD_APPLY_MG, hd.HD_APPLY_OP):
            assert _rel(_apply(a, which, x), _apply(b, which, x)) <= 1e-13
        ra, rb = a.solve(hd.GmresOptions(100, 1e-7)), b.solve(hd.GmresOptions(100, 1e-7))
    _same_solve(ra, rb, 1e-11)


@pytest.mark.parametrize("ne,p,k", [(31623, 4, 1000.0), (6000, 3, 300.0), (4000, 2, 200.0)])
def test_two_level_scan_matches_sequential_scan(monkeypatch, ne, p, k):
    s = hd.assemble(hd.point_source_1d(ne, p, k))
    a, b = _pair(monkeypatch, "HD_SEG_SEQSCAN", s, hd.to_spec("DC_MG", p, k, **BASE))
    with a, b:
        x = _rand(s.size, 12)
        # Q = Z E^-1 Z^T: the deflation solve is the segmented banded LU
        assert _rel(_apply(a, hd.HD_APPLY_Q, x), _apply(b, hd.HD_APPLY_Q, x)) <= 1e-12
        ra, rb = a.solve(hd.GmresOptions(100, 1e-7)), b.solve(hd.GmresOptions(100, 1e-7))
    _same_solve(ra, rb, 1e-9)


def test_folded_E_at_C5_matches_unfolded(monkeypatch):
    """C5's E factors are centro-symmetric to ~3e-13 relative, inside the 1e-12
    tolerance: the folded solve applies the inverse of the symmetrised E.  Its
    distance to the unfolded fast diagonalisation is held to 1e-8 per deflation
    application (the solution bar); measured 9e-12 on B200, below the unfolded
    FD's own distance to SuperLU at cond(E) ~ 5e5."""
    s = hd.assemble(hd.point_source_2d(1600, 3, 1000.0))
    a, b = _pair(monkeypatch, "HD_NOFOLD", s, hd.to_spec("DC_MG", 3, 1000.0, **BASE))
    with a, b:
        for seed in (13, 14):
            x = _rand(s.size, seed)
            d = _rel(_apply(a, hd.HD_APPLY_Q, x), _apply(b, hd.HD_APPLY_Q, x))
            print(f"folded vs unfolded Q at C5: {d:.2e}")
            assert d <= 1e-8
