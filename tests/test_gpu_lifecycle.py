"""Context lifecycle and error behaviour of the C-ABI on a GPU: no device
memory is leaked by create / solve / destroy cycles, contexts do not share
state, and bad input fails loudly with the documented status instead of
producing numbers (the reference throws std::runtime_error / returns
converged = false in the same places: src/linalg.cpp:10-25)."""
import numpy as np
import pytest

import paper_2010_10232_b200 as hd

pytestmark = pytest.mark.gpu
BASE = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)


def _free_bytes():
    import torch
    torch.cuda.synchronize()
    return torch.cuda.mem_get_info()[0]


@pytest.mark.parametrize("make,tag,p,k", [
    (lambda: hd.point_source_2d(96, 3, 60.0), "DC_MG", 3, 60.0),
    (lambda: hd.point_source_1d(4000, 3, 200.0), "DC_MG", 3, 200.0),
    (lambda: hd.wedge_2d(64, 3, 20.0), "DC_MG", 3, 20.0),
    (lambda: hd.layered_medium_2d(48, 2, 30.0), "C_ex", 2, 30.0),
])
def test_create_solve_destroy_does_not_leak_device_memory(make, tag, p, k):
    s = hd.assemble(make())
    spec = hd.to_spec(tag, p, k, **(BASE if tag != "C_ex" else dict(beta2="1/k")))
    with hd.Solver(s, spec) as solver:  # first cycle: library handles and module loading settle
        solver.solve(hd.GmresOptions(60, 1e-7))
    before = _free_bytes()
    for _ in range(5):
        with hd.Solver(s, spec) as solver:
            solver.solve(hd.GmresOptions(60, 1e-7))
            solver.solve(hd.GmresOptions(140, 1e-7))  # reallocates the Krylov buffers (exact-order MGS engine)
    after = _free_bytes()
    assert before - after <= 8 << 20, f"{(before - after) / 2**20:.1f} MiB not returned after 5 cycles"


def test_contexts_do_not_share_state():
    """Two contexts alive at once, solved alternately, give the bits each gives alone."""
    sa = hd.assemble(hd.point_source_2d(96, 3, 60.0))
    sb = hd.assemble(hd.point_source_2d(64, 2, 40.0))
    spa, spb = hd.to_spec("DC_MG", 3, 60.0, **BASE), hd.to_spec("DC_MG", 2, 40.0, **BASE)
    opt = hd.GmresOptions(100, 1e-7)
    with hd.Solver(sa, spa) as a:
        ra = a.solve(opt)
    with hd.Solver(sb, spb) as b:
        rb = b.solve(opt)
    with hd.Solver(sa, spa) as a, hd.Solver(sb, spb) as b:
        for _ in range(2):
            xa, xb = a.solve(opt), b.solve(opt)
            assert np.array_equal(xa.solution, ra.solution) and xa.residuals == ra.residuals
            assert np.array_equal(xb.solution, rb.solution) and xb.residuals == rb.residuals


def test_non_finite_right_hand_side_is_an_error():
    s = hd.assemble(hd.point_source_2d(64, 3, 40.0))
    rhs = s.rhs.copy()
    rhs[rhs.size // 2] = np.nan
    with hd.Solver(s, hd.to_spec("DC_MG", 3, 40.0, **BASE)) as solver:
        with pytest.raises(hd.HelmdefError) as e:
            solver.solve(hd.GmresOptions(50, 1e-7), rhs=rhs)
        assert e.value.status == hd.HD_ERR_NONFINITE
        # the context is still usable afterwards
        r = solver.solve(hd.GmresOptions(100, 1e-7))
        assert r.converged


def test_budget_and_tolerance_edge_cases():
    s = hd.assemble(hd.point_source_2d(64, 3, 40.0))
    with hd.Solver(s, hd.to_spec("DC_MG", 3, 40.0, **BASE)) as solver:
        full = solver.solve(hd.GmresOptions(100, 1e-7))
        # a budget below the converged count: not converged, exactly `budget` iterations, the same history prefix
        short = solver.solve(hd.GmresOptions(3, 1e-7))
        assert not short.converged and short.iterations == 3
        assert np.allclose(short.residuals, full.residuals[:3], rtol=0, atol=1e-12)
        # a tolerance the start vector already meets: zero or one monitored step, converged
        loose = solver.solve(hd.GmresOptions(100, 1e3))
        assert loose.converged and loose.iterations <= 1
        with pytest.raises(hd.HelmdefError) as e:
            solver.solve(hd.GmresOptions(-1, 1e-7))
        assert e.value.status == hd.HD_ERR_INVALID
