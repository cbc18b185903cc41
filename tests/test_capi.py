"""CPU tests of the C-ABI library: it loads, exports every symbol the header
declares, its native host assembly matches the oracle, and the solver fails
loudly (no CPU fallback) when no CUDA device is present."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2010_10232_b200 as hd
from oracle import helmdef_oracle as O

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "helmdef_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hd_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = hd.load_library()
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/helmdef_b200.h but not exported"
    assert sorted(hd.EXPORTS) == syms


def test_library_is_sm100a():
    data = hd.LIB_PATH.read_bytes()
    assert b"sm_100a" in data or b"sm_100" in data


@pytest.mark.parametrize("dim,p,ne,k", [(1, 1, 40, 10.0), (1, 2, 80, 50.0), (1, 5, 33, 7.0), (2, 2, 40, 20.0),
                                        (2, 3, 64, 40.0), (2, 4, 17, 5.0)])
def test_native_assembly_matches_oracle(dim, p, ne, k):
    s = hd.assemble(hd.point_source_2d(ne, p, k) if dim == 2 else hd.point_source_1d(ne, p, k))
    so = O.assemble(O.point_source_2d(ne, p, k) if dim == 2 else O.point_source_1d(ne, p, k))
    n = s.per_dim
    assert n == so.per_dim == ne + p - 2
    S1 = so.S1.toarray() if hasattr(so.S1, "toarray") else so.S1
    M1 = so.M1.toarray() if hasattr(so.M1, "toarray") else so.M1
    Sd, Md = np.zeros((n, n)), np.zeros((n, n))
    for i in range(n):
        for d in range(-p, p + 1):
            if 0 <= i + d < n:
                Sd[i, i + d] = s.stiffness_band[i, d + p]
                Md[i, i + d] = s.mass_band[i, d + p]
    assert np.abs(Sd - S1).max() <= 1e-13 * np.abs(S1).max()
    assert np.abs(Md - M1).max() <= 1e-13 * np.abs(M1).max()
    assert np.abs(s.rhs - so.rhs).max() <= 1e-15


def test_layered_interval_masses_sum_to_mass():
    s = hd.assemble(hd.layered_medium_2d(24, 3, 10.0))
    assert s.interval_mass is not None
    assert np.abs(s.interval_mass.sum(axis=0) - s.mass_band).max() < 1e-14


def test_assemble_rejects_bad_input():
    lib = hd.load_library()
    h = hd.HdProblem()
    h.dim, h.order, h.elements, h.k = 3, 2, 10, 1.0
    z = np.zeros(64)
    st = lib.hd_assemble(C.byref(h), hd._dp(z), hd._dp(z), None, hd._dp(z))
    assert st == 1 and b"dim" in lib.hd_last_error()


def test_solver_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present; the no-device path is exercised on CPU hosts")
    s = hd.assemble(hd.point_source_1d(80, 2, 50.0))
    with pytest.raises(hd.HelmdefError) as e:
        hd.Solver(s, hd.to_spec("DC_MG", 2, 50.0, beta2="0.5", omega=2 / 3))
    assert e.value.status == 4 and "no CPU fallback" in str(e.value)


def test_to_spec_mirrors_reference_mapping():
    s = hd.to_spec("Deps_C_MG", 5, 100.0, epsilon=0.1, beta2="4.2", cycles=12, smoothing=3,
                   omega_by_p={5: 0.5})
    assert (s.deflate, s.drop, s.shift, s.beta2, s.cycles, s.smooth_steps, s.omega) == \
        (True, 0.1, True, 4.2, 12, 3, 0.5)
    assert hd.to_spec("C_ex", 2, 300.0, beta2="1/(3k)").beta2 == 1.0 / 900.0
    assert hd.derived_elements(1000, 0.625, 3) == O.derived_elements(1000, 0.625, 3) == 1598
    with pytest.raises(ValueError):
        hd.to_spec("bogus", 1, 1.0)


@pytest.mark.parametrize("ne,p,k0", [(16, 2, 30.0), (24, 3, 30.0), (40, 3, 60.0), (20, 4, 25.0)])
def test_native_wedge_assembly_matches_oracle(ne, p, k0):
    """BASELINE config-4 wedge (oracle extension): the native K2 stencil and the
    off-centre point load equal the oracle's assembly."""
    s = hd.assemble(hd.wedge_2d(ne, p, k0))
    so = O.assemble(O.wedge_2d(ne, p, k0))
    n, NB = s.per_dim, 2 * p + 1
    K = s.shift_mass_2d.reshape(n, n, NB, NB).transpose(0, 2, 1, 3)
    assert np.abs(K - so.K2_stencil).max() <= 1e-14 * np.abs(so.K2_stencil).max()
    assert np.abs(s.rhs - so.rhs).max() == 0.0 and np.count_nonzero(s.rhs) > 0


def test_wedge_with_equal_layers_is_the_constant_field():
    """Pointwise Gauss sampling of a constant k reproduces k^2 M(x)M exactly
    (the (p+1)-point rule integrates the degree-2p products exactly)."""
    s = O.assemble(O.wedge_2d(24, 3, 17.0, multipliers=[1.0, 1.0, 1.0]))
    c = O.assemble(O.point_source_2d(24, 3, 17.0))
    assert abs(s.shift_mass - c.shift_mass).max() <= 1e-15 * abs(c.shift_mass).max() * 10
    assert abs(s.A - c.A).max() <= 1e-13


def test_wedge_layers():
    """k^2 sampling: the three layers and the strict interfaces."""
    m, ln = O.WEDGE_MULTIPLIERS, O.WEDGE_LINES
    k2 = lambda x, y: float(O.wedge_k2(np.array(x), np.array(y), 10.0, m, ln))
    assert k2(0.5, 0.9) == pytest.approx(144.0)     # top
    assert k2(0.5, 0.45) == pytest.approx(225.0)    # middle (0.35 < y <= 0.5 at x = 0.5)
    assert k2(0.5, 0.1) == pytest.approx(100.0)     # bottom
    assert k2(0.0, 0.6) == pytest.approx(225.0)     # on the top interface: not top
    assert k2(1.0, 0.41) == pytest.approx(144.0)    # right edge, the layers meet at y = 0.4
