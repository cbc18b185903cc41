"""The C++ host mirror of the reference API (include/helmdef_b200.hpp) through
its cell tool (tools/hd_cell, built by __graft_entry__.build()).

CPU: host assembly agrees with the oracle, and a solve without a GPU fails
loudly (no CPU fallback).  GPU: run_cell through the C++ API matches the
oracle's solve (iterations, counts, residual history 1e-10, |x|)."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import helmdef_oracle as O

ROOT = Path(__file__).resolve().parents[1]
TOOL = ROOT / "tools" / "hd_cell"


def _run(*args, check=True):
    p = subprocess.run([str(TOOL), *map(str, args)], capture_output=True, text=True, timeout=600)
    if check:
        assert p.returncode == 0, p.stderr
    return p


def _have_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def test_tool_built():
    assert TOOL.exists(), "run __graft_entry__.build()"


@pytest.mark.parametrize("problem,p,k,ne", [("point_source_1d", 2, 50.0, 80), ("point_source_2d", 3, 40.0, 64),
                                            ("layered_medium_2d", 2, 50.0, 79), ("wedge_2d", 3, 30.0, 40)])
def test_cpp_assembly_matches_oracle(problem, p, k, ne):
    d = json.loads(_run("--assemble", problem, p, k, ne).stdout)
    so = O.assemble(O.make_problem(problem, ne, p, k))
    assert d["per_dim"] == so.per_dim and d["size"] == so.rhs.size
    assert abs(d["rhs_norm"] - np.linalg.norm(so.rhs)) <= 1e-14 * np.linalg.norm(so.rhs)
    S1 = so.S1.toarray() if hasattr(so.S1, "toarray") else np.asarray(so.S1)
    M1 = so.M1.toarray() if hasattr(so.M1, "toarray") else np.asarray(so.M1)
    assert abs(d["stiffness_sum"] - S1.sum()) <= 1e-12 * abs(S1).sum()
    assert abs(d["mass_sum"] - M1.sum()) <= 1e-12 * abs(M1).sum()
    if problem == "wedge_2d":
        k2 = so.shift_mass.real
        assert abs(d["shift_mass_sum"] - k2.sum()) <= 1e-12 * abs(k2).sum()


def test_cpp_solve_fails_loudly_without_gpu():
    if _have_gpu():
        pytest.skip("a GPU is present")
    p = _run("point_source_1d", "DC_MG", 2, 50.0, 80, "0.5", 1, 1, 2.0 / 3.0, check=False)
    assert p.returncode == 2 and "no CUDA device" in p.stderr


def test_cpp_bad_tag_is_an_error():
    p = _run("point_source_1d", "XX", 2, 50.0, 80, check=False)
    assert p.returncode == 2 and "unknown preconditioner tag" in p.stderr


CELLS = [
    ("point_source_1d", "DC_MG", 2, 50.0, 80, dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)),
    ("point_source_2d", "DC_MG", 3, 40.0, 64, dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)),
    ("point_source_2d", "Deps_C_MG", 2, 30.0, 48, dict(beta2="1", cycles=2, smoothing=2, omega=0.6, epsilon=0.1)),
    ("layered_medium_2d", "DC_MG", 2, 50.0, 79, dict(beta2="4.2", cycles=12, smoothing=3, omega=0.6)),
    ("layered_medium_2d", "C_ex", 3, 50.0, 78, dict(beta2="1/(3k)", cycles=1, smoothing=1, omega=0.6)),
    ("wedge_2d", "DC_MG", 3, 40.0, 64, dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)),
]


@pytest.mark.gpu
@pytest.mark.parametrize("problem,tag,p,k,ne,kw", CELLS)
def test_cpp_run_cell_matches_oracle(problem, tag, p, k, ne, kw):
    args = [problem, tag, p, k, ne, kw["beta2"], kw["cycles"], kw["smoothing"], kw["omega"], 100, 1e-7,
            kw.get("epsilon", 0.1)]
    d = json.loads(_run(*args).stdout.strip().splitlines()[-1])
    so = O.assemble(O.make_problem(problem, ne, p, k))
    two_d_const = so.dim == 2 and so.separable
    st = O.compose(so, O.to_spec(tag, p, k, **kw), galerkin="kron" if two_d_const else "sparse",
                   e_solver="fd" if two_d_const else "splu")
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
    assert d["iterations"] == g.iterations and d["converged"] == g.converged
    assert (d["matvecs"], d["coarse_solves"], d["shift_solves"], d["vcycles"]) == \
        (st.counts.matvecs, st.counts.coarse_solves, st.counts.shift_solves, st.counts.vcycles)
    m = min(len(d["residuals"]), len(g.residuals))
    assert np.max(np.abs(np.array(d["residuals"][:m]) - np.array(g.residuals[:m]))) <= 1e-10
    xn = np.linalg.norm(g.solution)
    assert abs(d["solution_norm"] - xn) <= 1e-8 * xn
    assert d["tag"] == O.label(tag, kw["cycles"])
