"""Generates the committed golden fixtures of tests/golden/ from the CPU oracle.

Run from the repo root:  python tests/golden/make_golden.py
Each case stores the oracle's GmresResult (iterations, converged, residual
history, solution) and OperationCounts for a BASELINE-parameterised cell small
enough to commit; tests/test_gpu_parity.py checks the CUDA path against them.
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import helmdef_oracle as O  # noqa: E402

OUT = Path(__file__).resolve().parent
BASE = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)

# name: (problem, p, elements, k, tag, spec overrides)
CASES = {
    "C1": ("point_source_1d", 2, 80, 50.0, "DC_MG", {}),
    "C1_eps": ("point_source_1d", 2, 80, 50.0, "Deps_C_MG", {"epsilon": 0.1}),
    "1d_p4_k200": ("point_source_1d", 4, 317, 200.0, "DC_MG", {}),
    "1d_p1_k100_nu2c3": ("point_source_1d", 1, 160, 100.0, "DC_MG", {"smoothing": 2, "cycles": 3}),
    "1d_p5_k100_t4": ("point_source_1d", 5, 156, 100.0, "Deps_C_MG", {"beta2": "1", "omega": 0.6, "epsilon": 0.1}),
    "2d_p2_k20": ("point_source_2d", 2, 40, 20.0, "DC_MG", {}),
    "2d_p3_k40": ("point_source_2d", 3, 64, 40.0, "DC_MG", {}),
    "2d_p1_k20_D": ("point_source_2d", 1, 33, 20.0, "D", {}),
    "2d_p4_k30_eps_nu3": ("point_source_2d", 4, 45, 30.0, "Deps_C_MG",
                          {"epsilon": 0.1, "smoothing": 3, "beta2": "4.2", "omega": 0.6}),
    "2d_p5_k25_t5": ("point_source_2d", 5, 36, 25.0, "DC_MG", {"smoothing": 3, "beta2": "4.2", "omega": 0.5}),
    # exact shifted inverse (C_ex) cells of the reference tables (table3 1D, table5 2D)
    "1d_p3_k1000_Cex": ("point_source_1d", 3, 1598, 1000.0, "C_ex", {"beta2": "1/k"}),
    "2d_p2_k50_Cex": ("point_source_2d", 2, 79, 50.0, "C_ex", {"beta2": "1/(3k)"}),
    "2d_p3_k50_D_eps": ("point_source_2d", 3, 78, 50.0, "D_eps", {"epsilon": 0.1}),
}


def run(name):
    problem, p, ne, k, tag, over = CASES[name]
    kw = dict(BASE)
    kw.update(over)
    spec = O.to_spec(tag, p, k, **kw)
    pb = O.make_problem(problem, ne, p, k)
    s = O.assemble(pb)
    two_d = s.dim == 2
    st = O.compose(s, spec, galerkin="kron" if two_d else "sparse", e_solver="fd" if two_d else "splu")
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
    meta = dict(problem=problem, p=p, elements=ne, k=k, tag=tag, spec=kw, iterations=g.iterations,
                converged=g.converged, residuals=g.residuals,
                counts=dict(matvecs=st.counts.matvecs, coarse_solves=st.counts.coarse_solves,
                            shift_solves=st.counts.shift_solves, vcycles=st.counts.vcycles),
                oracle_mode=dict(galerkin="kron" if two_d else "sparse", e_solver="fd" if two_d else "splu"))
    np.savez_compressed(OUT / f"{name}.npz", solution=g.solution, meta=json.dumps(meta))
    return meta


if __name__ == "__main__":
    for n in sys.argv[1:] or CASES:
        m = run(n)
        print(n, m["iterations"], m["converged"], m["counts"])
