"""Oracle reference for the full-size C5 config (2D, k=1000, p=3, 1600^2
elements, DC_MG^1, beta2=0.5, omega=2/3): iteration count, converged flag,
residual history and seeded projections of the solution.  Takes ~8 minutes
on one CPU core (E solved by fast diagonalisation, Galerkin levels from 1D
factor products); run from the repo root: python tests/golden/make_c5.py"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import helmdef_oracle as O  # noqa: E402


def projections(x, n_proj=4, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_proj):
        r = rng.uniform(-1, 1, x.size) + 1j * rng.uniform(-1, 1, x.size)
        v = np.vdot(r, x)
        out.append([v.real, v.imag])
    return out


if __name__ == "__main__":
    p, ne, k = 3, 1600, 1000.0
    spec = O.to_spec("DC_MG", p, k, beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)
    s = O.assemble(O.point_source_2d(ne, p, k))
    st = O.compose(s, spec, galerkin="kron", e_solver="fd")
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
    out = dict(config="C5", p=p, elements=ne, k=k, iterations=g.iterations, converged=g.converged,
               residuals=g.residuals, solution_norm=float(np.linalg.norm(g.solution)),
               projections=projections(g.solution),
               counts=dict(matvecs=st.counts.matvecs, coarse_solves=st.counts.coarse_solves,
                           shift_solves=st.counts.shift_solves, vcycles=st.counts.vcycles))
    (Path(__file__).resolve().parent / "C5_oracle.json").write_text(json.dumps(out, indent=1))
    print(out["iterations"], out["converged"])
