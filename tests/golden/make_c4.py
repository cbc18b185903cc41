"""Oracle reference for the full-size C4 config (BASELINE config 4: the
three-layer wedge k = (1.2, 1.5, 1.0) x 150 split by y = 0.6 - 0.2x and
y = 0.3 + 0.1x, p = 3, 480^2 elements, point source at (0.5, 1 - 1/480),
DC_MG^1 with beta2 = 0.5, omega = 2/3, nu = 1): iteration count, converged
flag, residual history, counters and seeded projections of the solution.
The wedge is an oracle extension (oracle/helmdef_oracle.py wedge_2d; the
reference API cannot express it), solved with the
reference's own sparse algorithm: Galerkin triple products on the assembled
CSR matrices and SuperLU for E and the coarsest level.
Run from the repo root: python tests/golden/make_c4.py"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import helmdef_oracle as O  # noqa: E402
sys.path.insert(0, str(Path(__file__).resolve().parent))
from make_c5 import projections  # noqa: E402

if __name__ == "__main__":
    p, ne, k0 = 3, 480, 150.0
    spec = O.to_spec("DC_MG", p, k0, beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)
    t0 = time.time()
    s = O.assemble(O.wedge_2d(ne, p, k0))
    st = O.compose(s, spec)
    t1 = time.time()
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
    t2 = time.time()
    out = dict(config="C4", p=p, elements=ne, k0=k0, iterations=g.iterations, converged=g.converged,
               residuals=g.residuals, solution_norm=float(np.linalg.norm(g.solution)),
               projections=projections(g.solution),
               counts=dict(matvecs=st.counts.matvecs, coarse_solves=st.counts.coarse_solves,
                           shift_solves=st.counts.shift_solves, vcycles=st.counts.vcycles),
               oracle_seconds=dict(setup=t1 - t0, solve=t2 - t1))
    (Path(__file__).resolve().parent / "C4_oracle.json").write_text(json.dumps(out, indent=1))
    print(out["iterations"], out["converged"], out["oracle_seconds"])
