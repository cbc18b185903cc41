"""E-solver rounding envelope of the GMRES history: the oracle run of a
config with its deflation matrix E solved by two different exact direct
methods -- fast diagonalisation (FDSolver, the committed C5 oracle run) and
partial diagonalisation + banded LU with partial pivoting (PartialFDSolver),
plus SuperLU (the reference's own kind of solver, Eigen::SparseLU at
src/precond.cpp:95-104) where it is feasible (C3).  Every other operation is
identical, so the per-step history differences are what the rounding of an
exact E solve alone moves; the device's E solve is a third exact method and
is held to this envelope (tests/test_gpu_parity.py).

  python tests/golden/make_e_envelope.py C3|C5     (C5: ~15 min, ~10 GB)
writes tests/golden/<cfg>_E_envelope.json"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import helmdef_oracle as O  # noqa: E402

CFG = {"C3": (2, 320, 200.0, ("fd", "pfd", "splu")), "C5": (3, 1600, 1000.0, ("pfd",))}
BASE = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)

if __name__ == "__main__":
    name = sys.argv[1]
    p, ne, k, solvers = CFG[name]
    s = O.assemble(O.point_source_2d(ne, p, k))
    runs = {}
    if name == "C5":  # the FD run is the committed oracle reference
        ref = json.loads((ROOT / "tests/golden/C5_oracle.json").read_text())
        runs["fd"] = dict(iterations=ref["iterations"], converged=ref["converged"], residuals=ref["residuals"])
    for es in solvers:
        t = time.time()
        st = O.compose(s, O.to_spec("DC_MG", p, k, **BASE), galerkin="kron", e_solver=es)
        g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
        runs[es] = dict(iterations=g.iterations, converged=g.converged, residuals=g.residuals)
        print(es, g.iterations, g.converged, f"{time.time() - t:.0f}s", flush=True)
    keys = list(runs)
    m = min(len(r["residuals"]) for r in runs.values())
    env = [max(abs(runs[a]["residuals"][j] - runs[b]["residuals"][j]) for a in keys for b in keys)
           for j in range(m)]
    out = dict(config=name, solvers=keys, runs=runs, envelope=env,
               note="per-step max |r_a - r_b| over exact E solvers " + ", ".join(keys))
    (Path(__file__).resolve().parent / f"{name}_E_envelope.json").write_text(json.dumps(out, indent=1))
    print(" ".join(f"{x:.1e}" for x in env))
