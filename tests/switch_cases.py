"""One solve of a named case; prints a JSON line with the iteration count, the
history and the solution (run by tests/test_gpu_switches.py in a fresh process
per environment switch, since some switches are read once per process).

  python tests/switch_cases.py CASE"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2010_10232_b200 as hd  # noqa: E402

BASE = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)
CASES = {
    "2d_p3": lambda: (hd.assemble(hd.point_source_2d(96, 3, 60.0)), hd.to_spec("DC_MG", 3, 60.0, **BASE), {}),
    "2d_p2": lambda: (hd.assemble(hd.point_source_2d(128, 2, 80.0)), hd.to_spec("DC_MG", 2, 80.0, **BASE), {}),
    "1d_small": lambda: (hd.assemble(hd.point_source_1d(80, 2, 50.0)), hd.to_spec("DC_MG", 2, 50.0, **BASE), {}),
    "1d_mg": lambda: (hd.assemble(hd.point_source_1d(6000, 3, 300.0)), hd.to_spec("DC_MG", 3, 300.0, **BASE), {}),
    "slabs": lambda: (hd.assemble(hd.point_source_2d(129, 3, 60.0)), hd.to_spec("DC_MG", 3, 60.0, **BASE),
                      dict(slabs=2)),
}

if __name__ == "__main__":
    s, spec, kw = CASES[sys.argv[1]]()
    with hd.Solver(s, spec, **kw) as solver:
        r = solver.solve(hd.GmresOptions(100, 1e-7))
    print(json.dumps(dict(iterations=r.iterations, converged=bool(r.converged),
                          residuals=[float(x) for x in r.residuals],
                          counts=[r.counts.matvecs, r.counts.coarse_solves, r.counts.shift_solves],
                          re=r.solution.real.tolist(), im=r.solution.imag.tolist())))
