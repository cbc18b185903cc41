"""Run-to-run determinism of the device solve: the same context solves the same
system several times; prints the max history / solution differences."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2010_10232_b200 as hd  # noqa: E402

ne, p, k = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (130, 3, 80.0)
s = hd.assemble(hd.point_source_2d(ne, p, k))
spec = hd.to_spec("DC_MG", p, k, beta2="0.5", cycles=1, smoothing=1, omega=2 / 3)
with hd.Solver(s, spec) as sv:
    rs = [sv.solve(hd.GmresOptions(100, 1e-7)) for _ in range(4)]
h0 = np.array(rs[0].residuals)
for r in rs[1:]:
    h = np.array(r.residuals)
    m = min(len(h), len(h0))
    print(os.environ.get("HD_GRAPH", "graph"), "iters", r.iterations, "h[5]", repr(h[5]), "max|dhist|", np.max(np.abs(h[:m] - h0[:m])),
          "max|dx|", np.max(np.abs(r.solution - rs[0].solution)))
