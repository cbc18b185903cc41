"""Repeated C5 solves (device-resident rhs) to check timing stability."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_10232_b200 as hd  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dim, p, ne, k = {"C5": (2, 3, 1600, 1000.0), "C3": (2, 2, 320, 200.0), "C2": (1, 4, 31623, 1000.0),
                 "C1": (1, 2, 80, 50.0)}[cfg]
s = hd.assemble(hd.point_source_2d(ne, p, k) if dim == 2 else hd.point_source_1d(ne, p, k))
with hd.Solver(s, hd.to_spec("DC_MG", p, k, beta2="0.5", omega=2 / 3)) as solver:
    b = torch.from_numpy(s.rhs.view(np.float64)).cuda()
    x = torch.zeros_like(b)
    ts = []
    for _ in range(reps):
        r = solver.solve_device(b.data_ptr(), x.data_ptr(), hd.GmresOptions(100, 1e-7))
        ts.append(r.t_solve * 1e3)
    print(cfg, "iterations", r.iterations, "t_solve_ms", " ".join(f"{t:.2f}" for t in ts))
