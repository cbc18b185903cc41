"""Per-application time of the deflation E solve at a config (default C5),
for the solver HD_ESOLVE selects: profiled Q applications, per-kind CUDA-event
times.  python scripts/time_esolve.py [C5|C3] (env HD_ESOLVE=fd|pfd|fold)"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2010_10232_b200 as hd  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
p, ne, k = {"C5": (3, 1600, 1000.0), "C3": (2, 320, 200.0)}[cfg]
s = hd.assemble(hd.point_source_2d(ne, p, k))
sp = hd.to_spec("DC_MG", p, k, beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)
rng = np.random.default_rng(5)
x = torch.from_numpy(rng.uniform(-1, 1, s.size) + 1j * rng.uniform(-1, 1, s.size)).cuda()
y = torch.zeros_like(x)
with hd.Solver(s, sp) as solver:
    for _ in range(5):
        solver.apply(hd.HD_APPLY_Q, x.data_ptr(), y.data_ptr())
    solver.profile(True)
    reps = 20
    for _ in range(reps):
        solver.apply(hd.HD_APPLY_Q, x.data_ptr(), y.data_ptr())
    torch.cuda.synchronize()
    prof = solver.profile_read()
    solver.profile(False)
print(os.environ.get("HD_ESOLVE", "default"), cfg,
      {kk: (n // reps, round(1e3 * ms / reps, 1)) for kk, (n, ms, b) in prof.items()}, "us per Q application")
