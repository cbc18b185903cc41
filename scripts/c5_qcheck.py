"""Accuracy of the device's deflation solve at C5: Q v on the device vs the
oracle's Q v with E solved by fast diagonalisation (LAPACK eigh) and by
partial diagonalisation + banded LU, on one seeded vector."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2010_10232_b200 as hd  # noqa: E402
from oracle import helmdef_oracle as O  # noqa: E402

BASE = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)
p, ne, k = 3, int(sys.argv[1]) if len(sys.argv) > 1 else 1600, 1000.0 * (int(sys.argv[1]) if len(sys.argv) > 1 else 1600) / 1600
s = hd.assemble(hd.point_source_2d(ne, p, k))
rng = np.random.default_rng(3)
v = rng.uniform(-1, 1, s.size) + 1j * rng.uniform(-1, 1, s.size)
with hd.Solver(s, hd.to_spec("DC_MG", p, k, **BASE)) as solver:
    x = torch.from_numpy(v).cuda()
    y = torch.zeros_like(x)
    solver.apply(hd.HD_APPLY_Q, x.data_ptr(), y.data_ptr())
    torch.cuda.synchronize()
    qd = y.cpu().numpy()
so = O.assemble(O.point_source_2d(ne, p, k))
out = {}
for es in ("fd", "pfd"):
    t = time.time()
    st = O.compose(so, O.to_spec("DC_MG", p, k, **BASE), galerkin="kron", e_solver=es)
    out[es] = st.deflation.apply_Q(v)
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
print(f"ne={ne}: device vs fd {rel(qd, out['fd']):.2e}  device vs pfd {rel(qd, out['pfd']):.2e}  "
      f"pfd vs fd {rel(out['pfd'], out['fd']):.2e}")
