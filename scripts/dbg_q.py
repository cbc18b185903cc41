"""Debug: device Q = Z E^-1 Z^T v against the oracle for several grid sizes."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2010_10232_b200 as hd
from oracle import helmdef_oracle as O

for ne, p, k in [(60, 3, 20.0), (64, 3, 20.0), (66, 3, 20.0), (70, 2, 20.0), (130, 2, 40.0), (200, 3, 60.0)]:
    so = O.assemble(O.point_source_2d(ne, p, k))
    st = O.compose(so, O.to_spec("D", p, k), galerkin="kron", e_solver="fd")
    s = hd.assemble(hd.point_source_2d(ne, p, k))
    rng = np.random.default_rng(1)
    v = rng.uniform(-1, 1, s.size) + 1j * rng.uniform(-1, 1, s.size)
    ref = st.deflation.apply_Q(v)
    with hd.Solver(s, hd.to_spec("D", p, k)) as sol:
        xd = torch.from_numpy(v).cuda(); yd = torch.zeros_like(xd)
        sol.apply(hd.HD_APPLY_Q, xd.data_ptr(), yd.data_ptr())
        got = yd.cpu().numpy()
    print(ne, p, "nc", so.per_dim // 2, "rel", np.linalg.norm(got - ref) / np.linalg.norm(ref))
