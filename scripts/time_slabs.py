"""Slab program on one GPU: ms per solve for S slabs, graph-resident iteration
(default) vs host-driven loop (HD_GRAPH=0).  python scripts/time_slabs.py C5 2"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2010_10232_b200 as hd  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dim, p, ne, k = {"C5": (2, 3, 1600, 1000.0), "C3": (2, 2, 320, 200.0)}[cfg]
s = hd.assemble(hd.point_source_2d(ne, p, k))
solver = hd.Solver(s, hd.to_spec("DC_MG", p, k, beta2="0.5", omega=2 / 3), slabs=S)
rhs = torch.from_numpy(s.rhs.view(np.float64)).cuda()
x = torch.zeros_like(rhs)
opt = hd.GmresOptions(100, 1e-7)
for _ in range(2):
    r = solver.solve_device(rhs.data_ptr(), x.data_ptr(), opt)
ts = [solver.solve_device(rhs.data_ptr(), x.data_ptr(), opt).t_solve * 1e3 for _ in range(3)]
print(f"{cfg} slabs={S}: iterations {r.iterations}, ms/solve min {min(ts):.2f}, kernels {r.kernel_launches}")
