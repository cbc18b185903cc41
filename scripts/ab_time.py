"""A/B timing of library builds: C5 graph-path solves (CUDA events, L2 flushed
between solves).  HD_LIBRARY selects the build; prints ms per solve."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2010_10232_b200 as hd  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dim, p, ne, k = {"C5": (2, 3, 1600, 1000.0), "C3": (2, 2, 320, 200.0), "C2": (1, 4, 31623, 1000.0),
                 "C1": (1, 2, 80, 50.0), "C4": (2, 3, 480, 150.0)}[cfg]
if cfg == "C4":
    s = hd.assemble(hd.wedge_2d(ne, p, k))
else:
    s = hd.assemble(hd.point_source_2d(ne, p, k) if dim == 2 else hd.point_source_1d(ne, p, k))
solver = hd.Solver(s, hd.to_spec("DC_MG", p, k, beta2="0.5", omega=2 / 3))
st = torch.cuda.current_stream()
solver.set_stream(st.cuda_stream)
rhs = torch.from_numpy(s.rhs.view(np.float64)).cuda()
x = torch.zeros_like(rhs)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
opt = hd.GmresOptions(100, 1e-7)
for _ in range(3):
    r = solver.solve_device(rhs.data_ptr(), x.data_ptr(), opt)
ts = []
for _ in range(reps):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    r = solver.solve_device(rhs.data_ptr(), x.data_ptr(), opt)
    b.record(st)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(f"{hd.LIB_PATH.name} {cfg}: iterations {r.iterations}, ms/solve min {min(ts):.2f} median {sorted(ts)[len(ts)//2]:.2f}")
solver.close()
