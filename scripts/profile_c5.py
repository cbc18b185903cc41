"""Short C5 solve (a few GMRES iterations) for ncu captures of single kernels."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2010_10232_b200 as hd  # noqa: E402

maxit = int(sys.argv[1]) if len(sys.argv) > 1 else 6
cfg = sys.argv[2] if len(sys.argv) > 2 else "C5"
dim, p, ne, k = {"C5": (2, 3, 1600, 1000.0), "C4": (2, 3, 480, 150.0), "C3": (2, 2, 320, 200.0),
                 "C2": (1, 4, 31623, 1000.0)}[cfg]
if cfg == "C4":
    s = hd.assemble(hd.wedge_2d(ne, p, k))
else:
    s = hd.assemble(hd.point_source_2d(ne, p, k) if dim == 2 else hd.point_source_1d(ne, p, k))
with hd.Solver(s, hd.to_spec("DC_MG", p, k, beta2="0.5", omega=2 / 3)) as solver:
    r = solver.solve(hd.GmresOptions(maxit, 1e-7))
print("iterations", r.iterations, "t_solve_ms", r.t_solve * 1e3)
