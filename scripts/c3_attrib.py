"""C3 (2D k=200, p=2, 320^2) device history vs a live oracle run (FD and, when
asked, SuperLU E solves): python scripts/c3_attrib.py LABEL [splu]"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2010_10232_b200 as hd  # noqa: E402
from oracle import helmdef_oracle as O  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else "default"
BASE = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)
s = hd.assemble(hd.point_source_2d(320, 2, 200.0))
with hd.Solver(s, hd.to_spec("DC_MG", 2, 200.0, **BASE)) as solver:
    r = solver.solve(hd.GmresOptions(100, 1e-7))
out = dict(label=label, device=r.residuals, iterations=r.iterations)
for es in (["fd", "splu"] if "splu" in sys.argv else ["fd"]):
    so = O.assemble(O.point_source_2d(320, 2, 200.0))
    st = O.compose(so, O.to_spec("DC_MG", 2, 200.0, **BASE), galerkin="kron", e_solver=es)
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
    m = min(len(g.residuals), len(r.residuals))
    d = [abs(a - b) for a, b in zip(r.residuals[:m], g.residuals[:m])]
    rel = np.linalg.norm(r.solution - g.solution) / np.linalg.norm(g.solution)
    print(f"[{label}] device {r.iterations} oracle-{es} {g.iterations}; max|d| {max(d):.2e}; sol rel {rel:.2e}")
    print(" ".join(f"{x:.1e}" for x in d))
    out[es] = g.residuals
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / f"c3_attrib_{label}.json").write_text(json.dumps(out))
