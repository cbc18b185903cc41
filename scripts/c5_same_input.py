"""C5 (and C3) on the SAME assembled system as the oracle: the device is fed
the oracle's reduced 1D bands and load vector (tests/test_gpu_parity.py
`_same_input`), so the history differences are the solvers' alone.
python scripts/c5_same_input.py [C5|C3]"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2010_10232_b200 as hd  # noqa: E402
from oracle import helmdef_oracle as O  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
p, ne, k = {"C5": (3, 1600, 1000.0), "C3": (2, 320, 200.0)}[cfg]
BASE = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)
so = O.assemble(O.point_source_2d(ne, p, k))
s = hd.system_from_bands(hd.point_source_2d(ne, p, k), np.asarray(so.S1), np.asarray(so.M1), so.rhs)
with hd.Solver(s, hd.to_spec("DC_MG", p, k, **BASE)) as solver:
    r = solver.solve(hd.GmresOptions(100, 1e-7))
if cfg == "C5":
    ref = json.loads((ROOT / "tests/golden/C5_oracle.json").read_text())["residuals"]
    it = json.loads((ROOT / "tests/golden/C5_oracle.json").read_text())["iterations"]
else:
    st = O.compose(so, O.to_spec("DC_MG", p, k, **BASE), galerkin="kron", e_solver="fd")
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
    ref, it = g.residuals, g.iterations
    print("solution rel", np.linalg.norm(r.solution - g.solution) / np.linalg.norm(g.solution))
m = min(len(ref), len(r.residuals))
d = [abs(a - b) for a, b in zip(r.residuals[:m], ref[:m])]
print(f"[{cfg} same input] iterations {r.iterations} (oracle {it}); max|d| j<20 {max(d[:20]):.3e}")
print(" ".join(f"{x:.1e}" for x in d[:30]))
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / f"same_input_{cfg}.json").write_text(json.dumps(dict(residuals=r.residuals, d=d)))
