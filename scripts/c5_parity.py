"""C5 residual history vs the committed oracle run (per-iteration diffs)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2010_10232_b200 as hd  # noqa: E402

ref = json.loads((ROOT / "tests/golden/C5_oracle.json").read_text())
s = hd.assemble(hd.point_source_2d(1600, 3, 1000.0))
with hd.Solver(s, hd.to_spec("DC_MG", 3, 1000.0, beta2="0.5", omega=2 / 3)) as solver:
    r = solver.solve(hd.GmresOptions(100, 1e-7))
m = min(len(r.residuals), len(ref["residuals"]))
for j in range(m):
    a, b = r.residuals[j], ref["residuals"][j]
    print(f"{j:3d} gpu {a:.10e} ora {b:.10e} abs {abs(a-b):.2e} rel {abs(a-b)/b:.2e}")
print("iterations", r.iterations, ref["iterations"])
env = json.loads((ROOT / "tests/golden/C5_envelope.json").read_text())["envelope"]
worst = []
for j in range(min(m, len(env))):
    d = abs(r.residuals[j] - ref["residuals"][j])
    e = max(env[max(0, j - 2):j + 3])
    worst.append((d / max(e, 1e-12), j, d, e))
worst.sort(reverse=True)
print("worst ratios d/env:", [(f"{a:.1f}", j, f"{d:.1e}", f"{e:.1e}") for a, j, d, e in worst[:8]])
rng = np.random.default_rng(2024)
for re_, im_ in ref["projections"]:
    w = rng.uniform(-1, 1, r.solution.size) + 1j * rng.uniform(-1, 1, r.solution.size)
    got = np.vdot(w, r.solution)
    print("projection rel", abs(got - complex(re_, im_)) / abs(complex(re_, im_)))
print("norm rel", abs(np.linalg.norm(r.solution) - ref["solution_norm"]) / ref["solution_norm"])
