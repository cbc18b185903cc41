"""C5 pre-stagnation history deviation vs the committed oracle run, per solver
variant (run one variant per process: the env switches are read at create).

  python scripts/c5_attrib.py LABEL   (env: HD_ESOLVE / HD_ARNOLDI / ...)
prints max |dres| over steps 0..19 and per-step diffs, and writes
gpurun_out/c5_attrib_LABEL.json with the full history and projections."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2010_10232_b200 as hd  # noqa: E402

label = sys.argv[1] if len(sys.argv) > 1 else "default"
ref = json.loads((ROOT / "tests/golden/C5_oracle.json").read_text())
s = hd.assemble(hd.point_source_2d(1600, 3, 1000.0))
with hd.Solver(s, hd.to_spec("DC_MG", 3, 1000.0, beta2="0.5", cycles=1, smoothing=1, omega=2 / 3)) as solver:
    r = solver.solve(hd.GmresOptions(100, 1e-7))
m = min(len(r.residuals), len(ref["residuals"]))
d = [abs(r.residuals[j] - ref["residuals"][j]) for j in range(m)]
print(f"[{label}] iterations {r.iterations} (oracle {ref['iterations']}); max|d| j<20 {max(d[:20]):.3e} "
      f"j<23 {max(d[:23]):.3e}")
print(" ".join(f"{x:.1e}" for x in d[:30]))
rng = np.random.default_rng(2024)
proj = []
for re_, im_ in ref["projections"]:
    w = rng.uniform(-1, 1, r.solution.size) + 1j * rng.uniform(-1, 1, r.solution.size)
    got = np.vdot(w, r.solution)
    proj.append(abs(got - complex(re_, im_)) / abs(complex(re_, im_)))
print(f"[{label}] projections rel {max(proj):.2e}")
out = ROOT / "gpurun_out"
out.mkdir(exist_ok=True)
(out / f"c5_attrib_{label}.json").write_text(json.dumps(dict(label=label, residuals=r.residuals, d=d,
                                                             iterations=r.iterations, proj=proj)))
