"""Rounding envelope of the GMRES history: oracle runs of a config that are
all exact implementations of the reference algorithm and differ only in
rounding --
  * the deflation matrix E solved by fast diagonalisation with LAPACK dsygvd
    eigenvectors (FDSolver, the committed C5 oracle run) or with dsygv's
    (fd_gv: another eigen-algorithm, so other eigenvector rounding -- what
    separates the device's cuSOLVER eigenvectors from the oracle's), by
    partial diagonalisation + banded LU with partial pivoting
    (PartialFDSolver), and by SuperLU (the reference's own kind of solver,
    Eigen::SparseLU at src/precond.cpp:95-104) where that is feasible (C3);
  * every operator product through the assembled CSR matrix or through its
    Kronecker factors (apply="kron": another summation order, the device's).
The per-step spread of their histories is how far rounding alone moves the
history at that step; the device is one more exact implementation and is held
to this envelope (tests/test_gpu_parity.py).

  python tests/golden/make_e_envelope.py C3|C5     (C5: ~15 min per run, ~10 GB)
writes tests/golden/<cfg>_E_envelope.json (runs already in it are kept)"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import helmdef_oracle as O  # noqa: E402

CFG = {"C3": (2, 320, 200.0, (("fd", "csr"), ("pfd", "csr"), ("splu", "csr"), ("fd", "kron"), ("fd_gv", "csr"))),
       "C5": (3, 1600, 1000.0, (("pfd", "csr"), ("fd", "kron"), ("fd_gv", "csr")))}
BASE = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)

if __name__ == "__main__":
    name = sys.argv[1]
    p, ne, k, variants = CFG[name]
    out_path = Path(__file__).resolve().parent / f"{name}_E_envelope.json"
    runs = json.loads(out_path.read_text())["runs"] if out_path.exists() else {}
    runs = {(kk if "/" in kk else kk + "/csr"): v for kk, v in runs.items()}
    if name == "C5":  # the FD/CSR run is the committed oracle reference
        ref = json.loads((ROOT / "tests/golden/C5_oracle.json").read_text())
        runs["fd/csr"] = dict(iterations=ref["iterations"], converged=ref["converged"], residuals=ref["residuals"])
    O.use_c_spmv(8)
    s = O.assemble(O.point_source_2d(ne, p, k))
    for es, ap in variants:
        key = f"{es}/{ap}"
        if key in runs:
            continue
        t = time.time()
        st = O.compose(s, O.to_spec("DC_MG", p, k, **BASE), galerkin="kron", e_solver=es, apply=ap)
        g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(100, 1e-7))
        runs[key] = dict(iterations=g.iterations, converged=g.converged, residuals=g.residuals)
        print(key, g.iterations, g.converged, f"{time.time() - t:.0f}s", flush=True)
        keys = list(runs)
        m = min(len(r["residuals"]) for r in runs.values())
        env = [max(abs(runs[a]["residuals"][j] - runs[b]["residuals"][j]) for a in keys for b in keys)
               for j in range(m)]
        out = dict(config=name, variants=keys, runs=runs, envelope=env,
                   note="per-step max |r_a - r_b| over exact implementations (E solver / operator products): "
                        + ", ".join(keys))
        out_path.write_text(json.dumps(out, indent=1))
        print(" ".join(f"{x:.1e}" for x in env))
