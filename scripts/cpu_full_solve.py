"""One full CPU time-to-solution of a BASELINE config with the oracle port of the
reference algorithm on ONE host thread (the reference is
single-threaded per solve).  Writes gpurun_out/r2_cpu_full_<cfg>.json; the
committed copy under profiles/ is what bench.py's cpu_baseline.full_solve cites.
  python scripts/cpu_full_solve.py [C5]"""
import json
import os
import platform
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from threadpoolctl import threadpool_limits  # noqa: E402

import bench  # noqa: E402
from oracle import helmdef_oracle as O  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
dim, p, ne, k = bench.CONFIGS[cfg]
with threadpool_limits(limits=1):
    t0 = time.perf_counter()
    s = O.assemble(bench.make_problem(O, cfg))
    t_asm = time.perf_counter() - t0
    big = dim == 2 and s.A.shape[0] > 300_000 and s.separable
    spec = O.to_spec(bench.SPEC["tag"], p, k, beta2=bench.SPEC["beta2"], cycles=bench.SPEC["cycles"],
                     smoothing=bench.SPEC["smoothing"], omega=bench.SPEC["omega"])
    t0 = time.perf_counter()
    st = O.compose(s, spec, galerkin="kron" if dim == 2 and s.separable else "sparse",
                   e_solver="fd" if big else "splu")
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    g = O.gmres(st.op, st.rhs, st.start, st.monitor, O.GmresOptions(bench.MAXIT, bench.TOL))
    t_solve = time.perf_counter() - t0
cpu = ""
try:
    cpu = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
except Exception:
    cpu = platform.processor()
out = {"config": cfg, "workload": bench.workload_name(cfg), "threads": 1, "cpu": cpu, "host_cores": os.cpu_count(),
       "iterations": g.iterations, "converged": bool(g.converged), "final_residual": float(g.residuals[-1]),
       "t_assemble_s": round(t_asm, 2), "t_setup_s": round(t_setup, 2), "t_solve_s": round(t_solve, 2),
       "iterations_per_s": round(g.iterations / t_solve, 4),
       "method": "oracle/helmdef_oracle.py (scipy CSR products, " +
                 ("fast-diagonalisation" if big else "SuperLU") + " E solve), whole solve, 1 thread"}
(ROOT / "gpurun_out").mkdir(exist_ok=True)
(ROOT / "gpurun_out" / f"r2_cpu_full_{cfg}.json").write_text(json.dumps(out, indent=1))
print(json.dumps(out))
