"""Small solves over every device path, run by tests/test_gpu_poison.py with
and without HD_POISON=1 (poisoned allocations + guard zones: this build's
stand-in for compute-sanitizer initcheck / memcheck, which the GPU pool does
not allow).  Prints one JSON line: per case the iteration count, a hash of
the solution bytes and whether a repeated solve on the same context was
bit-identical, then the number of changed guard zones.

  python tests/poison_cases.py [case...]"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2010_10232_b200 as hd  # noqa: E402

BASE = dict(beta2="0.5", cycles=1, smoothing=1, omega=2.0 / 3.0)


def run(s, spec, budgets=(100, 100), **kw):
    out = []
    with hd.Solver(s, spec, **kw) as solver:
        for b in budgets:
            out.append(solver.solve(hd.GmresOptions(b, 1e-7)))
    a = out[0]
    # same budget: bit-identical; another budget (above 127: the exact-order MGS
    # engine, other rounding) must still converge in the same iteration count
    return dict(iterations=a.iterations, converged=a.converged,
                sha=hashlib.sha256(a.solution.tobytes()).hexdigest()[:16],
                residuals=[float(x) for x in a.residuals],
                repeat_identical=all(np.array_equal(a.solution, r.solution) if b == budgets[0]
                                     else r.iterations == a.iterations for b, r in zip(budgets[1:], out[1:])))


CASES = {
    "1d_small": lambda: run(hd.assemble(hd.point_source_1d(80, 2, 50.0)), hd.to_spec("DC_MG", 2, 50.0, **BASE)),
    "1d_mg": lambda: run(hd.assemble(hd.point_source_1d(2000, 3, 200.0)), hd.to_spec("DC_MG", 3, 200.0, **BASE)),
    "1d_cex": lambda: run(hd.assemble(hd.point_source_1d(400, 3, 100.0)), hd.to_spec("C_ex", 3, 100.0, beta2="1/k")),
    "2d": lambda: run(hd.assemble(hd.point_source_2d(64, 3, 40.0)), hd.to_spec("DC_MG", 3, 40.0, **BASE),
                      budgets=(100, 200, 100)),
    "2d_eps_nu3": lambda: run(hd.assemble(hd.point_source_2d(45, 4, 30.0)),
                              hd.to_spec("Deps_C_MG", 4, 30.0, beta2="4.2", cycles=3, smoothing=3, omega=0.6)),
    "2d_cex": lambda: run(hd.assemble(hd.point_source_2d(48, 2, 30.0)), hd.to_spec("C_ex", 2, 30.0, beta2="1/(3k)")),
    "layered": lambda: run(hd.assemble(hd.layered_medium_2d(48, 2, 30.0)),
                           hd.to_spec("DC_MG", 2, 30.0, beta2="4.2", cycles=2, smoothing=3, omega=0.6)),
    "wedge": lambda: run(hd.assemble(hd.wedge_2d(64, 3, 20.0)), hd.to_spec("DC_MG", 3, 20.0, **BASE)),
    "slabs": lambda: run(hd.assemble(hd.point_source_2d(128, 3, 60.0)), hd.to_spec("DC_MG", 3, 60.0, **BASE),
                         slabs=2),
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    res = {n: CASES[n]() for n in names}
    res["_guards_changed"] = hd.check_guards()
    print(json.dumps(res))
