"""Every environment switch of the library that selects another implementation
of the same mathematics (an A/B path kept for measurement or as the exact-order
reference) against the default path: equal iterations, counts and converged
flag, the final history entries within 1e-10, the solution within 1e-9 relative
(tests/test_gpu_variants.py holds the tighter per-operator comparisons of the
switches that can be set per context).  One fresh process per run: several
switches are read once per process."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

SWITCHES = [
    ("2d_p3", "HD_DGEMM", "dmma"),      # own FP64 tensor-core GEMM in the E solve (dgemm.cuh) vs cuBLAS
    ("2d_p2", "HD_DGEMM", "dmma"),
    ("2d_p3", "HD_NOFUSE", "1"),        # separate operator and restriction launches vs the fused K3/K6 kernels
    ("2d_p2", "HD_NOFUSE", "1"),
    ("2d_p3", "HD_LSA_MMA", "1"),       # Arnoldi pass 1 as an FP64 tensor-core GEMM (k_lsa_dots_mma)
    ("2d_p2", "HD_LSA_MMA", "1"),
    ("2d_p3", "HD_LSA_REV", "0"),       # pass 2 front to back
    ("2d_p3", "HD_ARNOLDI", "0"),       # exact-order MGS engine vs the one-reduction form
    ("2d_p3", "HD_ESOLVE", "fd"),       # unfolded fast diagonalisation of E
    ("2d_p3", "HD_CENTRO_TOL", "0"),    # never fold
    ("1d_small", "HD_SMALL", "0"),      # per-kernel path vs the single-CTA whole solve
    ("1d_mg", "HD_TAIL", "0"),          # per-level kernels vs the single-CTA multigrid tail
    ("1d_mg", "HD_SEG", "0"),           # single-lane banded sweeps vs the segmented ones
    ("slabs", "HD_DIST_E", "0"),        # redundant E solve vs the one split by slab
    ("2d_p3", "HD_GRAPH", "0"),         # host-driven loop vs the device-resident graph
]

_cache = {}


def _run(case, var=None, val=None):
    key = (case, var, val)
    if key not in _cache:
        env = {k: v for k, v in os.environ.items() if not k.startswith("HD_")}
        if var:
            env[var] = val
        r = subprocess.run([sys.executable, str(ROOT / "tests" / "switch_cases.py"), case], capture_output=True,
                           text=True, env=env, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        _cache[key] = json.loads(r.stdout.strip().splitlines()[-1])
    return _cache[key]


@pytest.mark.parametrize("case,var,val", SWITCHES)
def test_switch_matches_default(case, var, val):
    a, b = _run(case), _run(case, var, val)
    assert (a["iterations"], a["converged"], a["counts"]) == (b["iterations"], b["converged"], b["counts"])
    ha, hb = np.array(a["residuals"]), np.array(b["residuals"])
    assert np.max(np.abs(ha[-3:] - hb[-3:])) <= 1e-10
    assert np.all(np.abs(ha - hb) <= 1e-2 * np.maximum(ha, hb))  # transients amplify rounding
    xa = np.array(a["re"]) + 1j * np.array(a["im"])
    xb = np.array(b["re"]) + 1j * np.array(b["im"])
    assert np.linalg.norm(xa - xb) <= 1e-9 * np.linalg.norm(xa)
