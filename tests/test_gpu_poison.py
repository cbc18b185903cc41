"""Uninitialised reads and out-of-bounds stores, without compute-sanitizer
(closed on the GPU pool): every case of tests/poison_cases.py runs in a
process with HD_POISON=1 -- each device allocation filled with 0xFF bytes (NaN
doubles) and framed by poisoned guard zones -- and in a plain process.  Any
result that depends on never-written memory turns NaN or changes bits; any
out-of-bounds store changes a guard.  Required: bit-identical solutions and
histories in both processes, repeated solves on one context bit-identical
(including a budget change 100 -> 200 -> 100 that reallocates the basis under
the captured loop graph), and zero changed guards.

compute-sanitizer itself is closed on this GPU pool (runs under it left GPUs
needing a reset), so these runs are the memory checks of this build."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _run(poison, cases=()):
    env = dict(os.environ)
    env.pop("HD_POISON", None)
    if poison:
        env["HD_POISON"] = "1"
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "poison_cases.py"), *cases], capture_output=True,
                       text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_poisoned_allocations_do_not_change_results():
    plain, poisoned = _run(False), _run(True)
    assert poisoned["_guards_changed"] == 0
    for name, a in plain.items():
        if name.startswith("_"):
            continue
        b = poisoned[name]
        print(name, a["iterations"], a["sha"], b["sha"])
        assert a["repeat_identical"] and b["repeat_identical"], name
        assert (a["iterations"], a["converged"], a["sha"], a["residuals"]) == \
            (b["iterations"], b["converged"], b["sha"], b["residuals"]), name


def test_results_do_not_depend_on_process_history():
    """Each case alone in a fresh process gives the same bits as after all the
    other cases in one process (round 1 noted a transient that seemed to differ
    with earlier work in the process; poisoned allocations rule out stale
    memory, this rules out any other carried state: library handles, cached
    launch geometry, graph reuse)."""
    together = _run(False)
    for name in ("2d", "2d_eps_nu3", "wedge", "slabs"):
        alone = _run(False, (name,))[name]
        assert (alone["iterations"], alone["sha"], alone["residuals"]) == \
            (together[name]["iterations"], together[name]["sha"], together[name]["residuals"]), name
