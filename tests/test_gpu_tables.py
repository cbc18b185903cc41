"""The reference's own iteration tables on the device path (SURVEY.md §8(f)
rank 1), run the way the reference runs them: tools/hd_bench (the helmbench
mirror, C++ harness over the C-ABI) sweeps each config of
tests/golden/tables/ (data/config/tableN.json, k capped as the oracle pins)
and `hd_bench compare` checks every cell against the golden table under the
reference's compare rule (src/harness.cpp:547-592, exit 0 = all matched).
Every device cell is also held to the pinned oracle (tests/golden/
oracle_pins.csv) within +-1 iteration, and the records carry the config hash
and the counters of compose()'s call pattern.

table6 (layered medium) runs in tests/test_gpu_parity.py, with its one
documented SuperLU-rounding cell (k = 150, p = 3)."""
import csv
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
TAB = ROOT / "tests" / "golden" / "tables"
BENCH = ROOT / "tools" / "hd_bench"


def _pins(table):
    with open(ROOT / "tests" / "golden" / "oracle_pins.csv") as fh:
        return {(r["tag"], float(r["k"]), int(r["p"])): r for r in csv.DictReader(fh) if r["table"] == table}


@pytest.mark.parametrize("table", ["table2", "table3", "table4", "table5"])
def test_reference_table_on_device(table, tmp_path):
    assert BENCH.exists(), "tools/hd_bench not built (python -c 'import __graft_entry__ as g; g.build()')"
    rec = tmp_path / f"{table}.csv"
    r = subprocess.run([str(BENCH), "table", "--config", str(TAB / f"{table}.json"), "--out", str(rec)],
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr
    c = subprocess.run([str(BENCH), "compare", "--config", str(TAB / f"{table}.json"), "--reference",
                        str(TAB / f"{table}_golden.csv"), "--records", str(rec)], capture_output=True, text=True)
    print(c.stdout)
    assert c.returncode == 0, c.stdout + c.stderr
    assert "mismatched 0, missing 0" in c.stdout
    h = subprocess.run([str(BENCH), "hash", "--config", str(TAB / f"{table}.json")], capture_output=True, text=True)
    cfg_hash = h.stdout.strip()
    pins = _pins(table)
    with open(rec) as fh:
        rows = list(csv.DictReader(fh))
    assert len(rows) == len(pins)
    off = []
    for row in rows:
        pin = pins[(row["tag"], float(row["k"]), int(row["p"]))]
        assert row["config_hash"] == cfg_hash
        assert int(row["elements"]) == int(pin["elements"])
        assert row["converged"] == pin["converged"]
        d = int(row["iterations"]) - int(pin["oracle"])
        assert abs(d) <= 1, (row, pin)
        if d:
            off.append((row["tag"], row["k"], row["p"], d))
        it = int(row["iterations"])
        if row["converged"] == "1" and it > 0:
            # compose()'s call pattern (src/precond.cpp:236-256): one op per step + the initial residual's
            assert int(row["matvecs"]) == it + 1
    print(f"{table}: {len(rows)} cells, all within the golden rule; off the oracle pin by 1: {off}")


def test_check_direct_records_direct_gap(tmp_path):
    """`solve --check-direct` fills RunRecord::direct_gap from an exact device
    solve of A (src/harness.cpp:234-238); a converged GMRES run sits within
    the reference's Krylov-vs-direct bar (tests/test_acceptance.cpp:411-459)."""
    for problem, k, p in (("point_source_1d", 100, 2), ("point_source_2d", 30, 2), ("layered_medium_2d", 20, 2)):
        out = tmp_path / f"{problem}.csv"
        r = subprocess.run([str(BENCH), "solve", "--problem", problem, "--k", str(k), "--p", str(p), "--tag",
                            "DC_MG", "--beta2", "0.5", "--omega", "0.6667", "--check-direct", "--out", str(out)],
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        row = next(csv.DictReader(open(out)))
        assert row["converged"] == "1"
        gap = float(row["direct_gap"])
        assert 0.0 <= gap <= 1e-6, row
