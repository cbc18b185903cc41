"""Host-only checks of the C++ harness (include/helmdef_b200_harness.hpp)
through tools/hd_bench, the helmbench mirror -- the reference's test_harness
cases (tests/test_harness.cpp:55-143, 160-240) without a GPU:

  * config hash: FNV-1a of the canonical nlohmann dump(2) (src/harness.cpp:
    30-44, 130-131), stable and content sensitive, equal to an independent
    Python rendering of the same canonical form;
  * RunRecord CSV <-> JSON round trip, byte identical (src/harness.cpp:324-448);
  * compare_cells on records made from the pinned oracle counts: every golden
    table matches (exit 0), a moved cell or a non-convergence marker
    mismatches (exit 2), a malformed golden header is an error (exit 1)."""
import csv
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
TAB = ROOT / "tests" / "golden" / "tables"
BENCH = ROOT / "tools" / "hd_bench"
HEADER = ("problem,tag,k,p,elements,dofs,iterations,converged,residual,direct_gap,"
          "matvecs,shift_solves,vcycles,coarse_solves,seconds,config_hash")

pytestmark = pytest.mark.skipif(not BENCH.exists(), reason="tools/hd_bench not built")


def _run(*args):
    return subprocess.run([str(BENCH), *map(str, args)], capture_output=True, text=True, timeout=120)


def _py_hash(path):
    text = json.dumps(json.loads(Path(path).read_text()), indent=2, sort_keys=True)
    h = 1469598103934665603
    for b in text.encode():
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


@pytest.mark.parametrize("table", ["table2", "table3", "table4", "table5", "table6"])
def test_config_hash_matches_canonical_dump(table):
    r = _run("hash", "--config", TAB / f"{table}.json")
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == _py_hash(TAB / f"{table}.json")


def test_config_hash_is_content_sensitive(tmp_path):
    cfg = json.loads((TAB / "table4.json").read_text())
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    a.write_text(json.dumps(cfg))
    cfg["kh"] = 0.825
    b.write_text(json.dumps(cfg, indent=4))
    ha, hb = _run("hash", "--config", a).stdout, _run("hash", "--config", b).stdout
    assert ha == _run("hash", "--config", TAB / "table4.json").stdout  # formatting of the file is irrelevant
    assert ha != hb


def _records_from_pins(table, tmp_path, tweak=None):
    h = _run("hash", "--config", TAB / f"{table}.json").stdout.strip()
    cfg = json.loads((TAB / f"{table}.json").read_text())
    out = tmp_path / f"{table}_records.csv"
    with open(ROOT / "tests" / "golden" / "oracle_pins.csv") as fh, open(out, "w") as fo:
        fo.write(HEADER + "\n")
        for r in csv.DictReader(fh):
            if r["table"] != table:
                continue
            it, conv = int(r["oracle"]), r["converged"]
            if tweak:
                it, conv = tweak(r, it, conv)
            dofs = (int(r["elements"]) + int(r["p"]) - 2) ** (2 if "2d" in cfg["problem"] else 1)
            fo.write(f"{cfg['problem']},{r['tag']},{r['k']},{r['p']},{r['elements']},{dofs},{it},{conv},"
                     f"9.5e-08,nan,{it + 1},{it + 2},{it + 2},{it + 3},0.25,{h}\n")
    return out


@pytest.mark.parametrize("table", ["table2", "table3", "table4", "table5", "table6"])
def test_compare_pinned_oracle_records_match_golden(table, tmp_path):
    rec = _records_from_pins(table, tmp_path)
    r = _run("compare", "--config", TAB / f"{table}.json", "--reference", TAB / f"{table}_golden.csv",
             "--records", rec)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatched 0, missing 0" in r.stdout


def test_compare_flags_mismatches(tmp_path):
    moved = _records_from_pins("table4", tmp_path,
                               lambda r, it, c: (it + 10, c) if (r["k"], r["p"]) == ("1000", "3") else (it, c))
    r = _run("compare", "--config", TAB / "table4.json", "--reference", TAB / "table4_golden.csv", "--records", moved)
    assert r.returncode == 2 and "<-- MISMATCH" in r.stdout
    assert r.stdout.count("<-- MISMATCH") == 3  # the three table4 columns at (k=1000, p=3)
    starred = _records_from_pins("table2", tmp_path, lambda r, it, c: (100, "0") if r["p"] == "1" else (it, c))
    r = _run("compare", "--config", TAB / "table2.json", "--reference", TAB / "table2_golden.csv", "--records", starred)
    assert r.returncode == 2 and "got *" in r.stdout


def test_compare_rejects_unknown_golden_header(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("# comment\ntag,k,p,value\nD,100,1,5\n")
    rec = _records_from_pins("table2", tmp_path)
    r = _run("compare", "--config", TAB / "table2.json", "--reference", bad, "--records", rec)
    assert r.returncode == 1 and "unknown reference header" in r.stderr


def test_records_round_trip_byte_identical(tmp_path):
    src = tmp_path / "r.csv"
    src.write_text(HEADER + "\n"
                   "point_source_1d,D_eps,100,2,159,158,12,1,8.731e-08,3.2e-09,13,0,0,15,0.0123,0123456789abcdef\n"
                   "point_source_2d,DC_MG^1,1000,3,1600,2563201,100,0,0.000125,nan,101,102,102,103,1.5,0123456789abcdef\n")
    j = tmp_path / "r.json"
    assert _run("records", "--in", src, "--format", "json", "--out", j).returncode == 0
    data = json.loads(j.read_text())
    assert data["config"] is None and len(data["records"]) == 2
    assert "direct_gap" not in data["records"][1] and data["records"][0]["direct_gap"] == 3.2e-09
    back = _run("records", "--in", j, "--format", "csv")
    assert back.returncode == 0
    assert back.stdout == src.read_text()
