"""Sweep configs and golden tables of the reference's iteration studies, as
fixtures for the device runs (tests/test_gpu_tables.py through tools/hd_bench,
the helmbench mirror): tables/tableN.json and tables/tableN_golden.csv.

Configs: /root/reference/proj/data/config/tableN.json with k capped as in
make_pins.py (the oracle pins cover exactly these cells).  Golden tables:
the `golden` / `tol` columns of oracle_pins.csv (themselves read from
data/golden/tableN.csv by make_pins.py), in the reference's golden CSV format
(tag,k,p,elements,value,tol).  Needs /root/reference (this container only).
Run: python tests/golden/make_table_fixtures.py"""
import csv
import json
from pathlib import Path

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/proj/data/config")
KMAX = {"table2": 1e5, "table3": 1e4, "table4": 1e4, "table5": 150, "table6": 150}

if __name__ == "__main__":
    out = HERE / "tables"
    out.mkdir(exist_ok=True)
    with open(HERE / "oracle_pins.csv") as fh:
        pins = list(csv.DictReader(fh))
    for name, kmax in KMAX.items():
        cfg = json.loads((REF / f"{name}.json").read_text())
        cfg.pop("_note", None)
        cfg["k"] = [k for k in cfg["k"] if float(k) <= kmax]
        (out / f"{name}.json").write_text(json.dumps(cfg, indent=2) + "\n")
        with open(out / f"{name}_golden.csv", "w", newline="") as fh:
            w = csv.writer(fh, lineterminator="\n")
            w.writerow(["tag", "k", "p", "elements", "value", "tol"])
            for r in pins:
                if r["table"] == name:
                    w.writerow([r["tag"], r["k"], r["p"], "", r["golden"], r["tol"]])
        print(name, len(cfg["k"]), "k values")
