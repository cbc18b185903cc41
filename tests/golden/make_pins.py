"""Pins the oracle against the reference's golden iteration tables.

Runs the oracle over the sweep configs of /root/reference/proj/data/config
(table2/3/4: 1D, table5/6: 2D, capped k ranges as shipped) and compares every
cell with data/golden/table{2..6}.csv under the reference's own compare rule
(src/harness.cpp:547-592: |iterations - golden| <= per-row tol or the config's
compare.tolerance; '*' golden = not converged).  Writes oracle_pins.csv.

Needs /root/reference (this container only); the CSV is committed and checked
by tests/test_oracle_pins.py.  Run: python tests/golden/make_pins.py [table...]
"""
import csv
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import helmdef_oracle as O  # noqa: E402

REF = Path("/root/reference/proj/data")
OUT = Path(__file__).resolve().parent / "oracle_pins.csv"
TABLES = {"table2": 1e5, "table3": 1e4, "table4": 1e4, "table5": 150, "table6": 150}


def fmt(k):
    return str(int(k)) if float(k).is_integer() else repr(k)


def run_table(name, kmax):
    cfg = json.loads((REF / "config" / f"{name}.json").read_text())
    golden = {}
    with open(REF / "golden" / f"{name}.csv") as fh:
        rows = [r for r in fh if not r.startswith("#")]
    for r in csv.DictReader(rows):
        golden[(r["tag"], fmt(float(r["k"])), int(r["p"]))] = (r["value"], r.get("tol") or "")
    deftol = cfg.get("compare", {}).get("tolerance", 2)
    out = []
    for pc in cfg["preconditioners"]:
        tag = pc["tag"]
        label = O.label(tag, pc.get("cycles", 1))
        for p in cfg["p"]:
            for k in cfg["k"]:
                k = float(k)
                if k > kmax:
                    continue
                ne = O.derived_elements(k, cfg.get("kh", 0.625), p)
                spec = O.to_spec(tag, p, k, epsilon=pc.get("epsilon", 0.1), beta2=str(pc.get("beta2", "1")),
                                 cycles=pc.get("cycles", 1), smoothing=pc.get("smoothing", 1),
                                 omega=pc.get("omega", 0.6),
                                 smoothing_by_p={int(a): b for a, b in pc.get("smoothing_by_p", {}).items()},
                                 omega_by_p={int(a): b for a, b in pc.get("omega_by_p", {}).items()})
                t = time.perf_counter()
                rec, gr, _ = O.run_cell(cfg["problem"], spec, p, k, ne,
                                        O.GmresOptions(cfg["gmres"]["max_iterations"], cfg["gmres"]["tolerance"]),
                                        multipliers=cfg.get("multipliers"))
                g = golden.get((label, fmt(k), p))
                if g is None:
                    continue
                gval, gtol = g
                tol = float(gtol) if gtol else float(deftol)
                if gval == "*":
                    ok = not gr.converged
                else:
                    ok = gr.converged and abs(gr.iterations - int(gval)) <= tol
                out.append(dict(table=name, tag=label, k=fmt(k), p=p, elements=ne, golden=gval, tol=tol,
                                oracle=gr.iterations, converged=int(gr.converged), ok=int(ok),
                                seconds=round(time.perf_counter() - t, 2)))
                print(out[-1], flush=True)
    return out


if __name__ == "__main__":
    names = sys.argv[1:] or list(TABLES)
    rows = []
    if OUT.exists():
        with open(OUT) as fh:
            rows = [r for r in csv.DictReader(fh) if r["table"] not in names]
    for n in names:
        rows += run_table(n, TABLES[n])
    keys = ["table", "tag", "k", "p", "elements", "golden", "tol", "oracle", "converged", "ok", "seconds"]
    with open(OUT, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=keys)
        w.writeheader()
        for r in rows:
            w.writerow({k: r[k] for k in keys})
