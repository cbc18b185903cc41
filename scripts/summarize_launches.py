"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: share,
count and mean duration per kernel (cold-cache, serialised: compare SHARES)."""
import collections
import csv
import sys

UNITS = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}


def summarise(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"launches: {sum(v[0] for v in agg.values())}, total device time {tot/1e3:.2f} ms (ncu, serialised)",
           "| share | launches | mean us | kernel |", "|---:|---:|---:|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        out.append(f"| {v[1]/tot*100:.2f}% | {v[0]} | {v[1]/v[0]:.2f} | `{k}` |")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
