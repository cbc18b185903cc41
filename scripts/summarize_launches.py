"""Summarise an `ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum,...] --csv`
launch list: share, count, mean duration and (when captured) DRAM bytes per kernel
(cold-cache, serialised: compare SHARES)."""
import collections
import csv
import sys

UNITS = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}


def summarise(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    bunit = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0]
        metric = r[mi] if mi is not None else "gpu__time_duration.sum"
        val = float(r[vi].replace(",", ""))
        if metric == "gpu__time_duration.sum":
            agg[name][0] += 1
            agg[name][1] += val * UNITS.get(r[ui], 1.0)
        elif metric.startswith("dram__bytes"):
            agg[name][2] += val * bunit.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    has_b = any(v[2] > 0 for v in agg.values())
    out = [f"launches: {sum(v[0] for v in agg.values())}, total device time {tot/1e3:.2f} ms (ncu, serialised)",
           "| share | launches | mean us |" + (" DRAM GB/s | DRAM MB/launch |" if has_b else "") + " kernel |",
           "|---:|---:|---:|" + ("---:|---:|" if has_b else "") + "---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        extra = f" {v[2] / (v[1] * 1e-6) / 1e9:.0f} | {v[2] / v[0] / 1e6:.1f} |" if has_b else ""
        out.append(f"| {v[1]/tot*100:.2f}% | {v[0]} | {v[1]/v[0]:.2f} |{extra} `{k}` |")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
