"""Summarise an ncu --csv metrics log (gpu__time_duration, dram bytes) per kernel: launches,
mean time, mean DRAM bytes, achieved GB/s and fraction of MEASURED_PEAKS.json hbm_gbs (dev tool)."""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def table(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    H = rows[h]
    ki, mi, vi, idi = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value"), H.index("ID")
    d, names = collections.defaultdict(dict), {}
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        d[r[idi]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[idi]] = r[ki].split("(")[0].replace("(anonymous namespace)::", "").replace("unnamed>::", "").replace("void ", "")
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in d.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6444.7
    total = sum(a[1] for a in agg.values())
    out = ["| kernel | launches | mean us | share | DRAM MB / launch | GB/s | frac of HBM |", "|---|---|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        t = a[1] / a[0] / 1e3  # us
        b = a[2] / a[0]
        out.append(f"| `{k}` | {a[0]} | {t:.2f} | {100 * a[1] / total:.1f}% | {b / 1e6:.2f} | {b / (t * 1e3):.0f} | {b / (t * 1e3) / pk:.2f} |")
    return "\n".join(out)


if __name__ == "__main__":
    print(table(sys.argv[1]))
