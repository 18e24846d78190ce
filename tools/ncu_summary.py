"""Summarise ncu output brought back in gpurun_out/ into profiles/ (dev tool).

    python tools/ncu_summary.py <tag> [launches.csv] [full.ncu-rep]

Writes profiles/<tag>_launches.md (per-kernel share of device time from the
`--metrics gpu__time_duration.sum` launch list), profiles/<tag>_interior_solve.md (key
metrics of the `--set full` capture) and profiles/interior_solve_traffic.json (DRAM bytes
per interior-solve launch, read by bench.py as roofline.traffic).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__cluster_dim_x", "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
        "sm__cycles_elapsed.avg", "smsp__cycles_active.avg"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi, ui = h.index("Metric Name"), h.index("Metric Unit")
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hdr + 1:]:
        # one row per (launch, metric): only the duration rows count (a log with DRAM metrics too)
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        name = name.split("(")[0]
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)  # ns
        cnt[name] += 1
    T = sum(tot.values())
    out = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| `{k}` | {cnt[k]} | {v / 1e3:.1f} | {v / 1e3 / cnt[k]:.1f} | {100 * v / T:.1f}% |")
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        rec = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("unnamed>::", "")}
        for k in KEYS:
            if k in h:
                rec[k] = (r[h.index(k)], units[h.index(k)])
        recs.append(rec)
    return recs


def mbytes(v):
    val, unit = v
    x = float(val.replace(",", ""))
    return x * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)


def main():
    tag = sys.argv[1]
    lpath = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", "launches.csv")
    fpath = sys.argv[3] if len(sys.argv) > 3 else None
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if os.path.exists(lpath):
        with open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w") as f:
            f.write(f"# {tag}: device time per kernel (ncu gpu__time_duration.sum, --clock-control none)\n\n")
            cmd = os.environ.get("NCU_CMD", "python bench.py --steps 2 --warmup 3 --no-cpu-baseline")
            f.write(f"Cold-cache, serialised launches of `{cmd}`;\ncompare shares, not absolutes.\n\n")
            f.write(launches(lpath) + "\n")
    if fpath and os.path.exists(fpath):
        recs = full(fpath)
        lines = [f"# {tag}: `ncu --set full` of the interior solve (C2, 64 subdomains)\n"]
        for r in recs:
            lines.append(f"## `{r['kernel']}`\n")
            lines.append("| metric | value |\n|---|---|")
            for k in KEYS:
                if k in r:
                    lines.append(f"| {k} | {r[k][0]} {r[k][1]} |")
            lines.append("")
        with open(os.path.join(ROOT, "profiles", f"{tag}_interior_solve.md"), "w") as f:
            f.write("\n".join(lines) + "\n")
        solves = [r for r in recs if "interior_solve" in r["kernel"]]
        per = sum(mbytes(r["dram__bytes_read.sum"]) + mbytes(r["dram__bytes_write.sum"]) for r in solves) / len(solves)
        json.dump({"tag": tag, "kernel": "interior_solve_kernel", "launches": len(solves),
                   "dram_bytes_per_launch": per * 1e6,
                   "source": f"profiles/{tag}_interior_solve.md (ncu --set full, dram__bytes_read.sum + "
                             f"dram__bytes_write.sum, mean over captured launches)"},
                  open(os.path.join(ROOT, "profiles", "interior_solve_traffic.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
