"""Per-kernel DRAM bandwidth table from an ncu CSV (--metrics dram__bytes_read.sum,
dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --csv), as a fraction of the
measured HBM peak (MEASURED_PEAKS.json hbm_gbs).  Launch times under ncu are serialised and
cold-cache (ncu flushes caches before every launch), so this is each kernel's own roofline
position, not its share of a pipelined step.

    python tools/ncu_hbm_table.py LAUNCHES.csv [PEAK_GBS]
"""
import csv
import json
import os
import sys
from collections import defaultdict


def table(path, peak):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Name" in r)
    h = rows[hi]
    ki, mi, vi, ii, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID"),
                          h.index("Metric Unit"))
    per = defaultdict(dict)
    names = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki].split("(")[0].replace("mgnn::", "")
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0)
        a[3] += m.get("dram__bytes_write.sum", 0.0)
        a[4] += m.get("lts__t_bytes.sum", 0.0)
    out = [f"{'kernel':24s} {'n':>3s} {'avg us':>9s} {'DRAM MB/launch':>15s} {'DRAM GB/s':>10s} {'% HBM peak':>10s} {'L2 GB/s':>9s}"]
    for k, (n, t, rd, wr, l2) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = (rd + wr) / t / 1e9 if t else 0.0
        out.append(f"{k:24s} {n:3d} {1e6 * t / n:9.1f} {(rd + wr) / n / 1e6:15.1f} {gbs:10.0f} {100 * gbs / peak:9.1f}% "
                   f"{l2 / t / 1e9 if t else 0:9.0f}")
    return "\n".join(out)


if __name__ == "__main__":
    peak = float(sys.argv[2]) if len(sys.argv) > 2 else json.load(
        open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
    print(f"peak {peak} GB/s (MEASURED_PEAKS.json hbm_gbs)")
    print(table(sys.argv[1], peak))
