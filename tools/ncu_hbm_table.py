"""Per-kernel DRAM bandwidth table from an ncu CSV (--metrics dram__bytes_read.sum,
dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum --csv), as a fraction of the
measured HBM peak (MEASURED_PEAKS.json hbm_gbs).  Launch times under ncu are serialised and
cold-cache (ncu flushes caches before every launch), so this is each kernel's own roofline
position, not its share of a pipelined step.

    python tools/ncu_hbm_table.py LAUNCHES.csv [PEAK_GBS] [--json OUT --config NAME]

--json writes the per-config traffic table bench.py reads (profiles/r02/traffic_<config>.json):
per kernel the DRAM bytes per launch (the roofline line's `traffic`), the duration and the fraction
of the peak.  Capture it with `--cache-control none` so the bytes are the kernel's in-situ traffic.
"""
import csv
import json
import os
import sys
from collections import defaultdict


def aggregate(path):
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
        names[r[ii]] = r[ki].split("(")[0].replace("mgnn::", "").replace("void ", "").split("<")[0]
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0)
        a[3] += m.get("dram__bytes_write.sum", 0.0)
        a[4] += m.get("lts__t_bytes.sum", 0.0)
    return agg


def table(path, peak):
    agg = aggregate(path)
    out = [f"{'kernel':24s} {'n':>3s} {'avg us':>9s} {'DRAM MB/launch':>15s} {'DRAM GB/s':>10s} {'% HBM peak':>10s} {'L2 GB/s':>9s}"]
    for k, (n, t, rd, wr, l2) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = (rd + wr) / t / 1e9 if t else 0.0
        out.append(f"{k:24s} {n:3d} {1e6 * t / n:9.1f} {(rd + wr) / n / 1e6:15.1f} {gbs:10.0f} {100 * gbs / peak:9.1f}% "
                   f"{l2 / t / 1e9 if t else 0:9.0f}")
    return "\n".join(out)


def traffic_json(path, peak, config, out):
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    head = os.environ.get("MGNN_GIT_HEAD") or subprocess.run(   # the GPU box has no .git: passed in
        ["git", "rev-parse", "--short=12", "HEAD"], cwd=root, capture_output=True, text=True).stdout.strip()
    d = {"config": config, "source": os.path.relpath(path, root), "git_head": head,
         "note": "ncu --cache-control none --clock-control none launch list: dram__bytes_read.sum + "
                 "dram__bytes_write.sum per launch (serialised launches), averaged per kernel",
         "peak_gbs": peak, "kernels": {}}
    for k, (n, t, rd, wr, _) in aggregate(path).items():
        d["kernels"][k] = {"launches": n, "us_per_launch": 1e6 * t / n, "dram_bytes_per_launch": (rd + wr) / n,
                           "frac_of_peak": (rd + wr) / t / 1e9 / peak if t else None}
        if k.startswith("k_gather") or k.startswith("k_hop") or k in ("k_compact", "k_relabel"):
            d[k] = (rd + wr) / n
    with open(out, "w") as f:
        json.dump(d, f, indent=1)


if __name__ == "__main__":
    args = [a for a in sys.argv[1:]]
    js = cfg = None
    if "--json" in args:
        js = args[args.index("--json") + 1]
        cfg = args[args.index("--config") + 1]
        args = [a for a in args if a not in ("--json", js, "--config", cfg)]
    peak = float(args[1]) if len(args) > 1 else json.load(
        open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
    print(f"peak {peak} GB/s (MEASURED_PEAKS.json hbm_gbs)")
    print(table(args[0], peak))
    if js:
        traffic_json(args[0], peak, cfg, js)
