"""Top SASS instructions of an ncu report by warp-stall samples (needs --import-source / -lineinfo).

    python tools/ncu_hot.py REPORT [N] [KERNEL_INDEX]
KERNEL_INDEX picks one of several profiled launches (0-based, in report order)."""
import csv
import subprocess
import sys


def hot(path, n=30, which=0):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] or [0]
    lo = starts[which]
    hi_end = starts[which + 1] if which + 1 < len(starts) else len(rows)
    name = rows[lo][1] if rows[lo] and rows[lo][0] == "Kernel Name" else "?"
    hi = next(i for i in range(lo, hi_end) if "Address" in rows[i] and "Source" in rows[i])
    hdr = rows[hi]
    si, wi, ii = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    data = []
    for r in rows[hi + 1:hi_end]:
        try:
            data.append((int(r[wi] or 0), int(r[ii] or 0), r[si].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    toti = sum(d[1] for d in data)
    lines = [f"{name}: stall samples {tot}, warp-instructions executed {toti}"]
    for d in sorted(data, reverse=True)[:n]:
        lines.append(f"{d[0]:7d} {100 * d[0] / tot:5.1f}%  inst {d[1]:9d}  {d[2][:80]}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(hot(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30, int(sys.argv[3]) if len(sys.argv) > 3 else 0))
