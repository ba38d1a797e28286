"""Key metrics of an ncu --set full report (raw page), one line per launch."""
import csv
import subprocess
import sys

WANT = [
    ("Kernel Name", "kernel"), ("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("lts__t_bytes.sum", "l2_bytes"), ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"), ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"), ("launch__block_size", "block"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall_lsb"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall_bar"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall_lgthr"),
]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    cols = [(hdr.index(k), name) for k, name in WANT if k in hdr]
    lines = ["  ".join(f"{name}[{units[i]}]" for i, name in cols)]
    for r in rows[2:]:
        lines.append("  ".join(r[i][:28] for i, _ in cols))
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        print(summarise(p))
