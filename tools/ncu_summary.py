"""Summaries of ncu outputs for profiles/ (run here, on the CPU side).

  python tools/ncu_summary.py launches <launches.csv>          per-launch table
  python tools/ncu_summary.py full <report.ncu-rep> [regex]    key metrics per kernel
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

KEY_METRICS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = defaultdict(dict)
    names = {}
    for r in rows[hdr + 1:]:
        d[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        names[int(r[ii])] = re.sub(r"\(.*", "", r[ki]).replace("void ", "").replace("ozk::<unnamed>::", "")
    print("| id | kernel | ms | DRAM read GB | DRAM write GB | SM GHz |")
    print("|---|---|---|---|---|---|")
    for i in sorted(d):
        v = d[i]
        print(f"| {i} | {names[i][:48]} | {v.get('gpu__time_duration.sum', 0) / 1e6:.3f} | "
              f"{v.get('dram__bytes_read.sum', 0) / 1e9:.2f} | {v.get('dram__bytes_write.sum', 0) / 1e9:.2f} | "
              f"{v.get('sm__cycles_elapsed.avg.per_second', 0) / 1e9:.2f} |")


def full(path, pattern=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        if pattern and not re.search(pattern, name):
            continue
        short = name.split("(")[0]
        print(f"### {short}")
        for m in KEY_METRICS:
            if m in h:
                i = h.index(m)
                print(f"- {m}: {r[i]} {units[i]}")
        print()


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
