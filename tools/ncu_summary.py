"""Summarise an ncu report (--set full) or a launch-list CSV for profiles/.

    python tools/ncu_summary.py report.ncu-rep [out.txt]
    python tools/ncu_summary.py --launches launches.csv [out.txt]
"""

from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__warps_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warps_issue_stalled_wait_per_warp_active.pct",
    "smsp__warps_issue_stalled_short_scoreboard_per_warp_active.pct",
    "smsp__warps_issue_stalled_branch_resolving_per_warp_active.pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def report(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        out.append(f"kernel: {d.get('Kernel Name', '?')[:100]}")
        for k in KEYS:
            if k in d:
                out.append(f"  {k:70s} {d[k]:>18s} {u.get(k, '')}")
        dr, dw = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        if dr and dw:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            tot = float(dr.replace(",", "")) * scale.get(u.get("dram__bytes_read.sum"), 1) + \
                float(dw.replace(",", "")) * scale.get(u.get("dram__bytes_write.sum"), 1)
            out.append(f"  {'dram traffic (read + write), bytes':70s} {tot:18.0f}")
    return "\n".join(out) + "\n"


def launches(path: str) -> str:
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    per = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        if r.get("Metric Unit") == "usecond":
            v *= 1e3
        elif r.get("Metric Unit") == "msecond":
            v *= 1e6
        per[r["Kernel Name"].split("(")[0]].append(v)
    tot = sum(sum(v) for v in per.values()) or 1.0
    lines = [f"{'kernel':60s} {'launches':>8s} {'total ns':>14s} {'share':>7s}"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:60]:60s} {len(v):8d} {sum(v):14.0f} {sum(v) / tot * 100:6.1f}%")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        text = launches(sys.argv[2])
        dest = sys.argv[3] if len(sys.argv) > 3 else None
    else:
        text = report(sys.argv[1])
        dest = sys.argv[2] if len(sys.argv) > 2 else None
    if dest:
        open(dest, "w").write(text)
    print(text)
