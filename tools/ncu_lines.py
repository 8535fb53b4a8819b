"""Per-CUDA-source-line instruction counts and stall samples from an ncu report.

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows, fname, hdr = [], None, None
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "" or r[0] == "Function Name":
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        ins, samp = int(d["Instructions Executed"]), int(d["Warp Stall Sampling (All Samples)"])
    except (KeyError, ValueError):
        continue
    rows.append((ins, samp, f"{fname}:{r[0]}", r[1].strip()[:90]))
ti = sum(x[0] for x in rows) or 1
ts = sum(x[1] for x in rows) or 1
print(f"total warp instructions {ti}, stall samples {ts}")
for ins, samp, loc, src in sorted(rows, key=lambda x: -x[1])[:top]:
    print(f"{ins / ti * 100:6.2f}% inst {samp / ts * 100:6.2f}% samples  {loc:22s} {src}")
