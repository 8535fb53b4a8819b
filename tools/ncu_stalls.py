"""Stall-reason totals and the top stalled SASS instructions of an ncu report.

    python tools/ncu_stalls.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys
from collections import Counter

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ix = {h: hdr.index(h) for h in cols}
ie = hdr.index("Instructions Executed")
tot = Counter()
per = []
for r in data:
    if len(r) <= ie:
        continue
    s = {h: int(r[ix[h]]) for h in cols if r[ix[h]].isdigit()}
    tot.update(s)
    per.append((sum(s.values()), r[1].strip()[:60], int(r[ie]) if r[ie].isdigit() else 0,
                max(s, key=s.get) if s else ""))
T = sum(tot.values()) or 1
print("stall samples by reason:")
for k, v in tot.most_common(10):
    print(f"  {k:24s} {v / T * 100:5.1f}%")
print("top instructions:")
for smp, txt, ex, why in sorted(per, reverse=True)[:top]:
    print(f"  {smp / T * 100:5.1f}% {ex:>10} {why:22s} {txt}")
