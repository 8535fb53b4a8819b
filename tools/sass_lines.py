"""SASS instructions per source line of one kernel (nvdisasm -g output).

usage: python tools/sass_lines.py file.sass KERNEL_SUBSTR [--ops]
"""
import re
import sys
from collections import Counter, defaultdict

path, kern = sys.argv[1], sys.argv[2]
ops = "--ops" in sys.argv
cur_line, inside = None, False
per_line = Counter()
op_by_line = defaultdict(Counter)
for raw in open(path):
    if raw.startswith(".text.") or "//----" in raw and ".text." in raw:
        inside = kern in raw
        continue
    if not inside:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', raw)
    if "## File" in raw and m:
        cur_line = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r'\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)', raw)
    if m:
        per_line[cur_line] += 1
        op_by_line[cur_line][m.group(2).split(".")[0]] += 1
total = sum(per_line.values())
print("total", total)
for ln in sorted(per_line, key=lambda x: (x or ('', 0))):
    extra = " ".join(f"{k}:{v}" for k, v in op_by_line[ln].most_common(6)) if ops else ""
    print(f"{ln[0]}:{ln[1]:<5d} {per_line[ln]:5d} {extra}")
