#!/bin/bash
# Build compile-time variants and report ncu per-launch kernel times (mean us)
# for the kernels matching REGEX on a phase_times workload.
#   bash tools/kernel_variants.sh REGEX "ARGS" "" "-DFOO=1" ...
re="$1"; args="$2"; shift 2
for ex in "$@"; do
  touch paper_1712_05012_b200/csrc/*.cu
  make -s -C paper_1712_05012_b200/csrc -j16 EXTRA="$ex" >/dev/null 2>&1 || { echo "build failed: $ex"; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$re" --csv --log-file /tmp/kv.csv \
      python tools/phase_times.py $args > /dev/null 2>&1
  python - "$ex" <<'PY'
import csv, io, sys
from collections import defaultdict
t = open("/tmp/kv.csv").read(); t = t[t.find('"ID"'):]
per = defaultdict(list)
for r in csv.DictReader(io.StringIO(t)):
    if r.get("Metric Name") != "gpu__time_duration.sum": continue
    v = float(r["Metric Value"].replace(",", "")); u = r.get("Metric Unit")
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
    per[r["Kernel Name"].split("(")[0].replace("<unnamed>::", "")].append(v)
print(f"variant {sys.argv[1]!r}: " + ", ".join(f"{k} {sum(v)/len(v):.1f} us" for k, v in per.items()))
PY
done
touch paper_1712_05012_b200/csrc/*.cu
make -s -C paper_1712_05012_b200/csrc -j16 >/dev/null 2>&1
