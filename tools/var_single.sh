#!/bin/bash
# usage: var_single.sh "EXTRA1" "EXTRA2" ...
for ex in "$@"; do
  touch paper_1712_05012_b200/csrc/*.cu
  make -s -C paper_1712_05012_b200/csrc -j16 EXTRA="$ex" >/dev/null 2>&1 || { echo "build failed: $ex"; continue; }
  echo "== variant '$ex'"; python tools/single_rate.py --configs C2,C3 --iters 300 2>&1 | tail -2
done
touch paper_1712_05012_b200/csrc/*.cu; make -s -C paper_1712_05012_b200/csrc -j16 >/dev/null 2>&1
