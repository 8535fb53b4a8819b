#!/bin/bash
# Rebuild with solvation-kernel variants and time the water step per phase.
#   bash tools/time_solv.sh "" "-DSOLV_GROUP_THREADS=128"
set -e
for ex in "$@"; do
  touch paper_1712_05012_b200/csrc/kf_solvation.cu
  make -s -C paper_1712_05012_b200/csrc -j16 EXTRA="$ex" >/dev/null 2>&1
  echo "variant: '$ex'"
  python tools/phase_times.py --config C2 --ensemble 64 --water --iters 8 | grep -o "solv.: [0-9.]*"
  python tools/phase_times.py --config C3 --ensemble 1 --water --iters 8 | grep -o "solv.: [0-9.]*"
done
touch paper_1712_05012_b200/csrc/kf_solvation.cu
make -s -C paper_1712_05012_b200/csrc -j16 >/dev/null 2>&1
