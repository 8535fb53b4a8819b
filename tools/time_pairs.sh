#!/bin/bash
# Rebuild the library with compile-time variants and time C2 ensembles per phase.
#   bash tools/time_pairs.sh "" "-DPAIR_MINB_W=5" "-DRES_BATCH_N=64"
set -e
for ex in "$@"; do
  touch paper_1712_05012_b200/csrc/kf_nonbonded.cu
  make -s -C paper_1712_05012_b200/csrc -j16 EXTRA="$ex" >/dev/null 2>&1
  echo "variant: '$ex'"
  python tools/phase_times.py --config C2 --ensemble 256 --iters 10 | tail -1
  python tools/phase_times.py --config C2 --ensemble 1024 --iters 10 | tail -1
done
touch paper_1712_05012_b200/csrc/kf_nonbonded.cu
make -s -C paper_1712_05012_b200/csrc -j16 >/dev/null 2>&1
