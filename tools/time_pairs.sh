#!/bin/bash
# Rebuild with pair-kernel occupancy variants and time the C5 ensemble step per phase.
set -e
for mb in "$@"; do
  sed -i "s/__launch_bounds__(PAIR_WARPS \* 32, SPLIT ? PAIR_MINB : [0-9])/__launch_bounds__(PAIR_WARPS * 32, SPLIT ? PAIR_MINB : $mb)/" paper_1712_05012_b200/csrc/kf_nonbonded.cu
  make -s -C paper_1712_05012_b200/csrc -j16 >/dev/null 2>&1
  echo "minblocks=$mb"
  python tools/phase_times.py --config C2 --ensemble 1024 --iters 8
done
