#!/bin/bash
# Build compile-time variants of the library and run a command on each with a timeout.
#   bash tools/variants_dbg.sh "<cmd>" "" "-DFOO" ...
cmd="$1"; shift
for ex in "$@"; do
  touch paper_1712_05012_b200/csrc/kf_nonbonded.cu
  make -s -C paper_1712_05012_b200/csrc -j16 EXTRA="$ex" >/dev/null 2>&1 || { echo "build failed: $ex"; continue; }
  for i in 1 2 3; do
    timeout 40 bash -c "$cmd" > /tmp/v.log 2>&1; rc=$?
    echo "variant '$ex' run $i rc=$rc $(tail -1 /tmp/v.log | cut -c1-120)"
  done
done
touch paper_1712_05012_b200/csrc/kf_nonbonded.cu
make -s -C paper_1712_05012_b200/csrc -j16 >/dev/null 2>&1
