#!/bin/bash
# Golden run outputs of the reference CLI, made in the build
# container where /root/reference exists:  bash tests/golden/make_fold_batch.sh
set -e
tmp=$(mktemp -d)
( cd "$tmp" && PYTHONPATH=/root/reference/pkg/src python -m kinefold.cli fold \
    --seq "ALA CYS SER ALA GLY ALA SER CYS ALA ALA" --init random --seed 3 --batch 2 \
    --max-iters 25 --snapshot-every 10 --out out )
dst="$(dirname "$0")/fold_batch"
for f in summary.csv run_0000/log.csv run_0000/dihedrals.csv run_0000/final.pdb run_0000/snap_000010.pdb \
         run_0001/log.csv run_0001/dihedrals.csv run_0001/final.pdb; do
  mkdir -p "$dst/$(dirname "$f")"
  cp "$tmp/out/$f" "$dst/$f"
done
rm -rf "$tmp"
