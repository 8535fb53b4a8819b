#!/bin/bash
# Rebuild with a pair-kernel variant and time one eager ensemble iteration per phase.
set -e
for mb in "$@"; do
  make -s -C paper_1712_05012_b200/csrc clean >/dev/null
  make -s -C paper_1712_05012_b200/csrc EXTRA=-DPAIR_MINB=$mb -j16 >/dev/null 2>&1
  echo "PAIR_MINB=$mb"
  python bench.py --steps 10 --warmup 3 --no-extras | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['phase_ms_per_step'])"
done
