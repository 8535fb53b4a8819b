for ex in "$@"; do
  touch paper_1712_05012_b200/csrc/*.cu
  make -s -C paper_1712_05012_b200/csrc -j16 EXTRA="$ex" >/dev/null 2>&1 || { echo "build failed: $ex"; continue; }
  for B in 64 128 256; do echo "== '$ex' $(python tools/kernel_lat.py --config C2 --ensemble $B 2>&1 | tail -1)"; done
done
