for ex in "$@"; do
  touch paper_1712_05012_b200/csrc/*.cu
  make -s -C paper_1712_05012_b200/csrc -j16 EXTRA="$ex" >/dev/null 2>&1 || { echo "build failed: $ex"; continue; }
  echo "== '$ex' $(python tools/kernel_lat.py --config C2 2>&1 | tail -1)"
  python tools/single_rate.py --configs C2 --iters 300 | sed "s/^/== '$ex' /"
done
touch paper_1712_05012_b200/csrc/*.cu; make -s -C paper_1712_05012_b200/csrc -j16 >/dev/null 2>&1
