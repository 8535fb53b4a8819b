# parity of the ensemble kernels, then an A/B of built variants (args: variant names)
python -m pytest tests/test_gpu_bench_parity.py -q -x 2>&1 | tail -2
bash tools/ab.sh 1024 16 cur "$@"
