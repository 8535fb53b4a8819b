python -m pytest tests/test_gpu_bench_parity.py -q -x 2>&1 | tail -3
python -m pytest tests -m gpu -q -x -k "cluster or half_list or clash or ensemble" 2>&1 | tail -3
bash tools/ab.sh 1024 16 cur old
