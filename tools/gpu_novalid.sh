# no atom-exists tests outside the own-octet visits (cur) vs tested (base)
python -m pytest tests/test_gpu_bench_parity.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
bash tools/ab.sh 1024 16 cur base 2>&1 | sed 's/env={.*}//'
bash tools/ab.sh 128 16 cur base 2>&1 | sed 's/env={.*}//'
