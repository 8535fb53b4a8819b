# vdW-reach lean visits without the fp32-path vote (cur) vs with it (vote1)
python -m pytest tests/test_gpu_bench_parity.py -x -q 2>&1 | tail -1
bash tools/ab.sh 1024 16 cur vote1 2>&1 | sed 's/env={.*}//'
