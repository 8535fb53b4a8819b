# lean-unit operands staged through shared memory: 16-byte slot (cur), 8-byte slot (stage8), none (nostage)
KFB200_LIB=$PWD/_variants/stage8.so python -m pytest tests/test_gpu_bench_parity.py -x -q 2>&1 | tail -1
bash tools/ab.sh 1024 16 cur stage8 nostage 2>&1 | sed 's/env={.*}//'
bash tools/ab.sh 128 16 cur stage8 nostage 2>&1 | sed 's/env={.*}//'
