python -m pytest tests/test_gpu_bench_parity.py -q -x 2>&1 | tail -2
python tools/ens_rate.py 1024 16
KFB200_LIB=$PWD/_variants/w12b2.so python tools/ens_rate.py 1024 16
python tools/ens_rate.py 256 16
