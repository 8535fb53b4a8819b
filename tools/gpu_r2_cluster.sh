python -m pytest tests/test_gpu_bench_parity.py -q -x 2>&1 | tail -2
python tools/ens_rate.py 1024 16
for v in w12b2 w16b1; do KFB200_LIB=$PWD/_variants/$v.so python tools/ens_rate.py 1024 16 | sed "s/^/$v /"; done
python tools/ens_rate.py 128 16
