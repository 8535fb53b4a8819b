# predicated solvation walk (cur) vs branchy walk (base): parity + C5 water A/B
python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -x -q -k "solv or water or sasa or exposure" 2>&1 | tail -1
for rep in 1 2; do
  WATER=1 python tools/ens_rate.py 1024 4 | sed 's/env={.*}//;s/^/cur /'
  WATER=1 KFB200_LIB=$PWD/_variants/base.so python tools/ens_rate.py 1024 4 | sed 's/env={.*}//;s/^/base /'
done
