# rank sort by the sign of key differences (cur) vs compare + predicated add (base)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -x -q -k "solv or water or sasa or exposure" 2>&1 | tail -1
for rep in 1 2; do for v in cur base; do
  if [ $v = cur ]; then L=""; else L=$PWD/_variants/$v.so; fi
  WATER=1 KFB200_LIB=$L python tools/ens_rate.py 1024 4 | sed "s/env={.*}//;s/^/$v /"
done; done
