# water-mode parity tests, then the water ensemble rate for built variants (args)
python -m pytest tests -m gpu -q -x -k "water or solv or sasa or bin or grid or hash" 2>&1 | tail -2
for v in cur "$@"; do
  if [ "$v" = cur ]; then WATER=1 python tools/ens_rate.py 1024 4 | sed "s/^/cur /";
  else KFB200_LIB=$PWD/_variants/$v.so WATER=1 python tools/ens_rate.py 1024 4 | sed "s/^/$v /"; fi
done
