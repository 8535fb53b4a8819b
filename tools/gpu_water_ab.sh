# water-mode ensemble rate A/B of built variants (args)
for rep in 1 2; do for v in cur "$@"; do
  if [ "$v" = cur ]; then WATER=1 python tools/ens_rate.py 1024 4 | sed "s/^/cur /";
  else KFB200_LIB=$PWD/_variants/$v.so WATER=1 python tools/ens_rate.py 1024 4 | sed "s/^/$v /"; fi
done; done
