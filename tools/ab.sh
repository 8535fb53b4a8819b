# A/B: alternate builds in one call (same box): tools/ab.sh B K name1 name2 ...
B=$1; K=$2; shift 2
for rep in 1 2; do for v in "$@"; do
  if [ "$v" = cur ]; then python tools/ens_rate.py $B $K | sed "s/^/cur /"; else KFB200_LIB=$PWD/_variants/$v.so python tools/ens_rate.py $B $K | sed "s/^/$v /"; fi
done; done
