# FK variants A/B (fkold = committed build): phase clocks, C5 B = 128 / 1024, single C1 / C2
for v in fkt fkt12; do KFB200_LIB=$PWD/_variants/$v.so python tools/phase_times.py --ensemble 1 --iters 6 2>&1 | grep FKT | tail -1 | sed "s/^/$v /"; done
for rep in 1 2; do for v in cur fkold pu12 l1pf both; do
  if [ $v = cur ]; then L=""; else L=$PWD/_variants/$v.so; fi
  for B in 128 1024; do KFB200_LIB=$L python tools/ens_rate.py $B 16 | sed "s/^/$v /"; done
  KFB200_LIB=$L python tools/single_rate.py --configs C1,C2 --iters 300 | sed "s/^/$v /"
done; done
