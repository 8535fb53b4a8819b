# FK CTA width A/B: C5 at B = 128 / 1024 and single-trajectory C1 / C2
for rep in 1 2; do for v in cur fk256 fk512; do
  if [ $v = cur ]; then L=""; else L=$PWD/_variants/$v.so; fi
  for B in 128 1024; do KFB200_LIB=$L python tools/ens_rate.py $B 16 | sed "s/^/$v /"; done
  KFB200_LIB=$L python tools/single_rate.py --configs C1,C2 --iters 300 | sed "s/^/$v /"
done; done
