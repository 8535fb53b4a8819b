# A/B of environment switches on the C5 ensemble rate: tools/gpu_envab.sh "ENV1=.." "ENV2=.." ...
for rep in 1 2; do
  python tools/ens_rate.py 1024 16 | sed "s/^/base /"
  for e in "$@"; do env $e python tools/ens_rate.py 1024 16 | sed "s/^/$e /"; done
done
