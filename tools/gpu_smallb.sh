# small batches: graph-branch floor 64 (default) vs 32
for B in 64 128; do
  python tools/ens_rate.py $B 16
  KFB200_BRANCH_MIN=32 python tools/ens_rate.py $B 16
done
