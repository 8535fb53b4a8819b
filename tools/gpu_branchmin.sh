# graph branches at small batches: sub-batch floor 256 (default) vs 64 / 32
for B in 128 256 512; do
  python tools/ens_rate.py $B 16
  KFB200_BRANCH_MIN=64 python tools/ens_rate.py $B 16
  KFB200_BRANCH_MIN=32 python tools/ens_rate.py $B 16
done
