# cluster-path batch threshold sweep: dense half list vs cluster pairs at small B
for B in 32 64 96 128 160; do
  python tools/ens_rate.py $B 16
  KFB200_CLUSTER_MIN_B=16 python tools/ens_rate.py $B 16
done
