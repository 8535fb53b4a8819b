# trajectory split over a thread-block cluster at small B: parity, then rates vs split = 1
python -m pytest tests/test_gpu_bench_parity.py -q -x 2>&1 | tail -2
for B in 16 32 64 128 256; do
  KFB200_CLUSTER_MIN_B=1 python tools/ens_rate.py $B 16
  KFB200_CLUSTER_MIN_B=1 KFB200_CL_SPLIT=1 python tools/ens_rate.py $B 16
done
python tools/ens_rate.py 1024 16
