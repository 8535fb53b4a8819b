# single-trajectory C1 / C2 rates: dense path vs the split cluster path (S = 4 / 8 / 16)
python tools/single_rate.py --configs C1,C2 --iters 200
KFB200_CLUSTER_MIN_B=1 python tools/single_rate.py --configs C2 --iters 200
KFB200_CLUSTER_MIN_B=1 KFB200_CL_SPLIT=16 python tools/single_rate.py --configs C1,C2 --iters 200
KFB200_CLUSTER_MIN_B=1 KFB200_CL_SPLIT=4 python tools/single_rate.py --configs C1,C2 --iters 200
