# single-trajectory C1 / C2: separate kernels vs the fused iteration kernel (split 1)
python tools/single_rate.py --configs C1,C2 --iters 1000 | sed 's/^/base /'
KFB200_CL_SPLIT=1 python tools/single_rate.py --configs C1,C2 --iters 1000 | sed 's/^/split1 /'
KFB200_CL_SPLIT=1 KFB200_FUSED=1 python tools/single_rate.py --configs C1,C2 --iters 1000 | sed 's/^/fused /'
KFB200_CL_SPLIT=1 KFB200_FUSED=2 python tools/single_rate.py --configs C1,C2 --iters 1000 | sed 's/^/fkpairs /'
