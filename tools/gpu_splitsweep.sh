# cluster split sweep at small batches
for B in 64 128; do for S in 2 4 8; do KFB200_CL_SPLIT=$S python tools/ens_rate.py $B 16; done; done
