# B = 128 configurations: branch floor and cluster split
for rep in 1 2; do
python tools/ens_rate.py 128 16 | sed 's/env={.*}//;s/^/base /'
KFB200_BRANCH_MIN=32 python tools/ens_rate.py 128 16 | sed 's/env={.*}//;s/^/min32 /'
KFB200_CL_SPLIT=2 python tools/ens_rate.py 128 16 | sed 's/env={.*}//;s/^/split2 /'
KFB200_CL_SPLIT=8 python tools/ens_rate.py 128 16 | sed 's/env={.*}//;s/^/split8 /'
KFB200_BRANCHES=1 python tools/ens_rate.py 128 16 | sed 's/env={.*}//;s/^/nobr /'
done
