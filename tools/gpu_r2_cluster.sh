python tools/ens_rate.py 1024 16
for v in w16b1 w24b1 w12b2 w32b1; do KFB200_LIB=$PWD/_variants/$v.so python tools/ens_rate.py 1024 16 | sed "s/^/$v /"; done
