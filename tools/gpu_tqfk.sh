# torque + next-iteration FK in one kernel (KFB200_TQFK=1) vs separate kernels
KFB200_TQFK=1 python -m pytest tests/test_gpu_bench_parity.py -x -q 2>&1 | tail -2
for rep in 1 2; do
  for B in 128 1024; do
    python tools/ens_rate.py $B 16 | sed "s/^/base /"
    KFB200_TQFK=1 python tools/ens_rate.py $B 16 | sed "s/^/tqfk2 /"
    KFB200_TQFK=1 KFB200_LIB=$PWD/_variants/tqfk4.so python tools/ens_rate.py $B 16 | sed "s/^/tqfk4 /"
  done
  python tools/single_rate.py --configs C1,C2 --iters 300 | sed "s/^/base /"
  KFB200_TQFK=1 python tools/single_rate.py --configs C1,C2 --iters 300 | sed "s/^/tqfk2 /"
done
