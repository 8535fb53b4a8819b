#!/bin/bash
# Build libkfb200.so with extra -D flags into _variants/NAME.so (A/B measurements:
# run with KFB200_LIB=$PWD/_variants/NAME.so).  usage: tools/build_variant.sh NAME "-DFOO=1 ..."
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/_variants/$name
mkdir -p "$out"
cd "$root/paper_1712_05012_b200/csrc"
objs=""
for f in kf_api kf_kinematics kf_grid kf_nonbonded kf_solvation kf_torque kf_refgrid kf_peak kf_cluster; do
  if [ "$f" = kf_cluster ] || [ ! -f build/$f.o ]; then
    src=$f.cu
    [ "$f" = kf_cluster ] && [ -n "$CLSRC" ] && src=$CLSRC   # CLSRC: an alternative kf_cluster.cu (A/B)
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include -I. \
      --expt-relaxed-constexpr "$@" -c $src -o "$out/$f.o" &
    objs="$objs $out/$f.o"
  else
    objs="$objs build/$f.o"
  fi
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/_variants/$name.so" $objs -cudart static
echo "$root/_variants/$name.so"
