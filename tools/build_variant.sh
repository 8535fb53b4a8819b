#!/bin/bash
# Build libkfb200.so with extra -D flags into _variants/NAME.so (A/B measurements:
# run with KFB200_LIB=$PWD/_variants/NAME.so).
# usage: [SRCDIR=dir] [CLSRC=alt_kf_cluster.cu] [REBUILD="kf_xxx ..."] tools/build_variant.sh NAME -DFOO=1 ...
# kf_loop (the unity TU of kinematics, torque and cluster kernels) is always rebuilt.
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/_variants/$name
rm -rf "$out"; mkdir -p "$out/src"
src=${SRCDIR:-$root/paper_1712_05012_b200/csrc}
cp "$src"/*.cu "$src"/*.cuh "$out/src/"
[ -n "$CLSRC" ] && cp "$CLSRC" "$out/src/kf_cluster.cu"
cd "$out/src"
objs=""
for f in kf_api kf_loop kf_grid kf_nonbonded kf_solvation kf_refgrid kf_peak; do
  if [ "$f" = kf_loop ] || [[ " $REBUILD " == *" $f "* ]] || [ ! -f "$root/paper_1712_05012_b200/csrc/build/$f.o" ]; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I"$root/include" -I. \
      --expt-relaxed-constexpr "$@" -c $f.cu -o "$out/$f.o" &
    objs="$objs $out/$f.o"
  else
    objs="$objs $root/paper_1712_05012_b200/csrc/build/$f.o"
  fi
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$root/_variants/$name.so" $objs -cudart static
echo "$root/_variants/$name.so"
