#!/bin/bash
# Builds libbsg.so with extra nvcc defines into build/var/NAME/libbsg.so
# (development aid for same-session A/B: scripts/ab.py build/var/NAME/libbsg.so ...)
# usage: scripts/build_variant.sh NAME "-DKNOB=1 -DOTHER=2"
set -e
name=$1; shift
out=build/var/$name; mkdir -p $out
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 --expt-relaxed-constexpr -DBSG_DEV_KNOBS=1 $*"
S=${SRCDIR:-paper_1708_09495_b200/csrc}
objs=""
for f in api radix netsort pr mtgen staging msd; do
  $NV -c $S/$f.cu -o $out/$f.o & objs="$objs $out/$f.o"
done
$NV -x cu -c $S/host_util.cpp -o $out/host_util.o & objs="$objs $out/host_util.o"
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libbsg.so $objs -lpthread
echo built $out/libbsg.so
