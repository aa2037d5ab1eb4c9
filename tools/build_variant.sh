#!/bin/bash
# Build an experimental libtcb200 variant with extra nvcc defines (A/B measurements):
#   bash tools/build_variant.sh tools/sp_NAME.so "-DFLAG=VALUE ..."
# then run with TCB200_LIB=tools/sp_NAME.so.
set -e
cd "$(dirname "$0")/.."
OUT=$1; shift
D=$(mktemp -d)
F="-O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-fopenmp,-O3"
for s in paper_2510_12011_b200/csrc/*.cu paper_2510_12011_b200/csrc/*.cpp; do
  nvcc $F $@ -c $s -o $D/$(basename $s).o &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a $D/*.o -o $OUT -lgomp
rm -rf $D
