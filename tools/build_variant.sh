#!/bin/bash
# A/B builds of libpetals_b200.so with extra nvcc defines (experiments):
#   tools/build_variant.sh NAME -DFOO=1 ...   ->  paper_2209_01188_b200/build/NAME/libpetals_b200.so
# load one with PB_LIB=<path> (paper_2209_01188_b200/_lib.py).
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2209_01188_b200"
out=build/$name; mkdir -p $out
objs=""
for f in csrc/*.cu; do
  b=$(basename $f .cu); objs="$objs $out/$b.o"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" -c $f -o $out/$b.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libpetals_b200.so $objs -lcudart
echo $out/libpetals_b200.so
