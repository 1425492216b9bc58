#!/bin/bash
# A/B baseline: build libpetals_b200.so from a git revision (default HEAD) into
# paper_2209_01188_b200/build/NAME (load with PB_LIB=...).
#   tools/build_head_variant.sh base [REV]
set -e
name=$1; rev=${2:-HEAD}
root="$(cd "$(dirname "$0")/.." && pwd)"
wt=$(mktemp -d)/wt
git -C "$root" worktree add -f "$wt" "$rev" -q
out=$root/paper_2209_01188_b200/build/$name; mkdir -p $out
objs=""
for f in "$wt"/paper_2209_01188_b200/csrc/*.cu; do
  b=$(basename $f .cu); objs="$objs $out/$b.o"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -c $f -o $out/$b.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libpetals_b200.so $objs -lcudart
git -C "$root" worktree remove --force "$wt"
echo $out/libpetals_b200.so
