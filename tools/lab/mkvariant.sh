#!/bin/bash
# usage: tools/lab/mkvariant.sh NAME FILE.cu [extra nvcc flags]: relink the library with FILE.cu
# (a variant of one csrc/ source) in place of its namesake, into tools/lab/sweep/NAME.so
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
name=$1; src=$2; shift 2
base=$(basename "$src" .cu); base=${base#_v_}
B=$ROOT/paper_2210_05105_b200/build
tmp=$ROOT/paper_2210_05105_b200/csrc/_v_$base.cu
[ "$src" != "$tmp" ] && cp "$src" "$tmp"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 \
  --expt-relaxed-constexpr -cudart static -Xptxas -v "$@" -c "$tmp" -o /tmp/_v.o 2>&1 | grep -E "spill|Used" | tail -4 || true
rm -f "$tmp"
objs=$(ls $B/*.cu.o | grep -v "/$base.cu.o")
mkdir -p $ROOT/tools/lab/sweep
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $ROOT/tools/lab/sweep/$name.so $objs /tmp/_v.o
echo built tools/lab/sweep/$name.so
