#!/bin/bash
# Build a variant of libbsparse.so with one source recompiled under extra
# flags:  tools/variant.sh <name> <source.cu> <nvcc flags...>
# -> paper_1805_03380_b200/build/variants/<name>.so (load it with AS_LIB_PATH)
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
B=paper_1805_03380_b200/build
mkdir -p $B/variants/$name
base=$(basename $src .cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr "$@" \
  -c paper_1805_03380_b200/csrc/$base.cu -o $B/variants/$name/$base.o
objs=""
for o in $B/*.o; do
  if [ "$(basename $o)" = "$base.o" ]; then objs="$objs $B/variants/$name/$base.o"; else objs="$objs $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $B/variants/$name.so $objs
echo $B/variants/$name.so
