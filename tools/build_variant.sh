#!/bin/bash
# Build an A/B variant of libsketch_b200.so with one source recompiled under
# extra defines: tools/build_variant.sh <name> <source.cu> -DMACRO=value ...
# -> tools/libsketch_<name>.so (select it with SKT_LIB_PATH=...).
set -e
name=$1; src=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
csrc=$root/paper_1207_6365_b200/csrc
obj=$root/build/csrc
make -C "$csrc" -s >/dev/null
mkdir -p "$root/build/variant_$name"
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
     -I"$root/include" --expt-relaxed-constexpr "$@" -c "$csrc/$src" -o "$root/build/variant_$name/${src%.cu}.o"
objs=""
for o in "$obj"/*.o; do
  b=$(basename "$o")
  if [ "$b" = "${src%.cu}.o" ]; then objs="$objs $root/build/variant_$name/$b"; else objs="$objs $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$root/tools/libsketch_$name.so" $objs
echo "$root/tools/libsketch_$name.so"
