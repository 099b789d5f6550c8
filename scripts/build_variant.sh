#!/bin/bash
# Build an A/B variant library build/<name>/libhetsched_sm100a.so: the
# default objects, with <file.cu> recompiled from <src> (default: the
# working-tree file) under extra nvcc flags.
#   scripts/build_variant.sh NAME FILE.cu [SRC] [-- NVCC_FLAGS...]
set -e
cd "$(dirname "$0")/.."
name=$1; file=$2; shift 2
src=paper_2206_01288_b200/csrc/$file
if [ $# -gt 0 ] && [ "$1" != "--" ]; then src=$1; shift; fi
[ "${1:-}" = "--" ] && shift
out=build/$name
mkdir -p $out/obj
cp paper_2206_01288_b200/lib/obj/*.o $out/obj/
tmp=paper_2206_01288_b200/csrc/.variant_$name.cu
cp "$src" "$tmp"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false -std=c++17 -Xcompiler -fPIC "$@" \
  -c -o $out/obj/${file%.cu}.o "$tmp"
rm -f "$tmp"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libhetsched_sm100a.so $out/obj/*.o
echo "built $out"
