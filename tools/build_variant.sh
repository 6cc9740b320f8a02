#!/bin/bash
# Build libmehdg_b200.<name>.so with extra nvcc flags on one source file:
#   tools/build_variant.sh <name> <source.cu> <flags...>
# (load it with MEHDG_LIB_VARIANT=<name>)
set -e
name=$1; src=$2; shift 2
cd "$(dirname "$0")/.."
python -m paper_2302_10917_b200._build > /dev/null
objs=$(ls build/obj/*.o | grep -v "/$(basename $src).o")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O3 \
  -I include --expt-relaxed-constexpr "$@" -c paper_2302_10917_b200/csrc/$src -o build/variant_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2302_10917_b200/libmehdg_b200.$name.so \
  $objs build/variant_$name.o -ldl -lpthread
echo paper_2302_10917_b200/libmehdg_b200.$name.so
