#!/bin/bash
# Build an A/B variant of the library: one source recompiled with extra -D
# flags, linked with the in-tree objects of the others, into ab/lib_<name>.so.
#   tools/dbg/build_variant.sh <name> <source stem> [-DFOO=1 ...]
set -e
cd "$(dirname "$0")/../.."
name=$1; stem=$2; shift 2
mkdir -p ab/obj_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -fmad=false -Xcompiler -fPIC \
  -Xptxas -v -I include "$@" -c -o ab/obj_$name/$stem.o paper_1803_00737_b200/csrc/$stem.cu \
  2> ab/obj_$name/build.log
objs=$(ls paper_1803_00737_b200/build/*.o | grep -v "/$stem.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/lib_$name.so $objs ab/obj_$name/$stem.o -ldl
echo ab/lib_$name.so
