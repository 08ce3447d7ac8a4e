#!/bin/bash
# build_so.sh NAME "-DFLAGS..." [SOURCE.cu] [GIT_REV]: links build_variants/NAME.so with SOURCE
# (default fr_diffuse.cu) compiled under extra flags, optionally from a git revision of that
# file (load it with FR_LIB_PATH=build_variants/NAME.so)
set -e
src=${3:-fr_diffuse.cu}
base=${src%.cu}
cd "$(dirname "$0")/../paper_1202_6158_b200/csrc"
make -s
mkdir -p ../../build_variants
if [ -n "$4" ]; then
  git show "$4:paper_1202_6158_b200/csrc/$src" > /tmp/${base}_$1.cu
  cp fr_common.cuh /tmp/
  nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 -I. -I../../include $2 -c /tmp/${base}_$1.cu -o /tmp/${base}_$1.o
else
  nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 $2 -c $src -o /tmp/${base}_$1.o
fi
objs=$(ls build/*.o | grep -v "/$base.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../build_variants/$1.so $objs /tmp/${base}_$1.o
