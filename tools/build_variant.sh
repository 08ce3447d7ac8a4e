#!/bin/bash
# build_variant.sh NAME "-DFLAGS..." [GIT_REV]: links libfluidrank_b200.so with fr_diffuse.cu
# compiled under extra flags into build_variants/NAME.so (for A/B timing via FR_LIB_PATH)
set -e
cd "$(dirname "$0")/../paper_1202_6158_b200/csrc"
make -s
mkdir -p ../../build_variants
src=fr_diffuse.cu
if [ -n "$3" ]; then src=fr_diffuse_v_$1.cu; git show "$3":paper_1202_6158_b200/csrc/fr_diffuse.cu > $src; fi
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 $2 -c $src -o /tmp/fr_diffuse_$1.o
if [ -n "$3" ]; then rm -f $src; fi
objs=$(ls build/*.o | grep -v fr_diffuse.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../build_variants/$1.so $objs /tmp/fr_diffuse_$1.o
