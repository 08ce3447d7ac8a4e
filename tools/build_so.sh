#!/bin/bash
# build_so.sh NAME "-DFLAGS...": links build_variants/NAME.so with fr_diffuse.cu compiled
# under extra flags (load it with FR_LIB_PATH=build_variants/NAME.so)
set -e
cd "$(dirname "$0")/../paper_1202_6158_b200/csrc"
make -s
mkdir -p ../../build_variants
nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 $2 -c fr_diffuse.cu -o /tmp/fr_diffuse_$1.o
objs=$(ls build/*.o | grep -v fr_diffuse.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../build_variants/$1.so $objs /tmp/fr_diffuse_$1.o
