#!/bin/bash
# spmv_variants.sh "NAME:-DFLAGS" ...: fr_spmv.cu rebuilt with extra flags, timed by tools/spmv_prof.py
objs=$(ls paper_1202_6158_b200/csrc/build/*.o | grep -v fr_spmv.o)
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC $flags \
    -c paper_1202_6158_b200/csrc/fr_spmv.cu -o /tmp/spmv_$name.o &&
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o /tmp/spmv_$name.so $objs /tmp/spmv_$name.o &&
  FR_LIB_PATH=/tmp/spmv_$name.so python tools/spmv_prof.py 2>&1 | tail -1 | sed "s/^/$name /"
done
