#!/bin/bash
# ppr_variants.sh "NAME:-DFLAGS" ...: fr_ppr.cu rebuilt with extra flags, timed by tools/ppr_prof.py
objs=$(ls paper_1202_6158_b200/csrc/build/*.o | grep -v fr_ppr.o)
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC $flags \
    -c paper_1202_6158_b200/csrc/fr_ppr.cu -o /tmp/ppr_$name.o &&
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o /tmp/ppr_$name.so $objs /tmp/ppr_$name.o &&
  FR_LIB_PATH=/tmp/ppr_$name.so python tools/ppr_prof.py $PPR_ARGS 2>&1 | grep "^n=" | sed "s/^/$name /"
done
