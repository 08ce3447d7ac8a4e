#!/bin/bash
# Build a variant of libfluidrank_b200.so with extra -D flags into tools/variants/<name>.so
# usage: tools/build_variant.sh <name> "-DFR_SW_UNROLL=8 -DFR_SW_NT=128"
set -e
name=$1; defs=$2
root=$(cd "$(dirname "$0")/.." && pwd)
src=$root/paper_1202_6158_b200/csrc
out=$root/tools/variants; mkdir -p $out
tmp=$(mktemp -d)
for f in fr_capi fr_scan fr_gen fr_csr fr_util fr_diffuse fr_spmv fr_ppr; do
  nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-O3 $defs -c $src/$f.cu -o $tmp/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/$name.so $tmp/*.o
rm -rf $tmp
echo built $out/$name.so
