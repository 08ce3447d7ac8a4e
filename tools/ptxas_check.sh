#!/bin/bash
# ptxas_check.sh [KERNEL_SUBSTR] [extra nvcc flags...]: registers/spills of fr_diffuse.cu kernels
# (object left at /tmp/fd.o for cuobjdump)
cd "$(dirname "$0")/../paper_1202_6158_b200/csrc"
k=${1:-k_sweep}; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v "$@" -c fr_diffuse.cu -o /tmp/fd.o 2>&1 \
  | grep -E "error|$k" -A2 | grep -E "error|Compiling|spill|Used"
