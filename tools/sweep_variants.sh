#!/bin/bash
# time one config-5 solve with each variant build in tools/variants (tools/, not the product)
r=$(timeout 300 python tools/prof_solver.py 2>&1 | grep "kernel ms" | sed 's/launches.*//'); echo "default $r"
for so in tools/variants/*.so; do
  r=$(FR_LIB_PATH=$PWD/$so timeout 300 python tools/prof_solver.py 2>&1 | grep "kernel ms" | sed 's/launches.*//')
  echo "$(basename $so) $r"
done
