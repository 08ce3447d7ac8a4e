#!/bin/bash
# parameter sweep of the fused kernel's scheduling knobs (tools/, not part of the product)
for cfg in "64 8" "32 8" "128 8" "64 4" "64 16" "16 8"; do
  set -- $cfg
  r=$(FR_SEGS=$1 FR_CHUNK=$2 timeout 300 python tools/prof_solver.py 2>&1 | grep "kernel ms" | sed 's/launches.*//')
  echo "segs=$1 chunk=$2 $r"
done
