#!/bin/bash
# ab_libs.sh V1 V2 ...: time full config-5 solves (tools/path_ab.py, owned path, bench schedule)
# with each library variant build_variants/V.so (built by tools/build_variant.sh)
for v in "$@"; do
  FR_LIB_PATH=build_variants/$v.so timeout 600 python tools/path_ab.py --reps ${REPS:-5} owned 2>&1 | sed "s/^/$v /" | tail -1
done
