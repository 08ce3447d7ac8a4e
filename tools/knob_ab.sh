#!/bin/bash
# knob_ab.sh "ARGS" ...: tools/path_ab.py (owned path, bench schedule) once per argument set
for v in "$@"; do
  timeout 600 python tools/path_ab.py --reps ${REPS:-4} $v owned 2>&1 | tail -1 | sed "s/^/[$v] /"
done
