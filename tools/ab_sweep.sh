#!/usr/bin/env bash
# A/B timing of alternate builds of librs_b200.so (RS_B200_LIB) on one
# 1,184-scenario sweep batch: bash tools/ab_sweep.sh build/ab/*.so
for lib in "$@"; do
  for i in 1 2; do
    RS_B200_LIB=$lib python tools/prof_sweep.py 1184 3 | grep "rep 2" | grep -E "group_eval|fast_build" | sed "s|^|$(basename $lib) |"
  done
done
