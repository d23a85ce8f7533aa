#!/bin/bash
# A/B of variant libraries (build/variants/NAME) on BASELINE configs, twice
# each, interleaved: scripts/ab.sh "main pin pred" [configs] [extra sweep variants]
VARS=${1:-main}; CFGS=${2:-2,3,4}; SV=${3:-algo=0}
for rep in 1 2; do
  for v in $VARS; do
    if [ "$v" = main ]; then unset PMS_LIB_OVERRIDE; else export PMS_LIB_OVERRIDE=build/variants/$v/libpms_b200.so; fi
    python scripts/sweep.py --configs $CFGS --reps 9 --variants "$SV" 2>&1 | sed "s/^/$v /" | cut -c1-170
  done
done
