#!/bin/bash
# Build a variant library with extra nvcc defines and run the sweep on it.
#   scripts/variant.sh "-DFOO=1" "configs" "variants"
DEFS="$1"; CONFIGS=${2:-3,4}; VARS=${3:-algo=0}
OUT=/tmp/var_$$.so
for f in pms pms64 pms_slice pms_slice_ht pms_roof; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC $DEFS -I include \
       -I paper_1403_1313_b200/csrc -c paper_1403_1313_b200/csrc/$f.cu -o /tmp/v_$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared /tmp/v_pms.o /tmp/v_pms64.o /tmp/v_pms_slice.o /tmp/v_pms_slice_ht.o /tmp/v_pms_roof.o -o $OUT
echo "variant [$DEFS]"
PMS_LIB_OVERRIDE=$OUT python scripts/sweep.py --configs $CONFIGS --reps 8 --variants "$VARS" 2>&1 | tail -6
