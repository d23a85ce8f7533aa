#!/bin/bash
# Build a committed revision's library as build/variants/base (A/B baseline):
#   scripts/mkbase.sh [REV]   (default HEAD)
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/base && mkdir -p /tmp/base
git -C "$ROOT" archive "$REV" paper_1403_1313_b200 include | tar -x -C /tmp/base
cd /tmp/base
for f in pms pms64 pms_slice pms_slice_ht pms_slice_wide pms_roof; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -O3 \
       -I include -I paper_1403_1313_b200/csrc -c paper_1403_1313_b200/csrc/$f.cu -o /tmp/base/$f.o &
done
wait
mkdir -p "$ROOT/build/variants/base"
nvcc -gencode arch=compute_100a,code=sm_100a -shared /tmp/base/*.o -o "$ROOT/build/variants/base/libpms_b200.so"
echo "$ROOT/build/variants/base/libpms_b200.so"
