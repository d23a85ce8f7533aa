#!/bin/bash
# GPU box: ncu --set full capture of the default search kernel at (15,4) (after a plain run).
set -e
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 1 --candidate-steps 0 --rmix-steps 0 --no-cpu-baseline $2"
$CMD > gpurun_out/plain_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pms_search -s 3 -c 1 \
    -o gpurun_out/${1:-slice} $CMD > gpurun_out/ncu_full.log 2>&1
echo profile-ok
