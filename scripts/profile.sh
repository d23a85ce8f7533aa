#!/bin/bash
# Run on the GPU box (gpurun) from the repo root.  Produces, under gpurun_out/:
#   launches.csv  -- every kernel launch of the bench command with its device time
#   search.ncu-rep -- one `ncu --set full` capture of the search kernel
# Each ncu command runs only after the identical plain command exited 0.
set -e
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --candidate-steps 0 --rmix-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/plain_launches.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
CMD2="python bench.py --steps 1 --warmup 3 --e2e-steps 1 --candidate-steps 0 --rmix-steps 0 --no-cpu-baseline"
$CMD2 > gpurun_out/plain_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pms_search -s 3 -c 1 \
    -o gpurun_out/search $CMD2 > gpurun_out/ncu_full.log 2>&1
echo profile-ok
