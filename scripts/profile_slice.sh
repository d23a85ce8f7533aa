#!/bin/bash
# GPU box: ncu --set full capture of the default search kernel at (15,4), after
# the identical plain command exited 0; writes gpurun_out/$1.ncu-rep and the
# JSON summary bench.py's issue roofline reads.   usage: profile_slice.sh NAME [bench args]
set -e
NAME=${1:-slice}; shift || true
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 1 --candidate-steps 0 --no-cpu-baseline $*"
$CMD > gpurun_out/${NAME}_plain.json 2>gpurun_out/${NAME}_plain.err
ncu --set full --clock-control none --import-source on -k regex:pms_search -s 3 -c 1 \
    -o gpurun_out/$NAME $CMD > gpurun_out/${NAME}_ncu.log 2>&1
SCANS=$(python -c "import json;print(json.load(open('gpurun_out/${NAME}_plain.json'))['block_scans_per_launch'])")
CFG=$(python -c "import json;c=json.load(open('gpurun_out/${NAME}_plain.json'))['config'];print(json.dumps({k:c[k] for k in ('n','t','l','d')}|{'block_digits':c['kernel']['block_digits'],'algo':c['algo']}))")
python scripts/ncu_summary.py json gpurun_out/$NAME.ncu-rep --scans $SCANS --out gpurun_out/${NAME}_ncu.json \
    --note "default search kernel, bench.py headline workload (3 warm-up steps, 4th launch captured)" \
    --config "$CFG" > /dev/null
echo profile-ok $SCANS
