#!/bin/bash
# Here (after gpurun brought gpurun_out/ back from scripts/gpu_batch.sh): turn
# the batch's raw output into the tracked files under profiles/ and re-render
# the BASELINE.md table.   usage: scripts/collect_profiles.sh [r02]
set -e
R=${1:-r02}
G=gpurun_out
SCANS=$(python -c "import json;print(json.load(open('$G/${R}_slice_plain.json'))['block_scans_per_launch'])")
cp $G/${R}_bench.json profiles/${R}_bench.json
cp $G/${R}_configs.json profiles/${R}_configs.json
cp $G/${R}_gpu_tests.log profiles/${R}_gpu_tests.log
cp $G/${R}_gpu_tests_debug.log profiles/${R}_gpu_tests_debug.log
cat $G/${R}_stress.log $G/${R}_stress_sparse.log > profiles/${R}_stress_parity.log
cp $G/${R}_launches.csv profiles/${R}_launches.csv
python scripts/ncu_summary.py launches profiles/${R}_launches.csv > profiles/${R}_launches_summary.txt
python scripts/ncu_summary.py full $G/${R}_slice.ncu-rep --title "slice kernel (15,4) S=7, round 2 final" \
    > profiles/${R}_slice_ncu_summary.txt
python scripts/ncu_summary.py json $G/${R}_slice.ncu-rep --scans $SCANS --out profiles/slice_kernel_ncu.json \
    --note "default search kernel, bench.py headline workload (3 warm-up steps, 4th launch captured)" \
    --config "$(python -c "import json;print(json.dumps(json.load(open('$G/${R}_slice_ncu.json'))['config']))")" > /dev/null
python scripts/ncu_source.py $G/${R}_slice_source.csv --units $SCANS --top 25 > profiles/${R}_slice_source_summary.txt
python scripts/ncu_source.py $G/${R}_slice_source.csv --units $SCANS --top 30 --wavefronts \
    > profiles/${R}_slice_shared_wavefronts.txt
python scripts/baseline_table.py profiles/${R}_configs.json > /tmp/${R}_table.md
echo "table in /tmp/${R}_table.md ($(wc -l < /tmp/${R}_table.md) lines); SCANS=$SCANS"
