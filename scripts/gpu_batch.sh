#!/bin/bash
# End-of-phase GPU batch (round 2): the ncu capture first (the bench line's
# issue roofline reads its summary), then the default bench line, every
# config, tests (release + bounds/protocol-checked debug library), randomised
# stress (default hand-off choice, and the sparse mode forced everywhere), the
# ncu launch list.  Everything under gpurun_out/.
./scripts/profile_slice.sh r02_slice > gpurun_out/r02_profile.log 2>&1 && \
  cp gpurun_out/r02_slice_ncu.json profiles/slice_kernel_ncu.json && \
  ncu -i gpurun_out/r02_slice.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_slice_source.csv 2>/dev/null
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?" >> gpurun_out/r02_bench.err
python bench.py --all-configs --reps 9 --out gpurun_out/r02_configs.json > gpurun_out/r02_configs.log 2>&1; echo "configs rc=$?" >> gpurun_out/r02_configs.log
python -m pytest tests/ -q -m gpu > gpurun_out/r02_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02_gpu_tests.log
PMS_DEBUG_LIB=1 python -m pytest tests/ -q -m gpu > gpurun_out/r02_gpu_tests_debug.log 2>&1; echo "debug tests rc=$?" >> gpurun_out/r02_gpu_tests_debug.log
python tests/tools/stress_parity.py --seconds 150 --seed 4 > gpurun_out/r02_stress.log 2>&1; echo "stress rc=$?" >> gpurun_out/r02_stress.log
PMS_HANDOFF_TABLES=0 python tests/tools/stress_parity.py --seconds 150 --seed 5 > gpurun_out/r02_stress_sparse.log 2>&1; echo "stress (sparse mode forced) rc=$?" >> gpurun_out/r02_stress_sparse.log
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --candidate-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/r02_launch_plain.json 2>/dev/null && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/r02_launches_ncu.log 2>&1
for f in r02_profile.log r02_gpu_tests.log r02_gpu_tests_debug.log r02_configs.log r02_stress.log r02_stress_sparse.log; do tail -n 2 gpurun_out/$f; done
