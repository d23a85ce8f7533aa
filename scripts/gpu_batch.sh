#!/bin/bash
# End-of-phase GPU batch (round 2): tests (release + bounds/protocol-checked
# debug library), the default bench line, every config, randomised stress,
# the ncu launch list and one full capture.  Everything under gpurun_out/.
python -m pytest tests/ -q -m gpu > gpurun_out/r02_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02_gpu_tests.log
PMS_DEBUG_LIB=1 python -m pytest tests/ -q -m gpu > gpurun_out/r02_gpu_tests_debug.log 2>&1; echo "debug tests rc=$?" >> gpurun_out/r02_gpu_tests_debug.log
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?" >> gpurun_out/r02_bench.err
python bench.py --all-configs --reps 9 --out gpurun_out/r02_configs.json > gpurun_out/r02_configs.log 2>&1; echo "configs rc=$?" >> gpurun_out/r02_configs.log
python tests/tools/stress_parity.py --seconds 300 --seed 4 > gpurun_out/r02_stress.log 2>&1; echo "stress rc=$?" >> gpurun_out/r02_stress.log
CMD="python bench.py --steps 2 --warmup 3 --e2e-steps 1 --candidate-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/r02_launch_plain.json 2>/dev/null && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $CMD > gpurun_out/r02_launches_ncu.log 2>&1
./scripts/profile_slice.sh r02_slice > gpurun_out/r02_profile.log 2>&1
for f in r02_gpu_tests.log r02_gpu_tests_debug.log r02_configs.log r02_stress.log r02_profile.log; do tail -n 2 gpurun_out/$f; done
