#!/bin/bash
# Round-2 GPU batch: tests (release + bounds/protocol-checked debug library),
# per-config measurements, randomised stress.  Logs under gpurun_out/.
python -m pytest tests/ -q -m gpu > gpurun_out/r02_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02_gpu_tests.log
PMS_DEBUG_LIB=1 python -m pytest tests/ -q -m gpu > gpurun_out/r02_gpu_tests_debug.log 2>&1; echo "debug tests rc=$?" >> gpurun_out/r02_gpu_tests_debug.log
python bench.py --all-configs --reps 9 --out gpurun_out/r02_configs.json > gpurun_out/r02_configs.log 2>&1; echo "configs rc=$?" >> gpurun_out/r02_configs.log
python tests/tools/stress_parity.py --seconds 300 --seed 2 > gpurun_out/r02_stress.log 2>&1; echo "stress rc=$?" >> gpurun_out/r02_stress.log
tail -3 gpurun_out/r02_gpu_tests.log gpurun_out/r02_gpu_tests_debug.log gpurun_out/r02_configs.log gpurun_out/r02_stress.log
