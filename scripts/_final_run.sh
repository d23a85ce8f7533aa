set -x
python bench.py > gpurun_out/final_bench.json 2>gpurun_out/final_bench.err
bash scripts/profile.sh
python -m pytest tests -m gpu -q > gpurun_out/final_gpu_tests.log 2>&1
python bench.py --impl reference > gpurun_out/final_reference.json 2>gpurun_out/final_reference.err
python scripts/experiments.py --algo auto --out gpurun_out/final_experiments_auto > gpurun_out/final_experiments.log 2>&1
for c in 0 1 2 4; do python scripts/tune.py --cfg $c --reps 3 2>/dev/null | grep BEST; done > gpurun_out/final_configs.txt
