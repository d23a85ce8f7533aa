python bench.py --impl reference > gpurun_out/final_reference.json 2>gpurun_out/final_reference.err
for c in 0 1 2 4; do timeout 240 python scripts/tune.py --cfg $c --reps 3 2>/dev/null | grep BEST; done > gpurun_out/final_configs.txt
timeout 900 python scripts/experiments.py --algo auto --out gpurun_out/final_experiments_auto > gpurun_out/final_experiments.log 2>&1
