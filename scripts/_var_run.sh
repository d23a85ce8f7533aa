# tuning helper: bench each variant library on (15,4) and (17,6)
for v in "$@"; do
  if [ "$v" != "main" ]; then export PMS_LIB_OVERRIDE=build/variants/$v/libpms_b200.so; else unset PMS_LIB_OVERRIDE; fi
  python bench.py --steps 50 --candidate-steps 0 --rmix-steps 0 --e2e-steps 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['search_kernel_ms'], d['parity_vs_golden'])"
  python scripts/large_l.py --configs 17,6 --oracle-range 1000 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$v 17,6', d['search_ms'], d['oracle_range_parity'])"
done
