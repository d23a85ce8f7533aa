# tuning helper: bench each variant library on (15,4), (16,5) and (17,6), (19,7)
for v in "$@"; do
  if [ "$v" != "main" ]; then export PMS_LIB_OVERRIDE=build/variants/$v/libpms_b200.so; else unset PMS_LIB_OVERRIDE; fi
  python bench.py --steps 50 --candidate-steps 0 --rmix-steps 0 --e2e-steps 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['search_kernel_ms'], d['parity_vs_golden'])"
  python scripts/tune.py --cfg 4 --reps 3 2>/dev/null | grep BEST | python -c "import json,sys; d=json.loads(sys.stdin.read().split(' ',1)[1]); print('$v 16,5', d['search_ms'])"
  python tests/tools/large_l.py --configs 17,6 19,7 --oracle-range 1000 2>/dev/null | python -c "
import json,sys
for l in sys.stdin.read().splitlines(): d=json.loads(l); print('$v', d['l'], d['d'], d['search_ms'], d['oracle_range_parity'], d['consensus_found'])"
done
