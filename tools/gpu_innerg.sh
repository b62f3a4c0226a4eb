#!/bin/bash
# thread-per-parent mode for inner passes with more than 32 options (G lanes per parent): A/B
for g in 1 8; do
  echo "inner_gmax=$g $(CAMELOT_TMODE_INNER_G=$g timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sa --no-comm --no-sim --no-flat --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step', round(d['ms_per_step'],4), round(d['ms_per_step_median'],4), 'c4b', round(d['c4b']['ms_per_step_median'],4), 'b200', round(d['c4_b200']['ms_per_step_median'],4))")"
done
timeout 900 python -m pytest tests/test_gpu_certify.py tests/test_gpu_parity.py tests/test_plan_pair.py -q -x 2>&1 | tail -1
