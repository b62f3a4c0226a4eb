#!/bin/bash
# thread-per-parent threshold (x/16 of the resident warps): C4 / C4b / C4-b200 step times
for t in 32 16 8; do
  echo "tmode_min16=$t $(CAMELOT_TMODE_MIN16=$t timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sa --no-comm --no-sim --no-flat --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step', round(d['ms_per_step'],4), round(d['ms_per_step_median'],4), 'c4b', round(d['c4b']['ms_per_step_median'],4), 'b200', round(d['c4_b200']['ms_per_step_median'],4))")"
done
