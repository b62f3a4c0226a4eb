#!/bin/bash
# frontier clamp: C4 / C4b / C4-b200 step times (bench legs) at 2^20, 2^21, 2^22 nodes
for fm in 1048576 2097152 4194304; do
  echo "fmax=$fm $(CAMELOT_FRONTIER_MAX=$fm timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sa --no-comm --no-sim --no-flat --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step', round(d['ms_per_step'],4), round(d['ms_per_step_median'],4), 'c4b', round(d['c4b']['ms_per_step_median'],4), 'b200', round(d['c4_b200']['ms_per_step_median'],4))")"
done
