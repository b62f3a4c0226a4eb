#!/bin/bash
# compact depth-1 frontier: parity first, then A/B (alternating) of the C4 step
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do for c in 0 1; do
  echo "compact1=$c $(CAMELOT_COMPACT1=$c timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sa --no-comm --no-sim --no-flat --no-e2e --no-b200 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step', round(d['ms_per_step'],4), round(d['ms_per_step_median'],4), 'c4b', round(d['c4b']['ms_per_step_median'],4))")"
done; done
