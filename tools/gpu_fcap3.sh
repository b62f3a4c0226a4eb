#!/bin/bash
# frontier clamp 2^21 vs 2^23 nodes: bench legs and the heavy C4-shaped instances
for fm in 2097152 8388608; do
  echo "fmax=$fm $(CAMELOT_FRONTIER_MAX=$fm timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sa --no-comm --no-sim --no-flat --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step', round(d['ms_per_step'],4), round(d['ms_per_step_median'],4), 'c4b', round(d['c4b']['ms_per_step_median'],4), 'b200', round(d['c4_b200']['ms_per_step_median'],4))")"
  CAMELOT_FRONTIER_MAX=$fm timeout 900 python tools/cascade_probe3.py "50,11,4|50,20,7" 2>&1 | tail -1
done
