#!/bin/bash
# leaf passes in the thread-per-parent mode up to 128 (G 4) or 256 (G 8) options per parent
for g in 4 8; do
  echo "leaf_gmax=$g $(CAMELOT_TMODE_LEAF_G=$g timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sa --no-comm --no-sim --no-flat --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step', round(d['ms_per_step'],4), round(d['ms_per_step_median'],4), 'c4b', round(d['c4b']['ms_per_step_median'],4), 'b200', round(d['c4_b200']['ms_per_step_median'],4))")"
  CAMELOT_TMODE_LEAF_G=$g timeout 900 python tools/cascade_probe3.py "50,11,4|50,20,7" 2>&1 | tail -1
done
timeout 900 python -m pytest tests/test_gpu_certify.py tests/test_gpu_parity.py tests/test_plan_pair.py tests/test_sweep.py tests/test_comm.py -q -x 2>&1 | tail -1
