#!/bin/bash
# shared-policy kernel variant (one instantiation for both policies) vs default: cold probe, bench legs, parity
for v in default shared; do
  if [ $v = shared ]; then export CAMELOT_LIB=$PWD/exp/shared/libcamelot.so; else unset CAMELOT_LIB; fi
  echo "== $v"
  timeout 300 python tools/cold_probe.py 2>&1 | tail -4
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sa --no-comm --no-sim --no-flat --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step', round(d['ms_per_step'],4), round(d['ms_per_step_median'],4), 'c4b', round(d['c4b']['ms_per_step_median'],4), 'b200', round(d['c4_b200']['ms_per_step_median'],4))"
done
CAMELOT_LIB=$PWD/exp/shared/libcamelot.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_certify.py tests/test_plan_pair.py tests/test_comm.py -q -x 2>&1 | tail -1
