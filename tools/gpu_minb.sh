#!/bin/bash
# search kernel at 2 CTAs/SM (128 registers) vs the default (1 CTA/SM, 255 registers)
for v in default minb2s; do
  if [ $v = default ]; then unset CAMELOT_LIB; else export CAMELOT_LIB=$PWD/exp/$v/libcamelot.so; fi
  echo "$v $(timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sa --no-comm --no-sim --no-flat --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step', round(d['ms_per_step'],4), round(d['ms_per_step_median'],4), 'c4b', round(d['c4b']['ms_per_step_median'],4), 'b200', round(d['c4_b200']['ms_per_step_median'],4))")"
done
