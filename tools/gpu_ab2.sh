#!/bin/bash
# A/B of two library builds on one box (alternating): C4 bench step
for r in 1 2; do for v in current noinl; do
  if [ $v = current ]; then unset CAMELOT_LIB; else export CAMELOT_LIB=$PWD/exp/$v/libcamelot.so; fi
  echo "$v $(timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-sa --no-comm --no-sim --no-flat --no-e2e --no-hard --no-b200 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('step', round(d['ms_per_step'],4), round(d['ms_per_step_median'],4))")"
done; done
