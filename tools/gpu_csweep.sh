#!/bin/bash
# cascade-sweep variants: launch times of the two sweep launches of a fused C4 step
for fit in 0 1; do
  CAMELOT_SWEEP_FIT=$fit timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sweep_kernel --csv python tools/pair_step.py 4 4 2>/dev/null | grep sweep_kernel | tail -4 | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ' | sed "s/^/fit=$fit: /"; echo
done
for fit in 0 1; do
  echo "fit=$fit $(CAMELOT_SWEEP_FIT=$fit timeout 120 python tools/trace_probe.py 4 4 2>&1 | grep kernel | tail -2 | awk '{print $2, $6}' | tr '\n' ' ')"
done
timeout 300 python -m pytest tests/test_sweep.py tests/test_plan_pair.py -q -x 2>&1 | tail -1
