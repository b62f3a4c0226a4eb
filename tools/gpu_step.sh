#!/bin/bash
# step-level changes: plan-pair + parity tests, bench (short), ncu source of the cascade sweep
mkdir -p gpurun_out/prof
timeout 900 python -m pytest tests/test_plan_pair.py tests/test_gpu_parity.py tests/test_gpu_certify.py tests/test_sweep.py -q -x > gpurun_out/pytest_step.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_step.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sa --no-comm --no-sim > gpurun_out/bench_step.json 2> gpurun_out/bench_step.err; echo bench=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_step.json').read().strip().splitlines()[-1])
print('step', d['ms_per_step'], d['ms_per_step_median'], 'flat', d['flat_scan']['ms'], d['flat_scan']['roofline']['frac'], 'c4b', d['c4b']['ms_per_step_median'], 'wall', d['time_to_plan_wall_ms'])"



