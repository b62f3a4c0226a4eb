#!/bin/bash
# step-level changes: plan-pair + parity + certify + sweep tests, bench (short)
mkdir -p gpurun_out/prof
timeout 900 python -m pytest tests/test_plan_pair.py tests/test_gpu_parity.py tests/test_gpu_certify.py tests/test_sweep.py tests/test_comm.py -q -x > gpurun_out/pytest_step.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_step.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-sa --no-comm --no-sim > gpurun_out/bench_step.json 2> gpurun_out/bench_step.err; echo bench=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_step.json').read().strip().splitlines()[-1])
print('step', d['ms_per_step'], d['ms_per_step_median'], 'flat', d['flat_scan']['ms'], d['flat_scan']['roofline']['frac'], 'c4b', d['c4b']['ms_per_step_median'], 'b200', d['c4_b200']['ms_per_step_median'], 'wall', d['time_to_plan_wall_ms']['median'])"
timeout 120 python tools/trace_probe.py 4 2 > gpurun_out/trace_c4.txt 2>&1; tail -4 gpurun_out/trace_c4.txt | cut -c1-200
