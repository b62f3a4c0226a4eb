#!/bin/bash
# sweep change: all GPU tests, bench N=1, ncu --set full of the flat sweep
mkdir -p gpurun_out/prof
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench1=$?
tail -2 gpurun_out/bench_n1.err; python -c "
import json;d=json.loads(open('gpurun_out/bench_n1.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['flat_scan']['ms'], d['flat_scan']['roofline']['frac'], d['c4b']['ms_per_step_median'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o /tmp/flat_full python tools/ncu_flat.py 4 2147483648 > gpurun_out/prof/ncu_flat.log 2>&1; echo ncu3=$?
ncu -i /tmp/flat_full.ncu-rep --page raw --csv > gpurun_out/prof/flat_raw.csv 2>&1
ncu -i /tmp/flat_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof/flat_source.csv 2>&1
