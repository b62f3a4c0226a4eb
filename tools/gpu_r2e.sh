#!/bin/bash
# round-2 evidence v8: all GPU tests, bench N=1 and N=2 (two ranks share the device), launch
# list, --set full of both search launches and of the flat sweep (with source)
mkdir -p gpurun_out/prof
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench1=$?
python -c "
import json;d=json.loads(open('gpurun_out/bench_n1.json').read().strip().splitlines()[-1])
print('step', d['ms_per_step'], d['ms_per_step_median'], 'flat', d['flat_scan']['ms'], d['flat_scan']['roofline']['frac'], 'c4b', d['c4b']['ms_per_step_median'], 'e2e', d['e2e']['ms_per_step'], 'b200', d['c4_b200']['ms_per_step_median'])"
timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --no-sa --no-comm --no-sim --no-hard --no-b200 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo bench2=$?
cut -c1-300 gpurun_out/bench_n2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-flat --no-hard --no-sa --no-comm --no-sim > gpurun_out/prof/launch_bench.log 2>&1; echo ncu1=$?
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:search_level -s 2 -c 2 -o /tmp/search_full python tools/pair_step.py 4 2 > gpurun_out/prof/ncu_full.log 2>&1; echo ncu2=$?
ncu -i /tmp/search_full.ncu-rep --page raw --csv > gpurun_out/prof/search_raw.csv 2>&1
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o /tmp/flat_full python tools/ncu_flat.py 4 2147483648 > gpurun_out/prof/ncu_flat.log 2>&1; echo ncu3=$?
ncu -i /tmp/flat_full.ncu-rep --page raw --csv > gpurun_out/prof/flat_raw.csv 2>&1
ncu -i /tmp/flat_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof/flat_source.csv 2>&1
ncu -i /tmp/flat_full.ncu-rep --page details --csv > gpurun_out/prof/flat_details.csv 2>&1
cuobjdump -sass -fun '_ZN3cam12sweep_kernelILi8ELi5ELi0ELb0ELb0EEEvNS_7DevProbENS_9SweepArgsE' paper_2005_02088_b200/build/camelot_sweep.o | grep -E "UBLKCP|UTMALDG|SYNCS" | head -5 > gpurun_out/prof/sweep_tma_sass.txt
