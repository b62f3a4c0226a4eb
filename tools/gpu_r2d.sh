#!/bin/bash
# round-2 checkpoint: all GPU tests, bench N=1, launch list, --set full of the search launches and the flat sweep
mkdir -p gpurun_out/prof
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo bench1=$?
tail -3 gpurun_out/bench_n1.err; cut -c1-600 gpurun_out/bench_n1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-flat --no-hard --no-sa --no-comm --no-sim > gpurun_out/prof/launch_bench.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_level -s 2 -c 2 -o /tmp/search_full python tools/pair_step.py 4 2 > gpurun_out/prof/ncu_full.log 2>&1; echo ncu2=$?
ncu -i /tmp/search_full.ncu-rep --page raw --csv > gpurun_out/prof/search_raw.csv 2>&1
ncu -i /tmp/search_full.ncu-rep --page details --csv > gpurun_out/prof/search_details.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o /tmp/flat_full python tools/ncu_flat.py 4 2147483648 > gpurun_out/prof/ncu_flat.log 2>&1; echo ncu3=$?
ncu -i /tmp/flat_full.ncu-rep --page raw --csv > gpurun_out/prof/flat_raw.csv 2>&1
ncu -i /tmp/flat_full.ncu-rep --page details --csv > gpurun_out/prof/flat_details.csv 2>&1
ncu -i /tmp/flat_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof/flat_source.csv 2>&1
cp /tmp/flat_full.ncu-rep /tmp/search_full.ncu-rep gpurun_out/prof/ 2>/dev/null
ls -la gpurun_out/prof; du -sh gpurun_out
