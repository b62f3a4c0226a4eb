#!/bin/bash
# round-2 evidence of the current build (one GPU): smoke, all GPU tests, the bench at
# N=1 (all legs) and N=2 (two ranks on one device), ncu launch list of bench steps,
# --set full of both search launches and of the flat sweep (with source), phase traces
# and the time-to-plan of every config
mkdir -p gpurun_out/final
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/final/gpu.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/final/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench_n1.json 2> gpurun_out/final/bench_n1.err; echo bench1=$?
timeout 600 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-sa --no-comm --no-sim > gpurun_out/final/bench_n2.json 2> gpurun_out/final/bench_n2.err; echo bench2=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-flat --no-hard --no-sa --no-comm --no-sim > /dev/null 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_level -s 2 -c 2 -o /tmp/search_full python tools/pair_step.py 4 2 > gpurun_out/final/ncu_search.log 2>&1; echo ncu2=$?
ncu -i /tmp/search_full.ncu-rep --page raw --csv > gpurun_out/final/search_raw.csv 2>&1
ncu -i /tmp/search_full.ncu-rep --page details --csv > gpurun_out/final/search_details.csv 2>&1
ncu -i /tmp/search_full.ncu-rep --page source --csv --print-source cuda,sass > /tmp/search_source.csv 2>&1
python tools/ncu_lines.py /tmp/search_source.csv 40 > gpurun_out/final/search_lines.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o /tmp/flat_full python tools/ncu_flat.py 4 2147483648 > gpurun_out/final/ncu_flat.log 2>&1; echo ncu3=$?
ncu -i /tmp/flat_full.ncu-rep --page raw --csv > gpurun_out/final/flat_raw.csv 2>&1
ncu -i /tmp/flat_full.ncu-rep --page details --csv > gpurun_out/final/flat_details.csv 2>&1
ncu -i /tmp/flat_full.ncu-rep --page source --csv --print-source cuda,sass > /tmp/flat_source.csv 2>&1
python tools/ncu_lines.py /tmp/flat_source.csv 40 > gpurun_out/final/flat_lines.txt 2>&1
timeout 300 python tools/trace_probe.py 4 2 > gpurun_out/final/trace_c4.txt 2>&1
timeout 300 python tools/trace_probe.py 7 2 > gpurun_out/final/trace_c4b.txt 2>&1
timeout 600 python tools/configs_probe.py > gpurun_out/final/configs.txt 2>&1; echo configs=$?
ls -la gpurun_out/final
