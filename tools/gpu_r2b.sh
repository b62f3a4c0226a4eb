#!/bin/bash
# round-2 baseline check on one B200: smoke, all GPU tests, bench at N=1 and N=2 (two ranks on cuda:0), phase traces
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cut -c1-3000 gpurun_out/bench.json
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --no-sa --no-comm --no-sim > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo bench2=$?
tail -3 gpurun_out/bench_n2.err
timeout 300 python tools/trace_probe.py 4 2 > gpurun_out/trace_c4.txt 2>&1; echo trace=$?
timeout 300 python tools/trace_probe.py 7 2 > gpurun_out/trace_c4b.txt 2>&1; echo trace=$?
