#!/bin/bash
# host/device timing of the API calls, FTRACE phase trace, full bench, all GPU tests
mkdir -p gpurun_out
timeout 120 python tools/host_probe.py 4 6 > gpurun_out/host_probe.txt 2>&1; echo probe=$?
cat gpurun_out/host_probe.txt | tail -4
CAMELOT_LIB=$PWD/exp/libcamelot_ft.so timeout 200 python tools/trace_probe.py 4 2 > gpurun_out/ftrace_c4.txt 2>&1; echo ftrace=$?
timeout 600 python bench.py --steps 10 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
tail -4 gpurun_out/bench.err
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
