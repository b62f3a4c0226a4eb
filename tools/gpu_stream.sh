#!/bin/bash
# streaming phase: C4 phase trace (both modes), then the pruned-search parity tests
mkdir -p gpurun_out
timeout 120 python tools/trace_probe.py 4 2 > gpurun_out/trace_stream.txt 2>&1; echo trace=$?
tail -12 gpurun_out/trace_stream.txt | cut -c1-250
CAMELOT_STREAM=0 timeout 120 python tools/trace_probe.py 4 2 > gpurun_out/trace_sync.txt 2>&1; echo trace0=$?
grep "kernel" gpurun_out/trace_sync.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_certify.py tests/test_plan_pair.py -q -x > gpurun_out/pytest_stream.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_stream.log
