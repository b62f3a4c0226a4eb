#!/bin/bash
# round-2 check: sanitizer + certify tests, the new bench at N=1 and N=2 (gloo, one device), phase trace
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_sanitizer.py tests/test_gpu_certify.py -q > gpurun_out/pytest_r2a.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_r2a.log
timeout 900 python bench.py --steps 10 --warmup 5 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo bench=$?
timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --no-sa --no-comm --no-sim > gpurun_out/bench_r2a_n2.json 2> gpurun_out/bench_r2a_n2.err; echo bench2=$?
tail -3 gpurun_out/bench_r2a_n2.err
timeout 300 python tools/trace_probe.py 4 2 > gpurun_out/trace_c4.txt 2>&1; echo trace=$?
timeout 300 python tools/trace_probe.py 7 2 > gpurun_out/trace_c4b.txt 2>&1; echo trace=$?
