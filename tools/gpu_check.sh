#!/bin/bash
# one GPU round trip: build check, smoke, GPU tests, a short bench (scratch output in gpurun_out/)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py --steps 10 --warmup 5 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cut -c1-1500 gpurun_out/bench.json
fi
