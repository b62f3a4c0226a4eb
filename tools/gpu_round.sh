set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 10 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-flat --no-sa > /dev/null 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_level -c 6 -o gpurun_out/search_full python tools/ncu_one.py 4 > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search -c 3 -o gpurun_out/flat_full python tools/ncu_flat.py 6 > gpurun_out/ncu_flat.log 2>&1; echo ncu3=$?
