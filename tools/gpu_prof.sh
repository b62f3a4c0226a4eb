# ncu evidence of the current build (one GPU): launch list of bench steps, one
# --set full capture of the C4 search-level kernels and of the flat leaf sweep,
# exported to CSV on the box (the .ncu-rep files stay there).
set -x
mkdir -p gpurun_out/prof
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-flat --no-sa --no-comm --no-sim > gpurun_out/prof/launch_bench.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_level -c ${NCU_C:-6} -o /tmp/search_full python tools/ncu_one.py 4 > gpurun_out/prof/ncu_full.log 2>&1; echo ncu2=$?
ncu -i /tmp/search_full.ncu-rep --page raw --csv > gpurun_out/prof/search_raw.csv 2>&1
ncu -i /tmp/search_full.ncu-rep --page details --csv > gpurun_out/prof/search_details.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o /tmp/flat_full python tools/ncu_flat.py 4 2147483648 > gpurun_out/prof/ncu_flat.log 2>&1; echo ncu3=$?
ncu -i /tmp/flat_full.ncu-rep --page raw --csv > gpurun_out/prof/flat_raw.csv 2>&1
ncu -i /tmp/flat_full.ncu-rep --page details --csv > gpurun_out/prof/flat_details.csv 2>&1
ls -la gpurun_out/prof; du -sh gpurun_out
