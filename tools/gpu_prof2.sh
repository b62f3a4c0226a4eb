#!/bin/bash
# launch list of two C4 plan pairs; full capture of the cascade sweep and of the flat sweep
mkdir -p gpurun_out/prof
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches.csv python tools/ncu_one.py 4 > gpurun_out/prof/launch.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 -o /tmp/sw50 python tools/ncu_one.py 4 > gpurun_out/prof/sw50.log 2>&1; echo ncu2=$?
ncu -i /tmp/sw50.ncu-rep --page raw --csv > gpurun_out/prof/sw50_raw.csv 2>&1
ncu -i /tmp/sw50.ncu-rep --page details --csv > gpurun_out/prof/sw50_details.csv 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o /tmp/flat python tools/ncu_flat.py 4 2147483648 > gpurun_out/prof/flat.log 2>&1; echo ncu3=$?
ncu -i /tmp/flat.ncu-rep --page raw --csv > gpurun_out/prof/flat_raw.csv 2>&1
ncu -i /tmp/flat.ncu-rep --page details --csv > gpurun_out/prof/flat_details.csv 2>&1
ncu -i /tmp/flat.ncu-rep --page source --csv > gpurun_out/prof/flat_source.csv 2>&1
ls -la gpurun_out/prof
