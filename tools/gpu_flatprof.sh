#!/bin/bash
# ncu --set full (with source) of the flat sweep over a 2^31 C4 slice; flat timing
mkdir -p gpurun_out/prof
FLAT_SLICE=2147483648 timeout 300 python tools/flat_probe.py 4 > gpurun_out/flat_probe.txt 2>&1; echo probe=$?; tail -3 gpurun_out/flat_probe.txt | cut -c1-200
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o /tmp/flat_full python tools/ncu_flat.py 4 2147483648 > gpurun_out/prof/ncu_flat.log 2>&1; echo ncu3=$?
ncu -i /tmp/flat_full.ncu-rep --page raw --csv > gpurun_out/prof/flat_raw.csv 2>&1
ncu -i /tmp/flat_full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof/flat_source.csv 2>&1
