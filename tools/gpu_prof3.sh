#!/bin/bash
# FTRACE phase trace of the C4 plans; ncu --set full (with source) of the cascade sweep
mkdir -p gpurun_out/prof
CAMELOT_LIB=$PWD/exp/libcamelot_ft.so timeout 200 python tools/trace_probe.py 4 2 > gpurun_out/ftrace_c4.txt 2>&1; echo ftrace=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 -o /tmp/sw50 python tools/ncu_one.py 4 > gpurun_out/prof/sw50.log 2>&1; echo ncu2=$?
ncu -i /tmp/sw50.ncu-rep --page raw --csv > gpurun_out/prof/sw50_raw.csv 2>&1
ncu -i /tmp/sw50.ncu-rep --page details --csv > gpurun_out/prof/sw50_details.csv 2>&1
ncu -i /tmp/sw50.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof/sw50_source.csv 2>&1
ls -la gpurun_out/prof
