#!/bin/bash
# ncu source-level capture of the max-load search launch (warp-mode lines = shallow passes)
mkdir -p gpurun_out/prof
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:search_level -s 2 -c 1 -o /tmp/search_src python tools/pair_step.py 4 2 > gpurun_out/prof/ncu_src.log 2>&1; echo ncu=$?
ncu -i /tmp/search_src.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/prof/search_source.csv 2>&1
ls -la gpurun_out/prof/search_source.csv
