#!/bin/bash
# the heavy C4-shaped instances: per-pass mode (FTRACE build) and the frontier clamp
for fm in 2097152 8388608; do
  echo "== fmax=$fm"
  for x in x2 x3; do
    CAMELOT_FRONTIER_MAX=$fm CAMELOT_LIB=$PWD/exp/libcamelot_ft.so timeout 300 python tools/trace_probe.py $x 2 2>&1 | grep -A4 "max-load rep 1" | tail -1 | tr ' ' '\n' | grep -E "^p[0-9]=|par|bat[0-9]|maxb" | tr '\n' ' '; echo
    CAMELOT_FRONTIER_MAX=$fm timeout 300 python tools/trace_probe.py $x 2 2>&1 | grep kernel | tail -2
  done
done
