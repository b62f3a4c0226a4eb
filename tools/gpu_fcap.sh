#!/bin/bash
# frontier capacity vs the C4b main level (FTRACE build: per-pass parents, items, max items per warp)
for fm in 1048576 4194304 8388608; do
  echo "fmax=$fm"
  CAMELOT_FRONTIER_MAX=$fm CAMELOT_LIB=$PWD/exp/libcamelot_ft.so timeout 200 python tools/trace_probe.py 7 2 2>&1 | grep -A4 "max-load rep 1" | tail -1 | tr ' ' '\n' | grep -E "^p[0-9]=|par|bat[0-9]|maxb|tc" | tr '\n' ' '; echo
  CAMELOT_FRONTIER_MAX=$fm timeout 200 python tools/trace_probe.py 7 2 2>&1 | grep kernel | tail -2
done
