#!/bin/bash
# A/B of library variants on the C4 step (host probe: both policies through the per-policy API, warm L2)
mkdir -p gpurun_out
for v in paper_2005_02088_b200/libcamelot.so ${VARIANTS}; do
  echo "== $v"
  CAMELOT_LIB=$PWD/$v timeout 120 python tools/host_probe.py 4 8 2>&1 | tail -3
  CAMELOT_LIB=$PWD/$v timeout 120 python tools/host_probe.py 7 4 2>&1 | tail -1
done
