#!/bin/bash
for v in base minb3; do
  if [ $v = base ]; then L=""; else L="CAMELOT_LIB=$PWD/exp/$v/libcamelot.so"; fi
  env $L FLAT_SLICE=2147483648 timeout 300 python tools/flat_probe.py 4 2>&1 | tail -1 | cut -c1-90 | sed "s/^/$v /"
done
