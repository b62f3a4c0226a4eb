#!/bin/bash
# sweep work-item shapes: chunks per item x guided tail fraction (flat 2^31 C4 slice)
for cpg in 4 7 13; do for tail in 8 4 2; do
  echo "cpg=$cpg tail=1/$tail $(CAMELOT_SWEEP_TAIL=$tail CAMELOT_SWEEP_CPG=$cpg FLAT_SLICE=2147483648 timeout 300 python tools/flat_probe.py 4 2>&1 | tail -1 | cut -c40-52)"
done; done
