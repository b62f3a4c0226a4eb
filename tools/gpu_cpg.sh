#!/bin/bash
# sweep chunks per work item (grandparent placed once per item): flat 2^31 C4 slice, cascade, tests
for cpg in 1 4 13; do
  echo "cpg=$cpg $(CAMELOT_SWEEP_CPG=$cpg FLAT_SLICE=2147483648 timeout 300 python tools/flat_probe.py 4 2>&1 | tail -1 | cut -c1-60)"
done
timeout 600 python -m pytest tests/test_sweep.py tests/test_gpu_certify.py -q -x 2>&1 | tail -1
