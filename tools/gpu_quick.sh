#!/bin/bash
# quick round trip: GPU tests (all or PYTEST_K), bench core + flat leg, host probe, cascade probe (optional)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --no-sa --no-comm --no-sim > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_q.json").read())
print("step ms", d["ms_per_step"], "median", d["ms_per_step_median"], "e2e", d["e2e"]["ms_per_step"])
print("phases", {k: round(v, 4) for k, v in d["phases_ms"].items() if isinstance(v, float)})
print("flat", d["flat_scan"]["ms"], d["flat_scan"]["roofline"]["frac"], "c4b", d["c4b"]["ms_per_step_median"])
PY
timeout 120 python tools/host_probe.py 4 4 | tail -2
if [ -n "$CASCADE" ]; then timeout 600 python tools/cascade_probe.py 4; fi
if [ -n "$FTRACE" ]; then CAMELOT_LIB=$PWD/exp/libcamelot_ft.so timeout 200 python tools/trace_probe.py 4 2 > gpurun_out/ftrace_c4.txt 2>&1; echo ftrace=$?; fi
