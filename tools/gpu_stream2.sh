#!/bin/bash
# streaming-phase knobs: depths streamed and idle backoff, C4 kernel times
for k in 0 2 3; do for nap in 4096 32768; do
  echo "K=$k nap=$nap: $(CAMELOT_STREAM=$k CAMELOT_STREAM_NAP=$nap timeout 120 python tools/trace_probe.py 4 3 2>&1 | grep kernel | tail -4 | awk '{print $2, $6}' | tr '\n' ' ')"
done; done
