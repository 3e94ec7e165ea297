#!/bin/bash
# A/B of library builds given as arguments: parity subset + serialised ncu kernel
# times of one 4096^2 V-cycle (tools/ab3.sh), then event-timed sweep / V-cycle
# (tools/sweep_time.py) alternating over the builds twice.
export PYTHONPATH=.
for lib in "$@"; do echo "== $lib"; bash tools/ab3.sh $lib; done
for rep in 1 2; do
  for lib in "$@"; do
    echo -n "$lib: "; SVK_LIBRARY=$lib timeout 300 python tools/sweep_time.py 4096 2>&1 | head -1
  done
done
