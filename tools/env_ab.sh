#!/bin/bash
# same-box A/B of environment settings on the bench solve (alternating, 2 runs each):
#   bash tools/env_ab.sh "SVK_X=0" "SVK_X=1" [extra bench args]
A=$1; B=$2; shift 2
for rep in 1 2; do
  for e in "$A" "$B"; do
    env $e python bench.py --no-cpu-baseline --no-e2e "$@" 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('%-24s %8.2f ms  its %d  vcycle %6.1f ms  orth %6.1f ms  sweep %.3f ms  sm %s' % ('$e', d['ms_per_step'], d['iterations'],
      1e3*d['t_vcycle_s'], 1e3*d['t_orth_s'], d['roofline']['avg_ms'] if d['roofline'] else -1, d['clocks']['sm_mhz'] if d['clocks'] else '?'))"
  done
done
