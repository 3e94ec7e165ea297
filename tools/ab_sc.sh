#!/bin/bash
# small-cycle A/B: GPU tests, per-launch V-cycle times, solve A/B vs the previous build
export PYTHONPATH=.
timeout 900 python -m pytest tests -m gpu -x -q -k "not 8192 and not large" 2>&1 | tail -4
for lib in tools/libsvk_bd2.so tools/libsvk_sc.so; do
  echo "== $lib"
  SVK_LIBRARY=$lib timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/vcycle_launches.py 4096 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
ks=[(r[ki].split('(')[0].replace('void ',''), float(r[vi].replace(',',''))/1e3) for r in rows[1:]]
print(' '.join('%s:%.1f'%(k[:14],v) for k,v in ks if v < 60 or 'small' in k))
print('launches %d  vcycle total %.1f us'%(len(ks), sum(v for k,v in ks)))
"
done
bash tools/ab_bench.sh tools/libsvk_bd2.so tools/libsvk_sc.so
for lib in tools/libsvk_bd2.so tools/libsvk_sc.so; do
  SVK_LIBRARY=$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e --n 1024 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('1024 mms', '$lib', d['ms_per_step'], d['iterations'], d.get('t_vcycle_s'))"
done
