#!/bin/bash
# V-cycle (4096^2 and 1024^2) per-launch totals for several SVK_SMALL_N thresholds
export PYTHONPATH=.
for n in 4096 1024; do
for lc in 0 16 32 64; do
  echo -n "N=$n SVK_SMALL_N=$lc: "
  SVK_DEBUG_SMALL=1 SVK_SMALL_N=$lc timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/vcycle_launches.py $n 2>&1 | python -c "
import csv,sys
lines=sys.stdin.read().splitlines()
dbg=[l for l in lines if l.startswith('[small')]
rows=[r for r in csv.reader(lines) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
ks=[(r[ki].split('(')[0].replace('void ',''), float(r[vi].replace(',',''))/1e3) for r in rows[1:]]
sc=[v for k,v in ks if 'small' in k]
print('launches %d total %.1f us small %s %s'%(len(ks), sum(v for k,v in ks), sc, dbg[:1]))
"
done; done
