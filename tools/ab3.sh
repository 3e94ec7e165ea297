#!/bin/bash
# quick A/B of the sweep kernels: parity subset, then ncu device times (serialised,
# --clock-control none) of k_boundary_patches, k_vanka_fused, k_vanka_zero and the
# residual strips at 4096^2 inside one V-cycle.  Optional $1 = SVK_LIBRARY path.
[ -n "$1" ] && export SVK_LIBRARY=$1
export PYTHONPATH=.
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "sweep or vcycle or fullsize" 2>&1 | tail -1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/ncu_vcycle.py 4096 vcycle 2>/dev/null \
  | python -c "
import csv,sys,collections
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
t=collections.OrderedDict(); n=collections.Counter()
for r in rows[1:]:
    k=r[ki].split('(')[0].replace('void ','')
    t[k]=t.get(k,0)+float(r[vi].replace(',',''))/1e3; n[k]+=1
tot=sum(t.values())
for k,v in sorted(t.items(), key=lambda kv:-kv[1])[:8]: print('%-40s %3d launches %8.3f ms'%(k,n[k],v/1e3))
print('total %.3f ms'%(tot/1e3))
"
