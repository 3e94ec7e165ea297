export PYTHONPATH=.
timeout 900 python -m pytest tests -m gpu -x -q -k "not 8192 and not large" 2>&1 | tail -3
for lib in tools/libsvk_base.so tools/libsvk_bd2.so; do
  echo "== $lib"
  SVK_LIBRARY=$lib timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv python tools/vcycle_launches.py 4096 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
bd=[float(r[vi].replace(',',''))/1e3 for r in rows[1:] if 'boundary' in r[ki]]
tot=sum(float(r[vi].replace(',',''))/1e3 for r in rows[1:])
print('bd us:', ' '.join('%.1f'%v for v in bd), ' sum %.1f  vcycle total %.1f us'%(sum(bd),tot))
"
done
bash tools/ab_bench.sh tools/libsvk_base.so tools/libsvk_bd2.so
