#!/bin/bash
# Copy one GPU session's outputs (tools/gpu_full.sh TAG, compare_relax.sh TAG, sizes_probe) into profiles/.
TAG=${1:?tag}
set -e
python tools/ncu_summary.py gpurun_out/sweep_full_$TAG.ncu-rep > /tmp/sw.json
(echo "# ncu --set full --clock-control none --import-source on -k regex:k_vanka_fused -s 1 -c 1 python tools/ncu_sweep.py 4096"
 echo "# round 1 ($TAG), kernel v9: symmetry-shared coefficients, unmasked sweep residual, incremental ring slots, 64-row chunks, 2-warp strips, PDL"
 cat /tmp/sw.json) > profiles/r1_sweep_ncu.txt
python - <<'PY'
import json
d = json.load(open('/tmp/sw.json'))[0]
sc = {'Gbyte': 1e9, 'Mbyte': 1e6}
tot = sum(float(d[k].split()[0]) * sc[d[k].split()[1]] for k in ('dram__bytes_read.sum', 'dram__bytes_write.sum'))
t = json.load(open('profiles/traffic.json'))
t['bytes_per_launch'] = tot
json.dump(t, open('profiles/traffic.json', 'w'), indent=1)
print('traffic', tot, d['gpu__time_duration.sum'])
PY
cp gpurun_out/bench_$TAG.json profiles/r1_bench.json
cp gpurun_out/bench_ref_$TAG.json profiles/r1_bench_reference.json
cp gpurun_out/launches_$TAG.csv profiles/r1_launches.csv
cp gpurun_out/fp64_peak_$TAG.json profiles/r1_fp64_peak.json
python tools/launches.py profiles/r1_launches.csv > profiles/r1_launches_summary.txt
python tools/compare_assemble.py $TAG > /dev/null || true
if [ -f gpurun_out/sizes.json ]; then python - <<'PY'
import json
d = json.load(open('gpurun_out/sizes.json'))
p = json.load(open('profiles/r1_sizes.json'))
p['runs'] = d
json.dump(p, open('profiles/r1_sizes.json', 'w'), indent=1)
PY
fi
head -8 profiles/r1_launches_summary.txt
