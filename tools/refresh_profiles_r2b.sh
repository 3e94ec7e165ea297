#!/bin/bash
# Copy the round-2 late session (tools/refresh_r2b.sh TAG) into profiles/r2b_*.
TAG=${1:-r2b}
set -e
for k in sweep:k_vanka_fused zero:k_vanka_zero bd:k_boundary_patches sc:k_small_cycle; do
  n=${k%%:*}; kern=${k#*:}
  (echo "# ncu --set full --clock-control none (tools/refresh_r2b.sh): $kern, 4096^2 (first launch of a preconditioner V-cycle; the sweep: tools/ncu_sweep.py)"
   python tools/ncu_summary.py gpurun_out/${n}_full_$TAG.ncu-rep) > profiles/r2b_${n}_ncu.txt
done
cp gpurun_out/bench_$TAG.json profiles/r2b_bench.json
cp gpurun_out/bench_ref_$TAG.json profiles/r2b_bench_reference.json
cp gpurun_out/launches_$TAG.csv profiles/r2b_launches.csv
cp gpurun_out/fp64_peak_$TAG.json profiles/r2b_fp64_peak.json
python tools/launches.py profiles/r2b_launches.csv > profiles/r2b_launches_summary.txt
(echo "# per-launch device times of one 4096^2 preconditioner V-cycle (ncu, serialised; tools/vcycle_launches.py)"
 python tools/launches.py gpurun_out/vc_launches_$TAG.csv all) > profiles/r2b_vcycle_launches.txt
cp gpurun_out/sizes.json profiles/r2b_sizes.json
head -12 profiles/r2b_launches_summary.txt
