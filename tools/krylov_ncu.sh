#!/bin/bash
# ncu evidence for the Gram-Schmidt kernels (k_cgs_dots / k_cgs_update) inside one
# 4096^2 FGMRES solve: per-launch time + DRAM bytes for every launch, and one
# --set full capture of a late dots and a late update launch.
mkdir -p gpurun_out
TAG=${1:-r2}
PYTHONPATH=. timeout 900 ncu --profile-from-start off --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_cgs \
  --csv --log-file gpurun_out/krylov_launches_$TAG.csv python tools/ncu_vcycle.py 4096 fgmres > gpurun_out/krylov_ncu_$TAG.log 2>&1
PYTHONPATH=. timeout 900 ncu --profile-from-start off --clock-control none --set full --import-source on \
  -k regex:k_cgs -s 40 -c 3 -o gpurun_out/krylov_full_$TAG python tools/ncu_vcycle.py 4096 fgmres >> gpurun_out/krylov_ncu_$TAG.log 2>&1
tail -2 gpurun_out/krylov_ncu_$TAG.log
