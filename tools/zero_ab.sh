#!/bin/bash
# k_vanka_zero at 4096^2 (first launch of a preconditioner V-cycle) for library builds given as arguments
export PYTHONPATH=.
for lib in "$@"; do
  echo "== $lib"
  SVK_LIBRARY=$lib timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__occupancy_limit_registers,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:k_vanka_zero -c 1 --csv python tools/vcycle_launches.py 4096 2>/dev/null | grep k_vanka_zero | awk -F'","' '{print $(NF-3), $(NF-1), $NF}'
done
