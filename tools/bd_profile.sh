export PYTHONPATH=.
mkdir -p gpurun_out
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv python tools/vcycle_launches.py 4096 > gpurun_out/vc_launches_4096.csv 2>/dev/null
timeout 300 ncu --profile-from-start off --set full --clock-control none -k regex:k_boundary_patches -c 2 -o gpurun_out/bd_full python tools/vcycle_launches.py 4096 > /dev/null 2>&1
ncu -i gpurun_out/bd_full.ncu-rep --page raw --csv > gpurun_out/bd_full_raw.csv 2>/dev/null
ls -la gpurun_out
