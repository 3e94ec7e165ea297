#!/bin/bash
# Round-2 late GPU session (after the DMMA boundary kernel and the one-launch coarse
# cycle): smoke, FP64 peak, bench (both arms), ncu launch list of one bench solve,
# ncu --set full of the fused sweep, the x=0 sweep, the boundary kernel and the coarse
# cycle, sizes.  Outputs in gpurun_out/ (copied to profiles/ by tools/refresh_profiles_r2b.sh).
mkdir -p gpurun_out
export PYTHONPATH=.
TAG=${1:-r2b}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
./tools/fp64_peak > gpurun_out/fp64_peak_$TAG.json 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_vanka_fused -s 1 -c 1 \
    -o gpurun_out/sweep_full_$TAG python tools/ncu_sweep.py 4096 > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --profile-from-start off -k regex:k_vanka_zero -s 0 -c 1 \
    -o gpurun_out/zero_full_$TAG python tools/vcycle_launches.py 4096 > gpurun_out/ncu_zero_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --profile-from-start off -k regex:k_boundary_patches -s 0 -c 1 \
    -o gpurun_out/bd_full_$TAG python tools/vcycle_launches.py 4096 > gpurun_out/ncu_bd_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --profile-from-start off -k regex:k_small_cycle -s 0 -c 1 \
    -o gpurun_out/sc_full_$TAG python tools/vcycle_launches.py 4096 > gpurun_out/ncu_sc_$TAG.log 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/vcycle_launches.py 4096 > gpurun_out/vc_launches_$TAG.csv 2>/dev/null
timeout 1200 python tools/sizes_probe.py 1024 2048 4096 8192 > gpurun_out/sizes_$TAG.log 2>&1
tail -2 gpurun_out/smoke_$TAG.log; tail -c 400 gpurun_out/bench_$TAG.json; tail -c 300 gpurun_out/bench_ref_$TAG.json
