#!/bin/bash
# Round-2 GPU session for the committed profiles: smoke, FP64 peak probe, bench
# (both arms), ncu launch list of one bench solve, ncu --set full of the fused
# sweep, per-size probe.  Outputs in gpurun_out/ (copied to profiles/ by hand).
mkdir -p gpurun_out
TAG=${1:-r2final}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
./tools/fp64_peak > gpurun_out/fp64_peak_$TAG.json 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu_$TAG.log 2>&1
PYTHONPATH=. timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_vanka_fused -s 1 -c 1 \
    -o gpurun_out/sweep_full_$TAG python tools/ncu_sweep.py 4096 > gpurun_out/ncu_full_$TAG.log 2>&1
PYTHONPATH=. timeout 600 ncu --set full --clock-control none -k regex:k_vanka_zero -s 1 -c 1 \
    -o gpurun_out/zero_full_$TAG python tools/ncu_vcycle.py 4096 fgmres > gpurun_out/ncu_zero_$TAG.log 2>&1
PYTHONPATH=. timeout 1200 python tools/sizes_probe.py 1024 2048 4096 8192 > gpurun_out/sizes_$TAG.log 2>&1
tail -2 gpurun_out/smoke_$TAG.log; tail -c 400 gpurun_out/bench_$TAG.json; tail -c 300 gpurun_out/bench_ref_$TAG.json
