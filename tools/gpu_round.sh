#!/bin/bash
# One GPU session: smoke, bench (both arms), launch list and a full ncu capture
# of the fused sweep.  Outputs land in gpurun_out/ (merged back by gpurun).
set -x
mkdir -p gpurun_out
TAG=${1:-r1}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
./tools/fp64_peak > gpurun_out/fp64_peak_$TAG.json 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu_$TAG.log 2>&1
PYTHONPATH=. timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_vanka_fused -s 1 -c 1 \
    -o gpurun_out/sweep_full_$TAG python tools/ncu_sweep.py 4096 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -3 gpurun_out/smoke_$TAG.log; cat gpurun_out/bench_$TAG.json gpurun_out/bench_ref_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
