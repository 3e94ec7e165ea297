#!/bin/bash
# Round-2 final bench session: smoke, bench (both arms), ncu launch list of one bench solve,
# V-cycle launch list, sizes.  Copied to profiles/r2c_* by hand (see tools/README.md).
mkdir -p gpurun_out
export PYTHONPATH=.
TAG=${1:-r2c}
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu_$TAG.log 2>&1
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/vcycle_launches.py 4096 > gpurun_out/vc_launches_$TAG.csv 2>/dev/null
timeout 1200 python tools/sizes_probe.py 1024 2048 4096 8192 > gpurun_out/sizes_$TAG.log 2>&1
tail -2 gpurun_out/smoke_$TAG.log; tail -c 600 gpurun_out/bench_$TAG.json
