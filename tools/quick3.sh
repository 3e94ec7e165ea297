#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -q -x -k "sweep or vcycle or fgmres" 2>&1 | tail -2
PYTHONPATH=. timeout 120 python tools/level_probe.py 4096
PYTHONPATH=. timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/vcycle_launches.csv python tools/ncu_vcycle.py 4096 > /dev/null 2>&1
PYTHONPATH=. timeout 300 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_residual_strip -c 1 -o gpurun_out/rr_mode1 python tools/ncu_vcycle.py 4096 > gpurun_out/rr.log 2>&1; tail -2 gpurun_out/rr.log
