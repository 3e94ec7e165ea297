#!/bin/bash
# parity subset + device times (A/B of the x = 0 pre-smoothing kernel)
TAG=${1:-ab}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "vcycle or fgmres" 2>&1 | tail -2
PYTHONPATH=. timeout 120 python tools/sweep_time.py 4096 2>&1 | tail -2
SVK_ZERO_V8=1 PYTHONPATH=. timeout 120 python tools/sweep_time.py 4096 2>&1 | tail -2
PYTHONPATH=. timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/vc_launches_$TAG.csv python tools/ncu_vcycle.py 4096 > /dev/null 2>&1
