#!/bin/bash
# quick iteration: sweep/vcycle parity subset, perf probe, ncu of the fused kernel
TAG=${1:-q}
mkdir -p gpurun_out
timeout 240 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sweep or vcycle or fgmres" 2>&1 | tail -3
PYTHONPATH=. timeout 120 python tools/perf_probe.py 4096 2>&1 | head -3
PYTHONPATH=. timeout 240 ncu --set full --clock-control none --import-source on -k regex:k_vanka_fused -s 1 -c 1 -o gpurun_out/fused_$TAG python tools/ncu_sweep.py 4096 > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
