#!/bin/bash
# A/B of the sweep kernels: parity subset, device times, ncu capture
TAG=${1:-ab}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
for v in "SVK_NOTHING=1"; do
  echo "$v: $(env $v PYTHONPATH=. timeout 120 python tools/sweep_time.py 4096 2>&1 | tail -1)"
done
PYTHONPATH=. timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_vanka_fused -s 1 -c 1 -o gpurun_out/v8_${TAG} python tools/ncu_sweep.py 4096 > gpurun_out/ncu_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_${TAG}.log
