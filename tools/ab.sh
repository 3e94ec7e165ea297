#!/bin/bash
# parity + device times
TAG=${1:-ab}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_comparators.py -m gpu -q -x 2>&1 | tail -2
PYTHONPATH=. timeout 120 python tools/sweep_time.py 4096 2>&1 | tail -2
