#!/bin/bash
# multi-rank (emulated transport) parity + regression subset on one GPU
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -q -x 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_abi.py -m gpu -q -x 2>&1 | tail -5
