#!/bin/bash
# Full GPU session: all GPU tests, then smoke/bench/launch list/ncu (gpu_round.sh).
mkdir -p gpurun_out
TAG=${1:-r1}
timeout 1200 python -m pytest tests/ -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; tail -3 gpurun_out/pytest_gpu_$TAG.log
bash tools/gpu_round.sh $TAG
