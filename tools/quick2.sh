#!/bin/bash
# parity (all GPU tests) + per-level probe + V-cycle launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -q -x 2>&1 | tail -3
PYTHONPATH=. timeout 120 python tools/level_probe.py 4096
PYTHONPATH=. timeout 300 python tools/orth_probe.py 4096
PYTHONPATH=. timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/vcycle_launches.csv python tools/ncu_vcycle.py 4096 > /dev/null 2>&1
