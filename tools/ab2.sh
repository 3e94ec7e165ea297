#!/bin/bash
# quick A/B: parity subset, device times of the fused sweep / V-cycle / residual, x=0 sweep launch times
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sweep or vcycle or fgmres" 2>&1 | tail -2
PYTHONPATH=. timeout 120 python tools/sweep_time.py 4096 2>&1 | tail -2
PYTHONPATH=. timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_vanka -c 6 --csv python tools/zero_probe.py 4096 2>/dev/null | grep -E "k_vanka" | awk -F'","' '{print $5, $NF}' | head -6
