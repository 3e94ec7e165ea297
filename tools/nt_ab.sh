#!/bin/bash
# A/B of the strip CTA size (libsvk_nt64.so vs libsvk_nt128.so, built with -DSVK_STRIP_THREADS)
for V in 64 128; do
  cp paper_2401_06277_b200/libsvk_nt$V.so paper_2401_06277_b200/libsvk.so
  echo "NT=$V"
  timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -1
  PYTHONPATH=. timeout 120 python tools/sweep_time.py 4096 2>&1 | head -2
  PYTHONPATH=. timeout 120 python tools/sweep_time.py 2048 2>&1 | head -1
  timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['time_to_solve_s'], d['t_vcycle_s'], d['t_orth_s'], d['sweep']['ms'])"
done
