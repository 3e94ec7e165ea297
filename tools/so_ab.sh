#!/bin/bash
# A/B two prebuilt libraries (paper_2401_06277_b200/libsvk_<A>.so, libsvk_<B>.so) on the same box
for V in "$@"; do for rep in 1 2; do
  cp paper_2401_06277_b200/libsvk_$V.so paper_2401_06277_b200/libsvk.so
  echo -n "$V: "
  timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['time_to_solve_s'], d['t_vcycle_s'], d['t_orth_s'], d['sweep']['ms'])"
done; done
