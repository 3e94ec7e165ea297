#!/bin/bash
# configs[4]: the same solve with Vanka, Braess-Sarazin and Schur-Uzawa relaxation (1 GPU).
# 4096^2: Vanka and BS (SU needs ~2.4 GB of Krylov vectors per iteration and more
# iterations than fit in HBM unrestarted); 1024^2: all three.
TAG=${1:-r1}
mkdir -p gpurun_out
run() {  # n relax maxit
  out=gpurun_out/compare_$2_$1_$TAG.json
  timeout 900 python bench.py --n $1 --relax $2 --maxit $3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $out 2> ${out%.json}.err
  python -c "import json;d=json.load(open('$out'));print('$1', '$2', d['iterations'], round(d['time_to_solve_s'],4), 's', round(d['t_vcycle_s'],4), round(d['t_orth_s'],4), '%.2e'%d['rel_residual'])" || tail -3 ${out%.json}.err
}
run 4096 vanka 60
run 4096 bs 60
run 1024 vanka 60
run 1024 bs 60
run 1024 su 200
# block-triangular preconditioner (alg:bt)
for n in 4096 1024; do
  out=gpurun_out/compare_bt_${n}_$TAG.json
  timeout 900 python bench.py --n $n --precond bt --maxit 60 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $out 2> ${out%.json}.err
  python -c "import json;d=json.load(open('$out'));print('$n', 'bt', d['iterations'], round(d['time_to_solve_s'],4), 's', round(d['t_vcycle_s'],4), round(d['t_orth_s'],4), '%.2e'%d['rel_residual'])" || tail -3 ${out%.json}.err
done
# tuned (fused, 25 shared inverses) vs the paper's simple Vanka (per-patch inverses, unfused split)
runs() {  # n sweep
  out=gpurun_out/compare_sweep_$2_$1_$TAG.json
  timeout 900 python bench.py --n $1 --sweep $2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $out 2> ${out%.json}.err
  python -c "import json;d=json.load(open('$out'));print('$1', '$2', d['iterations'], round(d['time_to_solve_s'],4), 's', 'sweep', round(d['sweep']['ms'],3), 'ms', round(d['t_vcycle_s'],4), round(d['t_orth_s'],4))" || tail -3 ${out%.json}.err
}
runs 1024 unfused
runs 1024 simple
runs 2048 fused
runs 2048 unfused
runs 2048 simple
