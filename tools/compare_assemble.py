"""Assemble profiles/<tag>_compare.json from the bench lines tools/compare_relax.sh writes."""
import glob
import json
import os
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r1d"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out_path = os.path.join(ROOT, "profiles", "r1_compare.json")
old = json.load(open(out_path))
names = {"vanka": "V(1,1)-Vanka", "bs": "V(1,1)-Braess-Sarazin", "su": "V(1,1)-Schur-Uzawa", "bt": "block-triangular"}


def load(p):
    d = json.load(open(p))
    return d


runs, variants = [], []
for kind in ("vanka", "bs", "bt", "su"):
    for n in (4096, 1024):
        p = os.path.join(ROOT, "gpurun_out", "compare_%s_%d_%s.json" % (kind, n, tag))
        if not os.path.exists(p):
            continue
        d = load(p)
        runs.append({"N": n, "preconditioner": names[kind], "iterations": d["iterations"],
                     "time_to_solve_s": d["time_to_solve_s"], "t_precond_s": d["t_vcycle_s"], "t_orth_s": d["t_orth_s"],
                     "rel_residual": d["rel_residual"], "dof_per_s": d["value"]})
for p in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "compare_sweep_*_%s.json" % tag))):
    d = load(p)
    impl, n = os.path.basename(p).split("_")[2:4]
    variants.append({"N": int(n), "sweep_impl": impl, "iterations": d["iterations"],
                     "time_to_solve_s": d["time_to_solve_s"], "sweep_ms": d["sweep"]["ms"],
                     "t_precond_s": d["t_vcycle_s"], "t_orth_s": d["t_orth_s"]})
if not runs:
    sys.exit("no compare_*_%s.json in gpurun_out/: profiles/r1_compare.json left unchanged" % tag)
old["runs"] = runs
old["vanka_variants"]["runs"] = variants
old["measured"] = "round 1, %s (kernel v9: symmetry-shared coefficients)" % tag
json.dump(old, open(out_path, "w"), indent=1)
print(json.dumps(runs, indent=0)[:2000])
