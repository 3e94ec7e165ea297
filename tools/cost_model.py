"""the paper's operation-count model (tab:rwf, tab:aiperf,
P:486-535) next to this build's fused B200 kernels.  Writes profiles/<tag>_cost_model.md.

    python tools/cost_model.py [tag]   (reads profiles/<tag>_bench.json for measured times)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
A100_BW, A100_FP64 = 1264.42e9, 9472.34e9
B200_BW = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9 \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6454e9
B200_FP64 = 148 * 64 * 2 * 1.965e9


def paper_vanka(N):
    """tab:rwf Vanka rows (doubles / flops) with l = N - 1 (l + 2 nodal DOFs per dimension),
    plus the residual it needs (two Q2*Q2, two Q2Q1*Q2 (B), two Q2Q1*Q1 (B^T) products and an
    array minus), in the paper's own (dense-count) formulas with n = velocity, m = pressure DOFs."""
    l = N - 1
    form = 76 + 124 * l + 51 * l * l
    apply_r, apply_f = 1520 + 3968 * l + 2652 * l * l, 2888 + 7688 * l + 5202 * l * l
    upd = 76 + 124 * l + 51 * l * l          # reading 11: "51 l" read as 51 l^2
    return {"form": (form, form, 0), "apply": (apply_r, form, apply_f), "update": (upd, upd, upd)}


def row(name, r, w, f):
    ai = f / (8.0 * (r + w)) if r + w else 0.0
    t = max(8.0 * (r + w) / A100_BW, f / A100_FP64)
    tb = max(8.0 * (r + w) / B200_BW, f / B200_FP64)
    return "| %s | %.4g | %.4g | %.4g | %.4f | %.1f | %.3f | %.3f |" % (name, r, w, f, ai, f / t / 1e9 if t else 0, 1e3 * t, 1e3 * tb)


lines = ["# Cost model: the paper's counts (tab:rwf / tab:aiperf) vs the fused B200 sweep (%s)" % tag, "",
         "Doubles read / written and flops per Vanka sweep, AI = flops / (8 B x doubles) (P:510-516 with",
         "8-byte doubles, which reproduces tab:aiperf's AI column, `test_tab_aiperf_reproduces_with_8_byte_doubles`),",
         "and the roofline time max(bytes/BW, flops/peak) on the paper's A100 (1264.42 GB/s, 9472.34 GFLOP/s,",
         "P:397) and on B200 (%.0f GB/s measured, %.1f TFLOP/s FP64 derived)." % (B200_BW / 1e9, B200_FP64 / 1e12), ""]
try:
    bench = json.load(open(os.path.join(ROOT, "profiles", "%s_bench.json" % tag)))
    meas_ms = bench["sweep"]["ms"]
except Exception:
    bench, meas_ms = None, None
for N in (512, 4096):
    nodes = (N + 1) ** 2
    ndof = 2 * (2 * N + 1) ** 2 + nodes
    lines += ["## %d x %d elements (%d DOFs, %d patches)" % (N, N, ndof, nodes), "",
              "| kernel | reads [double] | writes [double] | flops | AI [flop/B] | A100 roofline GFLOP/s | A100 roofline ms | B200 roofline ms |",
              "|---|---|---|---|---|---|---|---|"]
    pv = paper_vanka(N)
    tot = [0, 0, 0]
    for k, name in (("form", "Vanka: form patch RHS (tab:rwf)"), ("apply", "Vanka: apply matrix inverse (tab:rwf)"),
                    ("update", "Vanka: update global solution (tab:rwf)")):
        r, w, f = pv[k]
        tot = [tot[0] + r, tot[1] + w, tot[2] + f]
        lines.append(row(name, r, w, f))
    # residual of the paper's split sweep: read x, b, write r (fused stencil, this build's flop count)
    res = (18 * nodes, 9 * nodes, 361 * nodes)
    lines.append(row("residual r = b - A x (stencil; 361 flop/node)", *res))
    tot = [tot[0] + res[0], tot[1] + res[1], tot[2] + res[2]]
    lines.append(row("**paper's split sweep, total** (apply reads every patch's inverse: simple Vanka)", *tot))
    form = pv["form"][0]
    tuned = (tot[0] - pv["apply"][0] + form, tot[1], tot[2])  # tuned: 25 shared inverses stay on chip, apply reads the RHS
    lines.append(row("**paper's split sweep, tuned** (25 shared inverses on chip, P:469)", *tuned))
    fused = (18 * nodes, 9 * nodes, 1316 * nodes)
    lines.append(row("**this build: fused sweep (27 doubles, 1316 flop per node)**", *fused))
    lines += ["", "Traffic ratio split (simple) / fused: %.1fx; split (tuned) / fused: %.1fx; flop ratio: %.1fx."
              % ((tot[0] + tot[1]) / (fused[0] + fused[1]), (tuned[0] + tuned[1]) / (fused[0] + fused[1]), tot[2] / fused[2])]
    if N == 4096 and meas_ms:
        lines += ["Measured fused sweep at 4096^2 (profiles/%s_bench.json): %.3f ms = %.1f%% of its B200 roofline time "
                  "(%.3f ms); the paper's split sweep could not run faster than %.3f ms (tuned) on B200 even at its roofline."
                  % (tag, meas_ms, 100 * max(8 * (fused[0] + fused[1]) / B200_BW, fused[2] / B200_FP64) * 1e3 / meas_ms,
                     1e3 * max(8 * (fused[0] + fused[1]) / B200_BW, fused[2] / B200_FP64),
                     1e3 * max(8 * (tuned[0] + tuned[1]) / B200_BW, tuned[2] / B200_FP64))]
    lines.append("")
lines += ["tab:aiperf's performance column is not reproduced from the stated A100 bandwidth (DESIGN.md reading 12);",
          "the paper reports the interior apply kernel at ~2145 GFLOP/s on A100 at 1024^2 (P:640)."]
out = os.path.join(ROOT, "profiles", "%s_cost_model.md" % tag)
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
