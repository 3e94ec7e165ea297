"""Generate paper_2401_06277_b200/csrc/solve_gen.cuh: the generic-patch solve
with every stored coefficient loaded once and applied at all the positions its
symmetry orbit covers.

Background.  In the reflection (even/odd) basis the generic
patch's velocity inverse is B = S T Lw^-1 T^T S (T = T5 (x) T5, S the folded
1/2 scaling), which is block diagonal (EE 9x9, EO 6x6, OE 6x6, OO 4x4) and
  * symmetric:            B[r][c] = B[c][r]            (Lw symmetric)
  * axis-swap invariant:  B[r][c] = B[sr][sc],  s(ty,tx) = (tx,ty)
                          (Lw = nu(M_w (x) K_w + K_w (x) M_w) is unchanged when
                          the two axes are swapped; this maps EE->EE, OO->OO,
                          EO<->OE)
and the Schur vectors satisfy chy = s(chx), cpy = s(cpx) (b_y is b_x with the
axes swapped).  k_factor_setup enforces these identities bitwise (it averages
each orbit), so one constant-bank load per orbit serves up to 4 positions x 2
velocity components = 8 FMAs instead of 2.  The kernel is bound by delivering
uniform constants to the FP64 pipe (tools/mb_cbank.cu measures DFMA throughput
at ~45% of peak when each DFMA needs its own streamed constant at 8 warps/SM),
so this is the lever; the FMA count itself is unchanged (169 per component).

Output: straight-line code, deterministic (fixed order per accumulator).
"""
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2401_06277_b200", "csrc")


def par(i):  # 0..2 even, 3..4 odd
    return i < 3


def sig(r):
    ty, tx = divmod(r, 5)
    return tx * 5 + ty


def stored(r, c):
    """parameter expression holding B[r][c] (r, c in the same parity block)"""
    ry, rx = divmod(r, 5)
    cy, cx = divmod(c, 5)
    assert par(ry) == par(cy) and par(rx) == par(cx)
    if par(ry) and par(rx):
        return "F.bee[%d][%d]" % (ry * 3 + rx, cy * 3 + cx)
    if par(ry) and not par(rx):
        return "F.beo[%d][%d]" % (ry * 2 + rx - 3, cy * 2 + cx - 3)
    if not par(ry) and par(rx):
        return "F.boe[%d][%d]" % ((ry - 3) * 3 + rx, (cy - 3) * 3 + cx)
    return "F.boo[%d][%d]" % ((ry - 3) * 2 + rx - 3, (cy - 3) * 2 + cx - 3)


def block_positions(kind):
    e = lambda i: i < 3
    out = []
    for r in range(25):
        ty, tx = divmod(r, 5)
        if kind == "EE" and e(ty) and e(tx):
            out.append(r)
        elif kind == "EOOE" and e(ty) != e(tx):
            out.append(r)
        elif kind == "EO" and e(ty) and not e(tx):
            out.append(r)
        elif kind == "OE" and not e(ty) and e(tx):
            out.append(r)
        elif kind == "OO" and not e(ty) and not e(tx):
            out.append(r)
    return out


def same_block(r, c):
    return par(r // 5) == par(c // 5) and par(r % 5) == par(c % 5)


def emit(kind):
    """declare accumulators up front, then orbit blocks, then write-back"""
    pos = block_positions(kind)
    L = ["  {  // %s: %d positions per component" % (kind, len(pos))]
    L.append("    double " + ", ".join("sx%d = 0.0, sy%d = 0.0" % (r, r) for r in pos) + ";")
    seen = set()
    for r in pos:
        for c in pos:
            if not same_block(r, c) or (r, c) in seen:
                continue
            orbit = []
            for m in [(r, c), (c, r), (sig(r), sig(c)), (sig(c), sig(r))]:
                if m[0] in pos and m not in orbit:
                    orbit.append(m)
            seen.update(orbit)
            L.append("    {")
            L.append("      const double k = %s;" % stored(r, c))
            for (rr, cc) in orbit:
                L.append("      sx%d = fma(k, vx[%d], sx%d);" % (rr, cc, rr))
                L.append("      sy%d = fma(k, vy[%d], sy%d);" % (rr, cc, rr))
            L.append("    }")
    for r in pos:
        L.append("    vx[%d] = sx%d;" % (r, r))
        L.append("    vy[%d] = sy%d;" % (r, r))
    L.append("  }")
    return L


def stencil_code():
    """Residual stencils of the fused sweep with shared constants.

    L part: output o in {0:(j0,c0), 1:(j0,c0+1), 2:(j1,c0), 3:(j1,c0+1)} of the
    5x5 window U (rows 2sp..2sp+4, columns c0-2..c0+2), centres (1,2) (1,3)
    (2,2) (2,3); row parity py = 1 (j0 odd) / 0, column parity px = 0 / 1.
    Coefficient L2D[py][px][db+2][da+2] = nu (M_py[db] K_px[da] + K_py[db] M_px[da])
    depends only on (|db|, |da|) (1D Q2 stencils are reflection symmetric) and
    L2D[py][px][b][a] = L2D[px][py][a][b]; one load per class of equal values.
    B part (interior pressure node): PBY[oy][ox] = PBX[ox][oy]."""
    taps = {}
    centres = {0: (1, 2, 1, 0), 1: (1, 3, 1, 1), 2: (2, 2, 0, 0), 3: (2, 3, 0, 1)}
    for o, (ry, rx, py, px) in centres.items():
        hb = 1 if py == 1 else 2
        ha = 1 if px == 1 else 2
        for db in range(-hb, hb + 1):
            for da in range(-ha, ha + 1):
                b, a = abs(db), abs(da)
                if (py, px) == (0, 1):
                    key = (1, 0, a, b)
                elif py == px:
                    key = (py, px, min(a, b), max(a, b))
                else:
                    key = (py, px, b, a)
                taps.setdefault(key, []).append((o, ry + db, rx + da))
    L = [
        "// L x on the four lattice points of the residual step (fused_residual_vals):",
        "// ax[0..3] u_x, ax[4..7] u_y; U/V = 5x5 windows.  Generated (see stencil_code).",
        "__device__ __forceinline__ void stencil_L_sym(const double (&U)[5][5], const double (&V)[5][5], double (&ax)[8],",
        "                                              const FusedFactors& F) {",
    ]
    for key in sorted(taps):
        py, px, b, a = key
        L.append("  {")
        L.append("    const double k = F.L2D[%d][%d][%d][%d];" % (py, px, b + 2, a + 2))
        for (o, r, c) in taps[key]:
            L.append("    ax[%d] = fma(k, U[%d][%d], ax[%d]);" % (o, r, c, o))
            L.append("    ax[%d] = fma(k, V[%d][%d], ax[%d]);" % (o + 4, r, c, o + 4))
        L.append("  }")
    L.append("}")
    L.append("// B u at an interior pressure node: PBY[oy][ox] = PBX[ox][oy]")
    L.append("__device__ __forceinline__ double stencil_B_sym(const double (&U)[5][5], const double (&V)[5][5],")
    L.append("                                                const FusedFactors& F) {")
    L.append("  double bu = 0.0, bv = 0.0;")
    for r in (1, 2, 3):
        for ox in (0, 1, 3, 4):
            L.append("  {")
            L.append("    const double k = F.PBX[%d][%d];" % (r, ox))
            L.append("    bu = fma(k, U[%d][%d], bu);" % (r, ox))
            L.append("    bv = fma(k, V[%d][%d], bv);" % (ox, r))
            L.append("  }")
    L.append("  return bu + bv;")
    L.append("}")
    return L


def main(outdir=CSRC):
    OUT = os.path.join(outdir, "solve_gen.cuh")
    OUT_ST = os.path.join(outdir, "stencil_gen.cuh")
    L = [
        "// solve_gen.cuh -- GENERATED by tools/gen_solve.py; do not edit.",
        "// Generic-patch solve in the reflection basis with symmetry-shared",
        "// coefficients (see the generator's docstring and DESIGN.md section 7).",
        "#pragma once",
        "",
        "namespace svk {",
        "",
        "// (vx, vy) = patch residual window in, (du, dv) out; rp = pressure residual;",
        "// returns dp.  Same steps as solve_generic (even/odd transform, blocks, Schur).",
        "__device__ __forceinline__ double solve_generic_sym(double (&vx)[25], double (&vy)[25], double rp,",
        "                                                    const FusedFactors& F) {",
        "  fwd_transform(vx);",
        "  fwd_transform(vy);",
        "  // Schur unknown: chy = s(chx), i.e. chy[b*3+a] = chx[a*2+b]",
        "  double sx = 0.0, sy = 0.0;",
    ]
    for a in range(3):
        for b in range(2):
            L.append("  {")
            L.append("    const double k = F.chx[%d];" % (a * 2 + b))
            L.append("    sx = fma(k, vx[%d], sx);" % (a * 5 + 3 + b))
            L.append("    sy = fma(k, vy[%d], sy);" % ((3 + b) * 5 + a))
            L.append("  }")
    L.append("  const double dp = (sx + sy - rp) * F.inv_sigma;")
    for kind in ("EE", "EO", "OE", "OO"):
        L += emit(kind)
    L.append("  // Schur correction: cpy = s(cpx)")
    L.append("  const double ndp = -dp;")
    for a in range(3):
        for b in range(2):
            L.append("  {")
            L.append("    const double k = F.cpx[%d];" % (a * 2 + b))
            L.append("    vx[%d] = fma(k, ndp, vx[%d]);" % (a * 5 + 3 + b, a * 5 + 3 + b))
            L.append("    vy[%d] = fma(k, ndp, vy[%d]);" % ((3 + b) * 5 + a, (3 + b) * 5 + a))
            L.append("  }")
    L.append("  inv_transform(vx);")
    L.append("  inv_transform(vy);")
    L.append("  return dp;")
    L.append("}")
    L.append("")
    L.append("}  // namespace svk")
    open(OUT, "w").write("\n".join(L) + "\n")
    S = ["// stencil_gen.cuh -- GENERATED by tools/gen_solve.py; do not edit.",
         "// Residual stencils with shared coefficients (DESIGN.md section 7).",
         "#pragma once", "", "namespace svk {", ""]
    S += stencil_code()
    S += ["", "}  // namespace svk"]
    open(OUT_ST, "w").write("\n".join(S) + "\n")
    print(OUT, OUT_ST)


if __name__ == "__main__":
    import sys
    main(sys.argv[1] if len(sys.argv) > 1 else CSRC)
