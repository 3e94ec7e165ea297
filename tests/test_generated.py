"""The generated kernel headers (csrc/solve_gen.cuh, csrc/stencil_gen.cuh) are what
tools/gen_solve.py produces, and the generated code covers every FMA of the forms
it replaces: each orbit of equal coefficients is applied at every member position."""
import importlib.util
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2401_06277_b200", "csrc")


def _gen():
    spec = importlib.util.spec_from_file_location("gen_solve", os.path.join(ROOT, "tools", "gen_solve.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_generated_headers_are_current(tmp_path):
    _gen().main(str(tmp_path))
    for name in ("solve_gen.cuh", "stencil_gen.cuh"):
        assert open(os.path.join(CSRC, name)).read() == open(os.path.join(tmp_path, name)).read(), name


def test_stencil_covers_every_tap():
    src = open(os.path.join(CSRC, "stencil_gen.cuh")).read()
    body = src[src.index("stencil_L_sym"):src.index("stencil_B_sym")]
    taps = re.findall(r"ax\[(\d)\] = fma\(k, U\[(\d)\]\[(\d)\]", body)
    per = {}
    for o, r, c in taps:
        per.setdefault(int(o), set()).add((int(r), int(c)))
    # odd row / even col 3x5, odd/odd 3x3, even/even 5x5, even row / odd col 5x3 taps
    assert [len(per[o]) for o in range(4)] == [15, 9, 25, 15]


def _solve_fn():
    """solve_generic_sym (csrc/solve_gen.cuh) translated statement by statement into
    Python: each generated line is a declaration, an fma or an assignment."""
    src = open(os.path.join(CSRC, "solve_gen.cuh")).read()
    body = src[src.index("solve_generic_sym"):]
    body = body[body.index("{") + 1:body.index("\n}\n")]
    out = []
    for line in body.split("\n"):
        line = line.split("//")[0].strip().rstrip(";")
        if line in ("", "{", "}"):
            continue
        m = re.match(r"(fwd|inv)_transform\((v[xy])\)$", line)
        if m:
            out.append("%s = _%s(%s)" % (m.group(2), m.group(1), m.group(2)))
            continue
        if line.startswith("return"):
            out.append(line)
            continue
        line = re.sub(r"^(const )?double ", "", line)
        for stmt in re.split(r", (?=[a-z]+\d* = )", line):
            out.append(stmt.replace("fma(", "_fma("))
    code = "def solve(vx, vy, rp, F):\n" + "\n".join("    " + s for s in out) + "\n"
    ns = {"_fma": lambda a, b, c: a * b + c}

    def split5(v, o, st):
        a, b, c, d, e = (v[o + i * st] for i in range(5))
        v[o], v[o + st], v[o + 2 * st], v[o + 3 * st], v[o + 4 * st] = a + e, b + d, c, a - e, b - d

    def unsplit5(v, o, st):
        e0, e1, e2, d0, d1 = (v[o + i * st] for i in range(5))
        v[o], v[o + st], v[o + 2 * st], v[o + 3 * st], v[o + 4 * st] = e0 + d0, e1 + d1, e2, e1 - d1, e0 - d0

    def fwd(v):  # SVK_SPLIT5 rows then columns (sweep_fused.cuh fwd_transform), in place
        for r in range(5):
            split5(v, r * 5, 1)
        for c in range(5):
            split5(v, c, 5)
        return v

    def inv(v):  # SVK_UNSPLIT5 columns then rows (inv_transform), in place
        for c in range(5):
            unsplit5(v, c, 5)
        for r in range(5):
            unsplit5(v, r * 5, 1)
        return v

    ns["_fwd"], ns["_inv"] = fwd, inv
    exec(code, ns)
    return ns["solve"]


def _factors(Lw, bx, by):
    """The FusedFactors fields solve_generic_sym reads, by their definitions in
    sweep_fused.cuh (k_factor_setup): B = S T Lw^-1 T^-1 per parity block, chat =
    T^-T c, cp = S T c."""
    import types

    import numpy as np
    T5 = np.array([[1, 0, 0, 0, 1], [0, 1, 0, 1, 0], [0, 0, 1, 0, 0], [1, 0, 0, 0, -1], [0, 1, 0, -1, 0]], float)
    S5 = np.array([.5, .5, 1, .5, .5])
    T, Ti, S = np.kron(T5, T5), np.linalg.inv(np.kron(T5, T5)), np.kron(S5, S5)
    Li = np.linalg.inv(Lw)
    B = S[:, None] * (T @ Li @ Ti)
    cx, cy = Li @ bx, Li @ by
    F = types.SimpleNamespace()
    ee = [ty * 5 + tx for ty in range(3) for tx in range(3)]
    eo = [ty * 5 + tx for ty in range(3) for tx in (3, 4)]
    oe = [ty * 5 + tx for ty in (3, 4) for tx in range(3)]
    oo = [ty * 5 + tx for ty in (3, 4) for tx in (3, 4)]
    F.bee, F.beo, F.boe, F.boo = (B[np.ix_(p, p)] for p in (ee, eo, oe, oo))
    F.chx, F.chy = (Ti.T @ cx)[eo], (Ti.T @ cy)[oe]
    F.cpx, F.cpy = (S * (T @ cx))[eo], (S * (T @ cy))[oe]
    F.inv_sigma = 1.0 / (bx @ cx + by @ cy)
    return F


def test_generated_solve_is_the_dense_patch_solve():
    # The generated straight-line solve (orbit-shared parity blocks, Schur rank-1
    # correction) applied to a random generic-patch residual equals the
    # dense solve of [[Lw, 0, bx], [0, Lw, by], [bx^T, by^T, 0]] (the 51x51 generic
    # patch matrix) for a D4-invariant Lw = M (x) K + K (x) M and b_y = s(b_x).
    import numpy as np
    rng = np.random.default_rng(7)
    J = np.eye(5)[::-1]

    def refl_spd():
        a = rng.standard_normal((5, 5))
        a = a @ a.T + 5 * np.eye(5)
        return 0.5 * (a + J @ a @ J)  # symmetric under reflection, SPD

    M, K = refl_spd(), refl_spd()
    Lw = np.kron(M, K) + np.kron(K, M)
    g = rng.standard_normal((5, 5))
    g = 0.5 * (g + g[::-1, :])          # even in y (rows)
    g = 0.5 * (g - g[:, ::-1])          # odd in x (columns)
    bx, by = g.reshape(25), g.T.reshape(25)
    F = _factors(Lw, bx, by)
    solve = _solve_fn()
    A = np.zeros((51, 51))
    A[:25, :25] = A[25:50, 25:50] = Lw
    A[:25, 50] = A[50, :25] = bx
    A[25:50, 50] = A[50, 25:50] = by
    for trial in range(3):
        r = rng.standard_normal(51)
        vx, vy = list(r[:25]), list(r[25:50])
        dp = solve(vx, vy, r[50], F)
        want = np.linalg.solve(A, r)
        got = np.concatenate([vx, vy, [dp]])
        assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want)), np.max(np.abs(got - want))


def test_generated_solve_fma_count():
    # parity blocks 9^2 + 6^2 + 6^2 + 4^2 = 169 FMAs per velocity component, plus the
    # 6 + 6 Schur FMAs per component
    src = open(os.path.join(CSRC, "solve_gen.cuh")).read()
    assert src.count("fma(") == 2 * 169 + 24
