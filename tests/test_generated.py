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


def test_block_solve_covers_every_block_entry():
    # every (row, column) pair of each parity block appears exactly once per component
    src = open(os.path.join(CSRC, "solve_gen.cuh")).read()
    pairs = re.findall(r"sx(\d+) = fma\(k, vx\[(\d+)\], sx\d+\)", src)
    seen = {}
    for r, c in pairs:
        seen[(int(r), int(c))] = seen.get((int(r), int(c)), 0) + 1
    par = lambda i: i < 3
    expect = {(r, c) for r in range(25) for c in range(25)
              if par(r // 5) == par(c // 5) and par(r % 5) == par(c % 5)}
    assert set(seen) == expect and all(v == 1 for v in seen.values())
    assert len(expect) == 81 + 36 + 36 + 16


def test_stencil_covers_every_tap():
    src = open(os.path.join(CSRC, "stencil_gen.cuh")).read()
    body = src[src.index("stencil_L_sym"):src.index("stencil_B_sym")]
    taps = re.findall(r"ax\[(\d)\] = fma\(k, U\[(\d)\]\[(\d)\]", body)
    per = {}
    for o, r, c in taps:
        per.setdefault(int(o), set()).add((int(r), int(c)))
    # odd row / even col 3x5, odd/odd 3x3, even/even 5x5, even row / odd col 5x3 taps
    assert [len(per[o]) for o in range(4)] == [15, 9, 25, 15]
