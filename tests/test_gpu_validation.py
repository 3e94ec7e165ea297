"""Validation mode ("only 25 different patch matrices",
S:391): every patch rebuilt and inverted on its own must equal its group's
stored inverse, and the generic reflection-basis factors must reproduce the
generic group's inverse, to 1e-12; a deliberately corrupted group must fail."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_validation_passes_on_every_level(gpu):
    from paper_2401_06277_b200 import Solver
    S = Solver(64, validate=True)          # svk_create validates every level
    for l in range(S.levels):
        dev, n = S.validate_patches(l)
        N = S.info[l].N
        assert n == (N + 1) ** 2
        assert dev <= 1e-12, (l, dev)


SCRIPT = r"""
import sys
from paper_2401_06277_b200 import Solver, SvkError
try:
    Solver(64, validate=True)
    print("CREATE-OK")
except SvkError as e:
    print("CREATE-FAIL", e)
S = Solver(64)
try:
    print("VALIDATE-OK", S.validate_patches(S.fine))
except SvkError as e:
    print("VALIDATE-FAIL", e)
"""


@pytest.mark.parametrize("group", [7, 12])  # a boundary group (cat 2,1) and the generic group (2,2)
def test_corrupted_group_is_caught(gpu, group):
    slot = 12 * 51 + 12  # u_x at the patch's own node, present in every group
    env = dict(os.environ, PYTHONPATH=ROOT, SVK_TEST_CORRUPT_GROUP="4,%d,%d" % (group, slot))
    out = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "CREATE-FAIL" in out.stdout and "validation" in out.stdout, out.stdout
    assert "VALIDATE-FAIL" in out.stdout, out.stdout
