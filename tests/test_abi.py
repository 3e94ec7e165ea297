"""CPU-side checks of the C-ABI boundary: libsvk.so builds for sm_100a, loads,
and exports every function include/svk.h declares (no compute without a GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "svk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*(?:const\s+)?[\w]+\*?\s+\*?(svk_\w+)\s*\(", src, flags=re.M))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2401_06277_b200 import build
    return build.build()


def test_header_parses():
    fns = header_functions()
    assert {"svk_create", "svk_vanka_sweep", "svk_fgmres", "svk_vcycle", "svk_residual"} <= fns


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (svk_\w+)", out))
    missing = header_functions() - exported
    assert not missing, missing


def test_binding_covers_header_and_loads(lib_path):
    from paper_2401_06277_b200 import svk
    assert set(svk.EXPORTS) == header_functions()
    lib = svk.load_library(lib_path)
    assert lib.svk_status_string(-4) == b"singular factorisation"
    assert lib.svk_last_error(None) == b"null context"


def test_library_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_config_defaults_and_invalid_configs(lib_path):
    import ctypes as C
    from paper_2401_06277_b200 import svk
    lib = svk.load_library(lib_path)
    cfg = svk.Config()
    assert lib.svk_config_default(C.byref(cfg), 64) == 0
    assert (cfg.n_elem, cfg.n_coarse, cfg.nu, cfg.omega_v, cfg.nu_pre, cfg.nu_post) == (64, 4, 1.0, 0.8, 1, 1)
    h = C.c_void_p()
    for bad in (dict(n_elem=48, n_coarse=4), dict(n_elem=2, n_coarse=2), dict(n_elem=64, n_coarse=3)):
        c = svk.Config()
        lib.svk_config_default(C.byref(c), bad["n_elem"])
        c.n_coarse = bad["n_coarse"]
        assert lib.svk_create(C.byref(c), C.byref(h)) == -1   # rejected before touching the GPU
    assert lib.svk_destroy(None) == -1
