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


@pytest.mark.parametrize("cname,pyname", [("svk_config", "Config"), ("svk_level", "LevelInfo"),
                                          ("svk_report", "Report")])
def test_struct_layouts_match_header(cname, pyname, tmp_path):
    """The ctypes structures of the binding have the header's field offsets and size
    (a C program built against include/svk.h prints offsetof of every field)."""
    import ctypes as C
    from paper_2401_06277_b200 import svk
    py = getattr(svk, pyname)
    fields = [f for f, _ in py._fields_]
    prog = tmp_path / "layout.c"
    prog.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"svk.h\"\nint main(void) {\n"
                    + "".join('  printf("%%s %%zu\\n", "%s", offsetof(%s, %s));\n' % (f, cname, f) for f in fields)
                    + '  printf("sizeof %%zu\\n", sizeof(%s));\n  return 0;\n}\n' % cname)
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)], check=True)
    out = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True, text=True,
                                                        check=True).stdout.splitlines())
    for f in fields:
        assert int(out[f]) == getattr(py, f).offset, f
    assert int(out["sizeof"]) == C.sizeof(py)


def test_allocator_callbacks_both_or_neither(lib_path):
    import ctypes as C
    from paper_2401_06277_b200 import svk
    lib = svk.load_library(lib_path)
    alloc, free = svk.ALLOC_FN(lambda n, d, u: None), svk.FREE_FN(lambda p, n, d, u: None)
    h = C.c_void_p()
    for a, f in ((alloc, None), (None, free)):
        c = svk.Config()
        lib.svk_config_default(C.byref(c), 64)
        c.alloc_fn = C.cast(a, C.c_void_p) if a else None
        c.free_fn = C.cast(f, C.c_void_p) if f else None
        assert lib.svk_create(C.byref(c), C.byref(h)) == -1   # rejected before touching the GPU
