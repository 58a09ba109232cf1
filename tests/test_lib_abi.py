"""CPU checks of the C-ABI library: it builds for sm_100a, loads, and exports
every function include/lfem.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2605_14035_b200 import build
    return build.build()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "lfem.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lfem_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("lfem_mesh_create", "lfem_assemble_symbolic", "lfem_assemble_numeric", "lfem_csr_get"):
        assert required in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_names_match_header():
    from paper_2605_14035_b200 import lfem
    assert set(lfem.EXPORTED) == set(declared_functions())
    for n in declared_functions():
        if n not in ("lfem_mesh_destroy", "lfem_plan_destroy", "lfem_error_element", "lfem_last_error"):
            assert hasattr(lfem, n), n


def test_sass_is_sm100a(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2605_14035_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "lfem_oracle" not in txt, f


def test_version_without_gpu(libpath):
    lib = ctypes.CDLL(libpath)
    lib.lfem_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.lfem_version()


def test_allocator_hook_argument_check_without_gpu(libpath):
    """lfem_set_allocator: both callbacks or neither (no device call involved)."""
    lib = ctypes.CDLL(libpath)
    lib.lfem_set_allocator.argtypes = [ctypes.c_void_p] * 3
    ALLOC = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
    a = ALLOC(lambda n, s, c: None)
    assert lib.lfem_set_allocator(ctypes.cast(a, ctypes.c_void_p), None, None) == 1  # INVALID_ARG
    assert lib.lfem_set_allocator(None, None, None) == 0


def header_enums():
    """NAME = value pairs of the enums in include/lfem.h."""
    src = open(os.path.join(ROOT, "include", "lfem.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return {k: int(v.rstrip("u")) for k, v in re.findall(r"\b(LFEM_[A-Z0-9_]+)\s*=\s*([0-9]+u?)", src)}


def test_binding_constants_match_the_header():
    """The Python binding's and the input generators' constants are the header's enums."""
    import lfem_inputs as li
    from paper_2605_14035_b200 import lfem
    e = header_enums()
    for name in ("LFEM_MASS", "LFEM_STIFF", "LFEM_STIFF_COEF", "LFEM_NUMERIC_AUTO", "LFEM_NUMERIC_V0",
                 "LFEM_NUMERIC_TILED", "LFEM_NUMERIC_ROWS", "LFEM_RHS_LOAD", "LFEM_RHS_KLL"):
        assert getattr(lfem, name) == e[name], name
    pairs = {"SURFACE_TRI": "LFEM_SURFACE_TRI", "BULK_TET": "LFEM_BULK_TET", "SURFACE_LINE": "LFEM_SURFACE_LINE",
             "QUAD_DEFAULT": "LFEM_QUAD_DEFAULT", "QUAD_TRI3_DEG2": "LFEM_QUAD_TRI3_DEG2",
             "QUAD_TRI6_DEG4": "LFEM_QUAD_TRI6_DEG4", "QUAD_TET4_DEG2": "LFEM_QUAD_TET4_DEG2",
             "QUAD_TET11_DEG4": "LFEM_QUAD_TET11_DEG4", "QUAD_TRI16_DEG8": "LFEM_QUAD_TRI16_DEG8",
             "QUAD_LINE2_DEG3": "LFEM_QUAD_LINE2_DEG3", "QUAD_LINE3_DEG5": "LFEM_QUAD_LINE3_DEG5"}
    for py, h in pairs.items():
        assert getattr(li, py) == e[h], (py, h)
