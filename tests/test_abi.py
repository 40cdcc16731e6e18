"""C-ABI library checks that need no GPU: it loads, and it exports every symbol
include/wf4dvar.h declares (no compute call is made here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "wf4dvar.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(wf4dvar_[a-z_A-Z0-9]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for need in ("wf4dvar_create", "wf4dvar_apply_A", "wf4dvar_apply_P", "wf4dvar_solve",
                 "wf4dvar_destroy", "wf4dvar_set_precond", "wf4dvar_local_windows",
                 "wf4dvar_vector_len", "wf4dvar_last_error"):
        assert need in syms


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2105_06975_b200 import _lib as L
    lib = ctypes.CDLL(L.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(L.EXPORTED)
    assert "sm_100a" in L.version()


def test_library_is_sm100a_code():
    from paper_2105_06975_b200 import _lib as L
    out = subprocess.run(["cuobjdump", "--list-elf", L.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_product_path_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2105_06975_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
