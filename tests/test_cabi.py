"""The C-ABI library loads, exports every symbol include/cgl_b200.h
declares, and validates arguments before touching a device (CPU-safe)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import REPO


def header_symbols():
    txt = open(os.path.join(REPO, "include", "cgl_b200.h")).read()
    return sorted(set(re.findall(r"\b(cgl_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_2403_02816_b200 import _lib
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)


def test_nm_dynamic_exports():
    from paper_2403_02816_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.lib_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (cgl_\w+)", out))
    assert set(header_symbols()) <= exported


def test_library_is_sm100a():
    from paper_2403_02816_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_abi():
    from paper_2403_02816_b200 import _lib
    lib = _lib.load()
    assert lib.cgl_abi_version() == 2
    assert b"sm_100a" in lib.cgl_version()


def test_shape_validation_without_device():
    from paper_2403_02816_b200 import _lib
    lib = _lib.load()
    shape = _lib.i64_array([4, 5])
    rc = lib.cgl_mode_product(None, 2, shape, 2, None, None, 4, None, None, 1.0, None, 0.0, None, 0)
    assert rc == -2
    assert b"axis" in lib.cgl_last_error()
    rc = lib.cgl_zgemm(None, -1, 2, 2, None, 2, 0, None, 2, 0, None, 2, 0, 1, 1.0, 0.0, None, 0, 0, 0.0, None, 0)
    assert rc == -2
    rc = lib.cgl_lincomb(None, 10, 7, _lib.dbl_array([1.0] * 7), None, None, None, 0)
    assert rc == -1
    rc = lib.cgl_tucker(None, 2, shape, 9, None, None, None, None, None, None, 0)
    assert rc == -1


def test_c_header_compiles_standalone(tmp_path):
    src = tmp_path / "t.c"
    src.write_text('#include "cgl_b200.h"\nint main(void){return cgl_abi_version()==CGL_ABI_VERSION?0:1;}\n')
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-c", str(src), "-I", os.path.join(REPO, "include"),
                        "-o", str(tmp_path / "t.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
