"""The C-ABI library loads and exports every symbol include/petals_b200.h
declares (CPU-only: no compute calls)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "petals_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pb_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_listed_in_binding():
    from paper_2209_01188_b200 import _lib

    assert sorted(_lib.EXPORTS) == header_symbols()


def test_library_exports_every_symbol():
    from paper_2209_01188_b200 import _lib, build

    if not os.path.exists(_lib.LIB_PATH):
        build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in header_symbols():
        assert hasattr(lib, name), name
    lib.pb_version.restype = ctypes.c_int
    assert lib.pb_version() == 1


def test_binding_signatures_load():
    from paper_2209_01188_b200 import _lib, build

    if not os.path.exists(_lib.LIB_PATH):
        build.build()
    L = _lib.lib()
    assert L.pb_last_error() is not None


def test_error_code_mapping():
    from paper_2209_01188_b200 import errors

    with pytest.raises(errors.InputError):
        errors.raise_for(errors.ERR_BAD_REQUEST, "x")
    with pytest.raises(errors.CapacityError):
        errors.raise_for(errors.ERR_CAPACITY, "x")
    with pytest.raises(errors.RemoteError) as ei:
        errors.raise_for(errors.ERR_BUSY, "x")
    assert ei.value.code == errors.ERR_BUSY
