"""The C-ABI library loads without a GPU and exports every symbol the header declares."""

import os
import re

import pytest

from paper_2509_18521_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "april_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ab_\w+)\s*\(", src, re.M)))


def test_header_declarations_are_bound():
    decl = _declared()
    assert len(decl) >= 20
    assert sorted(decl) == sorted(_capi.EXPORTS)


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_capi.LIB_PATH):
        pytest.skip("library not built")
    lib = _capi.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.ab_version() == 1


def test_struct_sizes_match_header_layout():
    import ctypes as C
    assert C.sizeof(_capi.SampleDesc) == 32
    assert C.sizeof(_capi.Event) == 32
    assert C.sizeof(_capi.Admit) == 16
    assert C.sizeof(_capi.RunArgs) == 48
