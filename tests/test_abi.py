"""The C-ABI library loads and exports every entry point include/auras_b200.h declares."""

import ctypes
import os
import re

from paper_2509_09560_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "auras_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(auras_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load(require_device=False)
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.exported_symbols())
    assert lib.auras_abi_version() == _lib.ABI_VERSION


def test_struct_layouts_are_stable():
    # auras_conv_op: 9 pointers + 25 int32 + reserved[3] -> 72 + 112 = 184 bytes
    assert ctypes.sizeof(_lib.ConvOp) == 9 * 8 + 28 * 4
    assert ctypes.sizeof(_lib.LinearOp) == 2 * 8 + 4 * 4
    assert ctypes.sizeof(_lib.Sched) == 7 * 8 + 4 * 4
