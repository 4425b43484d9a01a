"""The C-ABI library loads without a GPU and exports every symbol include/cw.h declares."""

import ctypes
import os
import re

from paper_2006_02464_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "cw.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cw_[a-z_0-9]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n


def test_binding_covers_header():
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == declared_functions()


def test_abi_version_and_struct_sizes():
    assert _lib.lib.cw_abi_version() == 2
    assert ctypes.sizeof(_lib.cw_op) == 24 * 4
    assert ctypes.sizeof(_lib.cw_tensor_loc) == 32
    assert ctypes.sizeof(_lib.cw_action) == 8 + 4 * 4 + 3 * 8 + 16 * 8
