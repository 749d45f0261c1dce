"""The C-ABI library loads without a GPU and exports every symbol the header declares."""

import ctypes
import os
import re

from paper_2004_03054_b200 import _native

HERE = os.path.dirname(os.path.abspath(__file__))
HEADER = os.path.join(os.path.dirname(HERE), "include", "luda_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(luda_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header_symbols():
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_declares_every_header_symbol():
    assert sorted(_native.EXPORTED) == header_symbols()


def test_load_without_gpu():
    L = _native.load()
    assert L.luda_abi_version() == 2
