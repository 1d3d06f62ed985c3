"""The C ABI library loads without a GPU, exports every symbol the header
declares, and rejects bad descriptors before touching the device."""

import ctypes
import os
import re

import pytest

from conftest import ROOT


def _declared():
    with open(os.path.join(ROOT, "include", "tsunami_b200.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(ts_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2408_07609_b200 import _native
    lib = _native.lib()
    names = _declared()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    assert set(_native.EXPORTED) == set(names)


def test_abi_version_and_invalid_descriptor():
    from paper_2408_07609_b200 import _native as N
    lib = N.lib()
    assert lib.ts_abi_version() == N.ABI_VERSION
    h = ctypes.c_void_p()
    assert lib.ts_create(None, ctypes.byref(h)) == N.TS_ERR_INVALID
    d = N.Desc()
    d.abi_version = 999
    assert lib.ts_create(ctypes.byref(d), ctypes.byref(h)) == N.TS_ERR_INVALID
    assert b"ABI version" in lib.ts_last_error()
    d.abi_version = N.ABI_VERSION
    d.n_blocks = 0
    assert lib.ts_create(ctypes.byref(d), ctypes.byref(h)) == N.TS_ERR_INVALID
    assert not h.value


def test_no_oracle_in_product():
    """The product never imports or links the oracle (it is test-only)."""
    pkg = os.path.join(ROOT, "paper_2408_07609_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                with open(os.path.join(dirpath, fn)) as f:
                    src = f.read()
                assert not re.search(r"^\s*(import|from)\s+oracle", src, re.M), fn
                assert not re.search(r'#include\s*["<][^">]*oracle', src), fn
