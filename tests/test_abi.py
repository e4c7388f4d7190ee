"""The C-ABI library: loads on a CPU-only host and exports every symbol
include/cltk_b200.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

from conftest import ROOT

import paper_2108_03076_b200 as E
from paper_2108_03076_b200 import _native


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "cltk_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cltk_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_native.EXPORTS) == syms


def test_version_and_closed_form():
    assert "sm_100a" in E.version()
    # proj/python/tests/test_smoke.py:50-51
    bs = E.black_scholes_call(100.0, 100.0, 0.05, 0.2, 90.0 / 365.0)
    assert abs(bs - 4.579032085233791) <= 1e-12 * bs


def test_library_is_sm100a():
    data = open(_native.LIB_PATH, "rb").read()
    assert b"sm_100a" in data
