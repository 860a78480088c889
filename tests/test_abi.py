"""The C ABI library loads and exports every entry point include/elastik_b200.h
declares (no compute calls: this runs on CPU-only machines too)."""

import ctypes
import os
import re

import pytest

from conftest import REPO
from paper_2102_05221_b200 import _lib

HEADER = os.path.join(REPO, "include", "elastik_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ek_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ("ek_distance_batch", "ek_nn", "ek_nn_dev", "ek_pairwise", "ek_subseq", "ek_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.fail("libelastik_b200.so not built (run __graft_entry__.build())")
    L = ctypes.CDLL(_lib.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert set(_lib.EXPORTS) <= set(declared_symbols())


def test_version_and_error_strings_without_gpu():
    L = _lib.lib()
    assert b"sm_100a" in L.ek_version()
    assert isinstance(L.ek_last_error(), bytes)
    assert L.ek_device_count() >= 0
