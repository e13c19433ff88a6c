"""The C-ABI library loads here (no GPU) and exports every symbol the header declares."""

import ctypes
import os
import re

import pytest

from conftest import REPO
from paper_1704_04139_b200 import _native
from paper_1704_04139_b200.errors import NativeError

HEADER = os.path.join(REPO, "include", "halfcell_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hc_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ("hc_operator_create", "hc_apply", "hc_jvp", "hc_newton_solve", "hc_step",
              "hc_step_host", "hc_solve_initial_potential", "hc_pod_gram"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = _native.load_library()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(_native.EXPORTED)


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(NativeError):
        _native.require_device()


def test_error_mapping():
    lib = _native.load_library()
    info = _native.HcInfo()
    # a null operator handle is an argument error surfaced through hc_last_error
    n = ctypes.c_int(-1)
    assert lib.hc_device_count(ctypes.byref(n)) == 0
