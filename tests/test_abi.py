"""CPU-only checks of the C-ABI library: it builds, loads, exports every symbol that
include/vr.h declares, and rejects bad arguments before touching a device."""
from __future__ import annotations

import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_2502_05063_b200 as vr
from paper_2502_05063_b200 import build as vrbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    txt = open(os.path.join(ROOT, "include", "vr.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(vr_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    vrbuild.build()
    return vr.load()


def test_every_declared_symbol_is_exported(lib):
    names = _declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name


def test_binary_is_sm100a(lib):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {vr.lib_path}").read()
    assert "sm_100a" in out


@pytest.mark.parametrize("n,max_dim,thr,code", [
    (0, 1, math.inf, vr.VR_EINVAL),
    (4, -1, math.inf, vr.VR_EINVAL),
    (4, 99, math.inf, vr.VR_EINVAL),
    (4, 1, float("nan"), vr.VR_EINVAL),
    (4, 1, -1.0, vr.VR_EINVAL),
    (70000, 1, math.inf, vr.VR_ECAPACITY),
])
def test_argument_errors_before_any_device_work(lib, n, max_dim, thr, code):
    lt = np.ones(6, np.float32)
    h = ctypes.c_void_p(1234)
    rc = lib.vr_barcodes(lt.ctypes.data, n, max_dim, thr, None, ctypes.byref(h))
    assert rc == code
    assert h.value is None  # *out = NULL on error
    assert len(lib.vr_last_error()) > 0


def test_capacity_error_for_huge_index_space(lib):
    # C(65535, 8) > 2^63: indices of the cofacets would not fit
    h = ctypes.c_void_p()
    rc = lib.vr_barcodes(ctypes.c_void_p(8), 65535, 6, math.inf, None, ctypes.byref(h))
    assert rc == vr.VR_ECAPACITY


def test_null_pointer_rejected(lib):
    h = ctypes.c_void_p()
    assert lib.vr_barcodes(None, 5, 1, math.inf, None, ctypes.byref(h)) == vr.VR_EINVAL
    assert lib.vr_barcodes(np.ones(10, np.float32).ctypes.data, 5, 1, math.inf, None, None) == vr.VR_EINVAL


def test_accessors_tolerate_null(lib):
    assert lib.vr_max_dim(None) == -1
    assert lib.vr_num_pairs(None, 0) == 0
    assert lib.vr_pairs(None, 0) is None
    lib.vr_free(None)
    lib.vr_plan_free(None)


def test_no_cpu_fallback_in_product_package():
    # the product package never imports the oracle
    pkg = os.path.join(ROOT, "paper_2502_05063_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.lower().replace("oracle-", ""), f
