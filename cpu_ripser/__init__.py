"""ctypes wrapper of the single-threaded Ripser-style CPU run (cpu_ripser/ripser_style.cpp).

BASELINE ONLY: BASELINE.json's north_star asks for "a single-threaded Ripser-style CPU run
timed on the box's own host cores" next to the GPU numbers.  bench.py times it, tests/
check it against the oracle; the product package never imports it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ripser_style.cpp")
_LIB = os.path.join(_HERE, "libripser_style.so")
_lib = None


def build(force: bool = False) -> str:
    """g++ -O3, single thread, no -march (the .so travels to the GPU box's host)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O3", "-std=c++17", "-Wall", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.rs_barcode.restype = ctypes.c_void_p
        lib.rs_barcode.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float]
        lib.rs_num_pairs.restype = ctypes.c_int64
        lib.rs_num_pairs.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.rs_get_pairs.restype = None
        lib.rs_get_pairs.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        lib.rs_stats.restype = None
        lib.rs_stats.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
        lib.rs_free.restype = None
        lib.rs_free.argtypes = [ctypes.c_void_p]
        _lib = lib
    return _lib


def barcode(lt: np.ndarray, n: int, max_dim: int, threshold: float):
    """-> (pairs, stats): pairs[d] = float32 (k, 2) array of (birth, death), birth < death,
    sorted; stats[d] = {columns, emergent, reduced, simplices, ms}."""
    lib = _load()
    lt = np.ascontiguousarray(lt, np.float32)
    h = lib.rs_barcode(lt.ctypes.data, int(n), int(max_dim), float(threshold))
    if not h:
        raise RuntimeError("ripser_style: bad arguments or out of memory")
    try:
        pairs, stats = [], []
        for d in range(max_dim + 1):
            k = lib.rs_num_pairs(h, d)
            b = np.empty(k, np.float32)
            e = np.empty(k, np.float32)
            lib.rs_get_pairs(h, d, b.ctypes.data, e.ctypes.data)
            arr = np.stack([b, e], 1) if k else np.zeros((0, 2), np.float32)
            if k:
                arr = arr[np.lexsort((arr[:, 1], arr[:, 0]))]
            pairs.append(arr)
            c = np.zeros(5, np.float64)
            lib.rs_stats(h, d, c.ctypes.data)
            stats.append({"columns": int(c[0]), "emergent": int(c[1]), "reduced": int(c[2]),
                          "simplices": int(c[3]), "ms": float(c[4])})
        return pairs, stats
    finally:
        lib.rs_free(h)
