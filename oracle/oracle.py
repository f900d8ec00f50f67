"""ctypes wrapper of the C oracle (oracle/vr_oracle.c) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and --impl
reference) may import this module.  The product package never imports it.

The oracle computes the persistence barcode by the textbook route (explicit boundary
matrix + Alg 2), see the header of vr_oracle.c for the
step-by-step citations.  Pins: tests/test_oracle_pins.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "vr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (single thread, -O2).  Idempotent."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        lib.oracle_barcode.restype = ctypes.c_void_p
        lib.oracle_barcode.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float,
                                       ctypes.POINTER(ctypes.c_int)]
        lib.oracle_num_pairs.restype = ctypes.c_int64
        lib.oracle_num_pairs.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.oracle_num_simplices.restype = ctypes.c_int64
        lib.oracle_num_simplices.argtypes = [ctypes.c_void_p, ctypes.c_int]
        lib.oracle_get_pairs.restype = None
        lib.oracle_get_pairs.argtypes = [ctypes.c_void_p, ctypes.c_int] + [ctypes.c_void_p] * 4
        lib.oracle_free.restype = None
        lib.oracle_free.argtypes = [ctypes.c_void_p]
        lib.oracle_apparent.restype = ctypes.c_int64
        lib.oracle_apparent.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_reduce_columns.restype = ctypes.c_int
        lib.oracle_reduce_columns.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_apparent_one.restype = ctypes.c_int
        lib.oracle_apparent_one.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_float, ctypes.c_void_p,
                                            ctypes.c_void_p]
        lib.oracle_enclosing_radius.restype = ctypes.c_float
        lib.oracle_enclosing_radius.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        _lib = lib
    return _lib


@dataclass
class DimPairs:
    birth: np.ndarray          # float32
    death: np.ndarray          # float32 (+inf = essential)
    birth_cidx: np.ndarray     # uint64 name of the birth simplex (dim p)
    death_cidx: np.ndarray     # uint64 name of the death simplex (dim p+1); 2^64-1 = essential


@dataclass
class OracleBarcode:
    max_dim: int
    dims: list = field(default_factory=list)       # DimPairs per dimension 0..max_dim
    n_simplices: list = field(default_factory=list)  # n_p for p = 0..max_dim+1

    def positive(self, dim: int) -> np.ndarray:
        """(birth, death) float32 pairs with birth < death, sorted — the reported barcode."""
        p = self.dims[dim]
        keep = p.birth < p.death
        arr = np.stack([p.birth[keep], p.death[keep]], 1) if keep.any() else np.zeros((0, 2), np.float32)
        order = np.lexsort((arr[:, 1], arr[:, 0])) if len(arr) else np.zeros(0, np.int64)
        return arr[order].astype(np.float32)

    def index_pairs(self, dim: int) -> set:
        p = self.dims[dim]
        return set(zip(p.birth_cidx.tolist(), p.death_cidx.tolist()))

    def num_pairs_all(self, dim: int) -> int:
        """P_dim: finite pairs incl. zero-length."""
        p = self.dims[dim]
        return int(np.isfinite(p.death).sum())

    def num_essential(self, dim: int) -> int:
        return int((~np.isfinite(self.dims[dim].death)).sum())


def barcode(lower_tri: np.ndarray, n: int, max_dim: int, threshold: float = float("inf")) -> OracleBarcode:
    lib = _load()
    lt = np.ascontiguousarray(lower_tri, dtype=np.float32)
    assert lt.size == n * (n - 1) // 2
    err = ctypes.c_int(0)
    h = lib.oracle_barcode(lt.ctypes.data if lt.size else None, n, max_dim, ctypes.c_float(threshold), ctypes.byref(err))
    if not h:
        raise ValueError(f"oracle_barcode failed with code {err.value}")
    try:
        out = OracleBarcode(max_dim)
        for d in range(max_dim + 1):
            m = lib.oracle_num_pairs(h, d)
            b = np.empty(m, np.float32); de = np.empty(m, np.float32)
            bc = np.empty(m, np.uint64); dc = np.empty(m, np.uint64)
            if m:
                lib.oracle_get_pairs(h, d, b.ctypes.data, de.ctypes.data, bc.ctypes.data, dc.ctypes.data)
            out.dims.append(DimPairs(b, de, bc, dc))
        out.n_simplices = [int(lib.oracle_num_simplices(h, d)) for d in range(max_dim + 2)]
        return out
    finally:
        lib.oracle_free(h)


def apparent(lower_tri: np.ndarray, n: int, d: int, threshold: float = float("inf")):
    """Def 5.3.4 on explicit sets: (cidx[], is_apparent[], partner_cidx[]) over all
    d-simplices with diam <= threshold, in cidx order."""
    lib = _load()
    lt = np.ascontiguousarray(lower_tri, dtype=np.float32)
    m = lib.oracle_apparent(lt.ctypes.data if lt.size else None, n, d, ctypes.c_float(threshold), None, None, None)
    c = np.empty(m, np.uint64); f = np.empty(m, np.int8); p = np.empty(m, np.uint64)
    if m:
        lib.oracle_apparent(lt.ctypes.data, n, d, ctypes.c_float(threshold), c.ctypes.data, f.ctypes.data, p.ctypes.data)
    return c, f.astype(bool), p


def apparent_one(lower_tri: np.ndarray, n: int, vertices, threshold: float = float("inf")):
    """Def 5.3.4 for one simplex by brute force: (is_apparent, partner_cidx or None);
    None if the simplex is over the threshold."""
    lt = np.ascontiguousarray(lower_tri, dtype=np.float32)
    v = np.ascontiguousarray(vertices, dtype=np.int32)
    p = ctypes.c_uint64(0)
    r = _load().oracle_apparent_one(lt.ctypes.data, n, v.size - 1, ctypes.c_float(threshold), v.ctypes.data, ctypes.byref(p))
    if r < 0:
        return None
    return bool(r), (int(p.value) if r else None)


def reduce_columns(columns: list[list[int]]) -> list[int]:
    """Alg 2 on an explicit Z/2 matrix given as row lists; returns low per column (-1 = zero)."""
    lib = _load()
    ptr = np.zeros(len(columns) + 1, np.int64)
    for j, c in enumerate(columns):
        ptr[j + 1] = ptr[j] + len(c)
    rows = np.array([r for c in columns for r in c] or [0], np.int32)
    low = np.empty(max(len(columns), 1), np.int32)
    rc = lib.oracle_reduce_columns(len(columns), ptr.ctypes.data, rows.ctypes.data, low.ctypes.data)
    if rc != 0:
        raise ValueError("bad matrix")
    return low[: len(columns)].tolist()


def reduce_csc(col_ptr: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """reduce_columns on a CSC matrix (col_ptr int64[ncols+1], rows int32[])."""
    lib = _load()
    ptr = np.ascontiguousarray(col_ptr, np.int64)
    rw = np.ascontiguousarray(rows, np.int32)
    n = ptr.size - 1
    low = np.empty(max(n, 1), np.int32)
    rc = lib.oracle_reduce_columns(n, ptr.ctypes.data, rw.ctypes.data if rw.size else None, low.ctypes.data)
    if rc != 0:
        raise ValueError("bad matrix")
    return low[:n]


def enclosing_radius(lower_tri: np.ndarray, n: int) -> float:
    lt = np.ascontiguousarray(lower_tri, dtype=np.float32)
    return float(_load().oracle_enclosing_radius(lt.ctypes.data if lt.size else None, n))
