"""paper_2502_05063_b200 — B200-native Vietoris–Rips persistence barcodes (Ripser++ hot path).

Thin ctypes binding over the C ABI in include/vr.h (libvr.so, built for sm_100a by
build.py).  Argument marshalling only: every step of the computation runs inside libvr
(CUDA kernels for the hot path, the library's own host code for dimension 0 and the
residual reduction).  There is no CPU fallback: if libvr.so is missing or no CUDA device
is present, the calls raise.

    import numpy as np, paper_2502_05063_b200 as vr
    bc = vr.barcodes(dist_lower_tri, n, max_dim=2)        # host numpy input
    bc.pairs[1]            # (k, 2) float32 (birth, death), birth < death, sorted
    bc.stats[1]["apparent"]
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

__all__ = ["barcodes", "barcodes_coo", "barcodes_device", "radix_sort_u64", "hypha_pivots", "min_cost_flow", "w1", "w1_network", "Plan", "Barcode", "VRError", "lib_path", "load"]

_HERE = os.path.dirname(os.path.abspath(__file__))
# VR_LIB: another build of the library (e.g. the bounds-checked libvr_checks.so, build.py --checks)
lib_path = os.environ.get("VR_LIB") or os.path.join(_HERE, "libvr.so")

VR_OK, VR_EINVAL, VR_EINPUT, VR_ECAPACITY, VR_EDEVICE = 0, 1, 2, 3, 4
_CODES = {1: "VR_EINVAL", 2: "VR_EINPUT", 3: "VR_ECAPACITY", 4: "VR_EDEVICE"}


class VRError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_CODES.get(code, code)}: {msg}")
        self.code = code


class _Pair(ctypes.Structure):
    _fields_ = [("birth", ctypes.c_float), ("death", ctypes.c_float)]


class _IndexPair(ctypes.Structure):
    _fields_ = [("birth_cidx", ctypes.c_uint64), ("death_cidx", ctypes.c_uint64)]


class _Options(ctypes.Structure):
    _fields_ = [("include_zero", ctypes.c_int32), ("index_pairs", ctypes.c_int32), ("residual_mode", ctypes.c_int32),
                ("apparent_steps", ctypes.c_int32), ("device", ctypes.c_int32), ("rows_per_grab", ctypes.c_int32),
                ("scan_variant", ctypes.c_int32), ("sparse_mode", ctypes.c_int32), ("num_gpus", ctypes.c_int32),
                ("hot_path_only", ctypes.c_int32), ("reserved", ctypes.c_int32 * 2)]


_STAT_FIELDS = ["candidates", "survivors", "apparent", "cleared", "residual_columns", "emergent", "pairs_all",
                "pairs_positive", "essential", "queued", "scanned"]
_STAT_TIMES = ["ms_enumerate", "ms_resolve", "ms_sort", "ms_residual", "ms_transfer"]


class _Stats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in _STAT_FIELDS] + [(f, ctypes.c_double) for f in _STAT_TIMES] + \
               [("kernels", ctypes.c_int64), ("bytes_l2", ctypes.c_int64), ("bytes_hbm", ctypes.c_int64),
                ("ms_exchange", ctypes.c_double)]


# vr_stats.kernels flags (include/vr.h)
KERNEL_ROW, KERNEL_FLAT, KERNEL_SPARSE, KERNEL_SMEM_WINDOW = 1, 2, 4, 8


_lib = None


def load() -> ctypes.CDLL:
    """Load libvr.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(lib_path):
        raise ImportError(f"libvr.so not found at {lib_path}: run `python paper_2502_05063_b200/build.py` "
                          "(there is no CPU fallback for the hot path)")
    if "VR_NCCL_LIB" not in os.environ:  # the NCCL torch uses (libvr loads it at the first communicator)
        try:
            import nvidia.nccl
            for d in nvidia.nccl.__path__:
                cand = os.path.join(d, "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ["VR_NCCL_LIB"] = cand
                    break
        except ImportError:
            pass
    lib = ctypes.CDLL(lib_path)
    vp, i64, i32, f32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_float
    sig = {
        "vr_barcodes": (ctypes.c_int, [vp, i64, i32, f32, vp, ctypes.POINTER(vp)]),
        "vr_barcodes_device": (ctypes.c_int, [vp, i64, i32, f32, vp, vp, ctypes.POINTER(vp)]),
        "vr_barcodes_coo": (ctypes.c_int, [i64, i64, vp, vp, vp, i32, f32, vp, ctypes.POINTER(vp)]),
        "vr_max_dim": (i32, [vp]),
        "vr_num_pairs": (i64, [vp, i32]),
        "vr_pairs": (vp, [vp, i32]),
        "vr_num_index_pairs": (i64, [vp, i32]),
        "vr_index_pairs": (vp, [vp, i32]),
        "vr_stats_get": (ctypes.c_int, [vp, i32, ctypes.POINTER(_Stats)]),
        "vr_threshold_used": (f32, [vp]),
        "vr_free": (None, [vp]),
        "vr_last_error": (ctypes.c_char_p, []),
        "vr_plan_create": (ctypes.c_int, [vp, i64, i32, f32, vp, vp, ctypes.POINTER(vp), ctypes.POINTER(vp)]),
        "vr_plan_replay": (ctypes.c_int, [vp, ctypes.POINTER(i64)]),
        "vr_plan_survivors": (i64, [vp]),
        "vr_plan_check": (ctypes.c_int, [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "vr_plan_timing": (ctypes.c_int, [vp, ctypes.POINTER(ctypes.c_double)]),
        "vr_plan_free": (None, [vp]),
        "vr_plan_dim_timing": (ctypes.c_int, [vp, i32, ctypes.POINTER(ctypes.c_double)]),
        "vr_radix_sort_u64": (ctypes.c_int, [vp, i64, i32, i32]),
        "vr_sort_columns_u64": (ctypes.c_int, [vp, i64, i32, i32, ctypes.c_uint64, ctypes.POINTER(i32)]),
        "vr_hypha_pivots": (ctypes.c_int, [vp, vp, i64, vp, i32, vp, vp]),
        "vr_min_cost_flow": (ctypes.c_int, [i64, vp, i64, vp, vp, vp, i64, vp, vp]),
        "vr_w1": (ctypes.c_int, [vp, i64, vp, i64, ctypes.c_double, ctypes.c_uint64, i32, i64, vp, vp]),
        "vr_w1_network": (ctypes.c_int, [vp, i64, vp, i64, ctypes.c_double, ctypes.c_uint64, i32, vp, vp]),
        "vr_w1_net_nodes": (i64, [vp]),
        "vr_w1_net_arcs": (i64, [vp]),
        "vr_w1_net_get": (None, [vp, vp, vp, vp, vp, vp]),
        "vr_w1_net_free": (None, [vp]),
        "vr_nccl_unique_id": (ctypes.c_int, [vp]),
        "vr_comm_nccl": (ctypes.c_int, [vp, i32, i32, i32, ctypes.POINTER(vp)]),
        "vr_comm_local": (ctypes.c_int, [i32, vp]),
        "vr_comm_free": (None, [vp]),
        "vr_barcodes_comm": (ctypes.c_int, [vp, i64, i32, f32, vp, vp, ctypes.POINTER(vp)]),
        "vr_plan_create_comm": (ctypes.c_int, [vp, i64, i32, f32, vp, vp, vp, ctypes.POINTER(vp), ctypes.POINTER(vp)]),
        "vr_plan_launches": (i64, [vp]),
        "vr_probe_peaks": (ctypes.c_int, [i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
        "vr_host_residual": (ctypes.c_int, [vp, vp, i64, i64, i32, ctypes.c_uint32, i32, vp, i64, i32, vp, vp, vp, vp,
                                            ctypes.POINTER(i64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(rc: int):
    if rc != VR_OK:
        raise VRError(rc, load().vr_last_error().decode(errors="replace"))


def _options(include_zero=False, index_pairs=False, residual_mode=0, apparent_steps=0, device=0, rows_per_grab=0,
             scan_variant=0, sparse_mode=0, num_gpus=0, hot_path_only=False) -> _Options:
    o = _Options()
    o.num_gpus, o.hot_path_only = int(num_gpus), int(hot_path_only)
    o.include_zero, o.index_pairs, o.residual_mode = int(include_zero), int(index_pairs), int(residual_mode)
    o.apparent_steps, o.device = int(apparent_steps), int(device)
    o.rows_per_grab, o.scan_variant, o.sparse_mode = int(rows_per_grab), int(scan_variant), int(sparse_mode)
    return o


@dataclass
class Barcode:
    max_dim: int
    threshold: float
    pairs: list = field(default_factory=list)        # per dim: (k, 2) float32
    index_pairs: list = field(default_factory=list)  # per dim: (k, 2) uint64 (birth cidx, death cidx)
    stats: list = field(default_factory=list)        # per dim: dict


def _collect(h) -> Barcode:
    lib = load()
    D = lib.vr_max_dim(h)
    bc = Barcode(D, float(lib.vr_threshold_used(h)))
    for d in range(D + 1):
        k = lib.vr_num_pairs(h, d)
        arr = np.zeros((k, 2), np.float32)
        if k:
            ctypes.memmove(arr.ctypes.data, lib.vr_pairs(h, d), k * 8)
        bc.pairs.append(arr)
        k = lib.vr_num_index_pairs(h, d)
        ip = np.zeros((k, 2), np.uint64)
        if k:
            ctypes.memmove(ip.ctypes.data, lib.vr_index_pairs(h, d), k * 16)
        bc.index_pairs.append(ip)
        s = _Stats()
        _check(lib.vr_stats_get(h, d, ctypes.byref(s)))
        bc.stats.append({f: getattr(s, f) for f in _STAT_FIELDS + _STAT_TIMES + ["kernels", "bytes_l2", "bytes_hbm",
                                                                                "ms_exchange"]})
    return bc


def barcodes(dist_lower_tri, n: int, max_dim: int, threshold: float = math.inf, **opts) -> Barcode:
    """vr_barcodes: host fp32 lower-distance vector (Ripser order, n(n-1)/2 values)."""
    lib = load()
    lt = np.ascontiguousarray(dist_lower_tri, dtype=np.float32)
    if lt.size != n * (n - 1) // 2:
        raise ValueError("dist_lower_tri must hold n(n-1)/2 values")
    h = ctypes.c_void_p()
    o = _options(**opts)
    rc = lib.vr_barcodes(lt.ctypes.data if lt.size else None, n, max_dim, threshold, ctypes.byref(o), ctypes.byref(h))
    _check(rc)
    try:
        return _collect(h)
    finally:
        lib.vr_free(h)


def barcodes_coo(n: int, rows, cols, dist, max_dim: int, threshold: float = math.inf, **opts) -> Barcode:
    """vr_barcodes_coo: the distance matrix as (rows[k], cols[k], dist[k]) entries; absent
    pairs are absent edges."""
    lib = load()
    r = np.ascontiguousarray(rows, dtype=np.int32)
    c = np.ascontiguousarray(cols, dtype=np.int32)
    d = np.ascontiguousarray(dist, dtype=np.float32)
    if not (r.size == c.size == d.size):
        raise ValueError("rows, cols and dist must have the same length")
    h = ctypes.c_void_p()
    o = _options(**opts)
    _check(lib.vr_barcodes_coo(n, r.size, r.ctypes.data if r.size else None, c.ctypes.data if c.size else None,
                               d.ctypes.data if d.size else None, max_dim, threshold, ctypes.byref(o), ctypes.byref(h)))
    try:
        return _collect(h)
    finally:
        lib.vr_free(h)


def barcodes_device(d_dist_lower_tri, n: int, max_dim: int, threshold: float = math.inf, stream=None, **opts) -> Barcode:
    """vr_barcodes_device: `d_dist_lower_tri` is a CUDA float32 torch tensor (or a raw device
    pointer int) on the current device; `stream` a torch.cuda.Stream (None = current)."""
    lib = load()
    ptr, st = _device_ptr_and_stream(d_dist_lower_tri, n, stream)
    h = ctypes.c_void_p()
    o = _options(**opts)
    _check(lib.vr_barcodes_device(ptr, n, max_dim, threshold, ctypes.byref(o), st, ctypes.byref(h)))
    try:
        return _collect(h)
    finally:
        lib.vr_free(h)


def _device_ptr_and_stream(t, n, stream):
    if isinstance(t, int):
        ptr = t
    else:
        if not (t.is_cuda and t.dtype.is_floating_point and t.element_size() == 4 and t.is_contiguous()):
            raise ValueError("expected a contiguous CUDA float32 tensor")
        if t.numel() != n * (n - 1) // 2:
            raise ValueError("tensor must hold n(n-1)/2 values")
        ptr = t.data_ptr()
    if stream is None:
        try:
            import torch
            st = torch.cuda.current_stream().cuda_stream
        except Exception:  # pragma: no cover
            st = 0
    else:
        st = getattr(stream, "cuda_stream", stream)
    return ctypes.c_void_p(ptr or None), ctypes.c_void_p(st or None)


class _HyphaStats(ctypes.Structure):
    _fields_ = [("stable", ctypes.c_int64), ("unstable", ctypes.c_int64), ("cleared", ctypes.c_int64),
                ("compressed", ctypes.c_int64), ("additions", ctypes.c_int64), ("ms_gpu_scan", ctypes.c_double),
                ("ms_host", ctypes.c_double), ("ms_compress_scan", ctypes.c_double), ("ms_reduce", ctypes.c_double),
                ("ms_total", ctypes.c_double), ("ms_prepare", ctypes.c_double), ("threads", ctypes.c_int64)]


def hypha_pivots(col_ptr, rows, dims=None, compression: bool = True, clearing: bool = True):
    """HYPHA (Ch.4) on an explicit CSC boundary matrix: (low per column, stats dict).
    For a matrix that is not a boundary matrix pass dims=None, compression=clearing=False."""
    lib = load()
    cp = np.ascontiguousarray(col_ptr, dtype=np.int64)
    rw = np.ascontiguousarray(rows, dtype=np.int32)
    n = cp.size - 1
    dm = None if dims is None else np.ascontiguousarray(dims, dtype=np.int32)
    low = np.zeros(max(n, 1), np.int32)
    st = _HyphaStats()
    _check(lib.vr_hypha_pivots(cp.ctypes.data, rw.ctypes.data if rw.size else None, n,
                               dm.ctypes.data if dm is not None else None,
                               (1 if compression else 0) | (2 if clearing else 0),
                               low.ctypes.data, ctypes.byref(st)))
    return low[:n], {f: getattr(st, f) for f, _ in _HyphaStats._fields_}


class _McfStats(ctypes.Structure):
    _fields_ = [("pivots", ctypes.c_int64), ("degenerate", ctypes.c_int64), ("blocks", ctypes.c_int64),
                ("optimal", ctypes.c_int32), ("infeasible", ctypes.c_int32), ("ms_pricing", ctypes.c_double),
                ("ms_update", ctypes.c_double)]


def min_cost_flow(supply, tail, head, cost, max_blocks: int = 0):
    """Uncapacitated min-cost flow (network simplex, block search): (total cost, stats)."""
    lib = load()
    sp = np.ascontiguousarray(supply, dtype=np.int64)
    t = np.ascontiguousarray(tail, dtype=np.int32)
    h = np.ascontiguousarray(head, dtype=np.int32)
    c = np.ascontiguousarray(cost, dtype=np.float64)
    out = ctypes.c_double(0.0)
    st = _McfStats()
    _check(lib.vr_min_cost_flow(sp.size, sp.ctypes.data if sp.size else None, t.size, t.ctypes.data if t.size else None,
                                h.ctypes.data if h.size else None, c.ctypes.data if c.size else None, int(max_blocks),
                                ctypes.byref(out), ctypes.byref(st)))
    return out.value, {f: getattr(st, f) for f, _ in _McfStats._fields_}


W1_EXACT = 1
W1_NO_CONDENSE = 2


class _W1Stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in ("points_a", "points_b", "nodes", "arcs", "wspd_pairs", "tree_height",
                                                "wspd_levels", "pivots", "degenerate", "blocks")] + \
               [("optimal", ctypes.c_int32), ("condensed", ctypes.c_int32), ("warm_start", ctypes.c_int32),
                ("pad_", ctypes.c_int32)] + \
               [(k, ctypes.c_double) for k in ("rwmd", "delta", "eps_condense", "eps_spanner", "bound_lo", "bound_hi",
                                                 "ms_h2d", "ms_rwmd", "ms_condense", "ms_tree", "ms_wspd", "ms_arcs",
                                                 "ms_d2h", "ms_build", "ms_simplex", "ms_total",
                                                 "ms_pricing", "ms_update")]


def _diagram(P):
    P = np.ascontiguousarray(np.asarray(P, dtype=np.float32).reshape(-1, 2))
    return P, P.shape[0]


W1_WARM_DIAGONAL = 4


def _w1_flags(exact, condense, warm=False):
    return (W1_EXACT if exact else 0) | (0 if condense else W1_NO_CONDENSE) | (W1_WARM_DIAGONAL if warm else 0)


def w1(A, B, s: float = 18.0, seed: int = 0, exact: bool = False, condense: bool = True, max_blocks: int = 0,
       warm: bool = False):
    """PDoptFlow (Ch.6): W1 between diagrams A, B ((n, 2) birth/death): (value, stats)."""
    lib = load()
    A, na = _diagram(A)
    B, nb = _diagram(B)
    out = ctypes.c_double(0.0)
    st = _W1Stats()
    _check(lib.vr_w1(A.ctypes.data if na else None, na, B.ctypes.data if nb else None, nb, float(s), int(seed) & (2**64 - 1),
                     _w1_flags(exact, condense, warm), int(max_blocks), ctypes.byref(out), ctypes.byref(st)))
    return out.value, {f: getattr(st, f) for f, _ in _W1Stats._fields_}


def w1_network(A, B, s: float = 18.0, seed: int = 0, exact: bool = False, condense: bool = True):
    """The transshipment network PDoptFlow builds (Alg 22 lines 1-5), as numpy arrays."""
    lib = load()
    A, na = _diagram(A)
    B, nb = _diagram(B)
    h = ctypes.c_void_p()
    st = _W1Stats()
    _check(lib.vr_w1_network(A.ctypes.data if na else None, na, B.ctypes.data if nb else None, nb, float(s),
                             int(seed) & (2**64 - 1), _w1_flags(exact, condense), ctypes.byref(h), ctypes.byref(st)))
    try:
        N = lib.vr_w1_net_nodes(h)
        M = lib.vr_w1_net_arcs(h)
        xy = np.zeros((max(N, 1), 2), np.float64)
        sup = np.zeros(max(N, 1), np.int64)
        t = np.zeros(max(M, 1), np.int32)
        hd = np.zeros(max(M, 1), np.int32)
        c = np.zeros(max(M, 1), np.float64)
        lib.vr_w1_net_get(h, xy.ctypes.data, sup.ctypes.data, t.ctypes.data, hd.ctypes.data, c.ctypes.data)
    finally:
        lib.vr_w1_net_free(h)
    return {"xy": xy[:N], "supply": sup[:N], "tail": t[:M], "head": hd[:M], "cost": c[:M],
            "stats": {f: getattr(st, f) for f, _ in _W1Stats._fields_}}


def radix_sort_u64(keys: np.ndarray, begin_bit: int = 0, end_bit: int = 64) -> np.ndarray:
    """The library's device LSD radix sort on bits [begin_bit, end_bit) (component test entry)."""
    a = np.ascontiguousarray(keys, dtype=np.uint64).copy()
    _check(load().vr_radix_sort_u64(a.ctypes.data if a.size else None, a.size, begin_bit, end_bit))
    return a


def sort_columns_u64(keys: np.ndarray, cbits: int, end_bit: int, bins: int, mode: int = -1):
    """The library's residual-column sort (component test entry).  Returns (sorted, path)."""
    a = np.ascontiguousarray(keys, dtype=np.uint64).copy()
    m = ctypes.c_int32(mode)
    _check(load().vr_sort_columns_u64(a.ctypes.data if a.size else None, a.size, cbits, end_bit, bins, ctypes.byref(m)))
    return a, int(m.value)


def host_residual(rank: np.ndarray, values: np.ndarray, n: int, d: int, maxr: int, cbits: int, keys: np.ndarray,
                  mode: int = 0):
    """The library's host residual reduction (component entry; no GPU needed).  Returns
    (birth, death, birth_cidx, death_cidx, emergent) per column."""
    lib = load()
    R = np.ascontiguousarray(rank, dtype=np.uint32)
    V = np.ascontiguousarray(values, dtype=np.float32)
    K = np.ascontiguousarray(keys, dtype=np.uint64)
    m = K.size
    b = np.zeros(max(m, 1), np.float32); de = np.zeros(max(m, 1), np.float32)
    bc = np.zeros(max(m, 1), np.uint64); dc = np.zeros(max(m, 1), np.uint64)
    em = ctypes.c_int64(0)
    _check(lib.vr_host_residual(R.ctypes.data, V.ctypes.data, V.size, n, d, maxr, cbits, K.ctypes.data if m else None, m,
                                mode, b.ctypes.data, de.ctypes.data, bc.ctypes.data, dc.ctypes.data, ctypes.byref(em)))
    return b[:m], de[:m], bc[:m], dc[:m], int(em.value)


class Plan:
    """vr_plan: one full run, then `replay()` re-launches the GPU hot path of every
    dimension (a0..a6) with the recorded sizes, asynchronously on `stream`."""

    def __init__(self, d_dist_lower_tri, n: int, max_dim: int, threshold: float = math.inf, stream=None, comm=None,
                 **opts):
        """comm: a dist.Comm — this rank's part of a sharded plan (vr_plan_create_comm)."""
        lib = load()
        self._keep = (d_dist_lower_tri, comm)
        ptr, st = _device_ptr_and_stream(d_dist_lower_tri, n, stream)
        self._h = ctypes.c_void_p()
        r = ctypes.c_void_p()
        o = _options(**opts)
        if comm is None:
            _check(lib.vr_plan_create(ptr, n, max_dim, threshold, ctypes.byref(o), st, ctypes.byref(self._h),
                                      ctypes.byref(r)))
        else:
            _check(lib.vr_plan_create_comm(ptr, n, max_dim, threshold, ctypes.byref(o), comm.ptr, st,
                                           ctypes.byref(self._h), ctypes.byref(r)))
        try:
            self.result = _collect(r)
        finally:
            lib.vr_free(r)
        self.survivors = int(lib.vr_plan_survivors(self._h))

    def replay(self) -> int:
        n = ctypes.c_int64(0)
        _check(load().vr_plan_replay(self._h, ctypes.byref(n)))
        return int(n.value)

    def check(self):
        a, r = ctypes.c_int64(0), ctypes.c_int64(0)
        _check(load().vr_plan_check(self._h, ctypes.byref(a), ctypes.byref(r)))
        return int(a.value), int(r.value)

    def timing(self) -> dict:
        """Device ms of the last replay's stages + the first run's work counters."""
        out = (ctypes.c_double * 9)()
        _check(load().vr_plan_timing(self._h, out))
        keys = ["ms_tables", "ms_enumerate", "ms_resolve", "ms_sort", "candidates", "survivors", "scanned",
                "rank_ops_enumerate", "rank_ops_resolve"]
        return dict(zip(keys, list(out)))

    def dim_timing(self, d: int) -> dict:
        """Per-dimension device ms of the last replay + the first run's work (vr_plan_dim_timing)."""
        out = (ctypes.c_double * 10)()
        _check(load().vr_plan_dim_timing(self._h, d, out))
        keys = ["ms_enumerate", "ms_resolve", "ms_sort", "ms_setup", "survivors", "reads_a1", "reads_a5",
                "reads_a5_phase2", "decode", "kernels"]
        return dict(zip(keys, list(out)))

    def close(self):
        if self._h:
            load().vr_plan_free(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
