"""Multi-GPU driver: one process per GPU, shards of every dimension's hot path, and the
two exchanges of SURVEY.md §8(e) per dimension over torch.distributed (NCCL on GPUs).

Per dimension d (include/vr.h "Distributed stepping"):
  1. every rank runs its shard of the hot path (vr_dist_dim_local): enumeration, apparent
     test, clearing, compaction and the local radix sort of its residual columns;
  2. exchange A — the next dimension's clearing bitmap: SUM all-reduce.  A death simplex
     is the apparent cofacet of exactly one column, found by exactly one rank, so no two
     ranks set the same bit and the integer sum of the words is their bitwise OR;
  3. exchange B — the residual columns: all-gather of the locally sorted keys, merged by
     key (the key order is the coboundary order, so the merge is deterministic);
  4. every rank runs the host residual on the merged columns (vr_dist_dim_finish), so all
     ranks hold the same deaths for the next dimension and the same barcode at the end.

The device stage sits behind `Backend` so the orchestration and the collectives can be
exercised on CPU with gloo (tests/test_dist_cpu.py); `LibBackend` is the real one.
Argument marshalling only: the computation happens in libvr.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

from . import Barcode, _check, _collect, _device_ptr_and_stream, _options, load

__all__ = ["barcodes_sharded", "LibBackend", "merge_sorted_keys", "orchestrate", "globalize_stats"]


def merge_sorted_keys(parts: list) -> np.ndarray:
    """k-way merge of per-rank ascending uint64 key arrays (keys are distinct simplices)."""
    parts = [np.asarray(p, dtype=np.uint64) for p in parts if len(p)]
    if not parts:
        return np.zeros(0, np.uint64)
    out = np.concatenate(parts)
    out.sort(kind="stable")
    return out


class LibBackend:
    """The device stage of one rank, through the C ABI (torch tensors for the buffers
    the collectives touch)."""

    def __init__(self, d_dist_lower_tri, n, max_dim, threshold, rank, world, stream=None, **opts):
        import torch
        self.torch = torch
        self.lib = load()
        self.keep = d_dist_lower_tri
        ptr, st = _device_ptr_and_stream(d_dist_lower_tri, n, stream)
        self.h = ctypes.c_void_p()
        o = _options(**opts)
        _check(self.lib.vr_dist_begin(ptr, n, max_dim, threshold, ctypes.byref(o), st, rank, world, ctypes.byref(self.h)))
        self.device = d_dist_lower_tri.device

    def dim_local(self, d):
        nk, words = ctypes.c_int64(0), ctypes.c_int64(0)
        _check(self.lib.vr_dist_dim_local(self.h, d, ctypes.byref(nk), ctypes.byref(words)))
        return int(nk.value), int(words.value)

    def local_keys(self, d, nkeys):
        t = self.torch.empty(max(nkeys, 1), dtype=self.torch.int64, device=self.device)
        _check(self.lib.vr_dist_copy_keys(self.h, d, ctypes.c_void_p(t.data_ptr())))
        return t[:nkeys]

    def bitmap_out(self, d, words):
        t = self.torch.empty(words, dtype=self.torch.int32, device=self.device)
        _check(self.lib.vr_dist_bitmap(self.h, d, ctypes.c_void_p(t.data_ptr()), 0))
        return t

    def bitmap_in(self, d, t):
        _check(self.lib.vr_dist_bitmap(self.h, d, ctypes.c_void_p(t.data_ptr()), 1))

    def counters(self, d):
        out = (ctypes.c_int64 * 6)()
        _check(self.lib.vr_dist_counters(self.h, d, out))
        return list(out)

    def dim_finish(self, d, merged: np.ndarray):
        a = np.ascontiguousarray(merged, dtype=np.uint64)
        _check(self.lib.vr_dist_dim_finish(self.h, d, a.ctypes.data if a.size else None, a.size))

    def end(self) -> Barcode:
        r = ctypes.c_void_p()
        _check(self.lib.vr_dist_end(self.h, ctypes.byref(r)))
        try:
            return _collect(r)
        finally:
            self.lib.vr_free(r)

    def close(self):
        if self.h:
            self.lib.vr_plan_free(self.h)
            self.h = ctypes.c_void_p()


def _all_gather_varlen(t, group, dist, torch):
    """all-gather of a 1-D tensor whose length differs per rank (padded to the max)."""
    world = dist.get_world_size(group)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes) if sizes else 0
    buf = torch.zeros(max(m, 1), dtype=t.dtype, device=t.device)
    buf[: t.numel()] = t
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf, group=group)
    return [o[:s] for o, s in zip(outs, sizes)]


def orchestrate(backend, max_dim: int, group=None):
    """Run dimensions 1..max_dim with the two exchanges.  Returns (barcode, per-dimension
    summed hot-path counters, per-dimension local counters)."""
    import torch
    import torch.distributed as dist
    names = ["survivors", "apparent", "cleared", "queued", "scanned", "residual_local"]
    totals, local = {}, {}
    for d in range(1, max_dim + 1):
        nkeys, words = backend.dim_local(d)
        if words:  # exchange A: clearing bitmap of d+1, sum == OR (disjoint bits)
            bm = backend.bitmap_out(d + 1, words)
            dist.all_reduce(bm, op=dist.ReduceOp.SUM, group=group)
            backend.bitmap_in(d + 1, bm)
        # exchange B: residual columns
        parts = _all_gather_varlen(backend.local_keys(d, nkeys), group, dist, torch)
        merged = merge_sorted_keys([p.cpu().numpy().view(np.uint64) for p in parts])
        backend.dim_finish(d, merged)
        lc = backend.counters(d)
        local[d] = dict(zip(names, lc))
        local[d]["next_bitmap_words"] = words
        c = torch.tensor(lc, dtype=torch.int64, device=backend.device)
        dist.all_reduce(c, op=dist.ReduceOp.SUM, group=group)
        totals[d] = dict(zip(names, [int(x) for x in c.cpu().tolist()]))
    return backend.end(), totals, local


def globalize_stats(bc: Barcode, totals: dict, local: dict) -> Barcode:
    """Hot-path counters of the returned barcode are local to the rank: replace them by
    the sums over the ranks (pairs_all counts the apparent pairs, zero-length)."""
    for d, t in totals.items():
        bc.stats[d]["pairs_all"] += t["apparent"] - local[d]["apparent"]
        for k in ("survivors", "apparent", "cleared", "queued", "scanned"):
            bc.stats[d][k] = t[k]
    return bc


class ShardedHotPath:
    """Benchmark harness for N ranks: one full distributed run, then `step()` replays
    this rank's shard of the GPU hot path of every dimension with the two exchanges
    (bitmap SUM all-reduce, all-gather of the sorted residual keys) — device work and
    NCCL collectives only, asynchronous on the current stream."""

    def __init__(self, d_dist_lower_tri, n, max_dim, threshold=math.inf, group=None, **opts):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.D = max_dim
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        self.be = LibBackend(d_dist_lower_tri, n, max_dim, threshold, rank, world, **opts)
        self.result, self.totals, self.local = orchestrate(self.be, max_dim, group)
        self.result = globalize_stats(self.result, self.totals, self.local)
        self.survivors_total = sum(t["survivors"] for t in self.totals.values())
        lib, h = self.be.lib, self.be.h
        self.lib, self.h = lib, h
        # fixed buffers for the exchanges (sizes of the first run are deterministic)
        self.words, self.bm, self.keys, self.gathered = {}, {}, {}, {}
        for d in range(1, max_dim + 1):
            nk = self.local[d]["residual_local"]
            nmax = torch.tensor([nk], dtype=torch.int64, device=self.be.device)
            dist.all_reduce(nmax, op=dist.ReduceOp.MAX, group=group)
            m = max(int(nmax.item()), 1)
            self.keys[d] = torch.zeros(m, dtype=torch.int64, device=self.be.device)
            self.gathered[d] = [torch.zeros(m, dtype=torch.int64, device=self.be.device) for _ in range(world)]
        for d in range(1, max_dim + 1):
            w = self.local[d]["next_bitmap_words"]  # bitmap of d+1; 0 = recompute mode
            if w:
                self.words[d] = w
                self.bm[d] = torch.zeros(w, dtype=torch.int32, device=self.be.device)

    def step(self) -> int:
        """One hot-path pass over every dimension; returns the kernels launched."""
        lib, h, dist, g = self.lib, self.h, self.dist, self.group
        before = lib.vr_plan_launches(h)
        _check(lib.vr_dist_replay_tables(h))
        for d in range(1, self.D + 1):
            _check(lib.vr_dist_replay_dim(h, d))
            if d in self.bm:  # exchange A
                _check(lib.vr_dist_bitmap(h, d + 1, ctypes.c_void_p(self.bm[d].data_ptr()), 2))
                dist.all_reduce(self.bm[d], op=dist.ReduceOp.SUM, group=g)
                _check(lib.vr_dist_bitmap(h, d + 1, ctypes.c_void_p(self.bm[d].data_ptr()), 3))
            # exchange B
            _check(lib.vr_dist_copy_keys_async(h, d, ctypes.c_void_p(self.keys[d].data_ptr())))
            dist.all_gather(self.gathered[d], self.keys[d], group=g)
            _check(lib.vr_dist_replay_deaths(h, d))
        return int(lib.vr_plan_launches(h) - before)

    def close(self):
        self.be.close()


def barcodes_sharded(d_dist_lower_tri, n: int, max_dim: int, threshold: float = math.inf, group=None, **opts):
    """Multi-GPU vr_barcodes: call on every rank of `group` with the same input (a CUDA
    tensor on this rank's device).  Every rank returns the same barcode; the hot-path
    counters in the returned stats are summed over the ranks."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    be = LibBackend(d_dist_lower_tri, n, max_dim, threshold, rank, world, **opts)
    try:
        bc, totals, local = orchestrate(be, max_dim, group)
    finally:
        be.close()
    return globalize_stats(bc, totals, local)
