"""Test-only model of the sharded protocol (include/vr.h "Multi-GPU", implemented by the
library in C++: vr_api.cu run_distributed) on CPU: one rank's device stage, for tiny inputs,
and the per-dimension orchestration with the exchanges over torch.distributed (gloo).  The
GPU tests run the library's own implementation with emulated ranks (dist.run_ranks).

The per-simplex facts the GPU kernels compute — survival under the threshold, the
apparent pair (Def 5.3.4), clearing — are taken from the CPU oracle; the residual
reduction is the library's own host code (vr_host_residual, no GPU needed).  The shard of
a rank follows the dense kernel's rule: prefix row r (colex rank of the top d vertices)
belongs to rank (C(n,d) - 1 - r) mod world.
"""
from __future__ import annotations

import itertools
import math

import numpy as np
import torch

import paper_2502_05063_b200 as vr
from datagen import clouds as G
from oracle import oracle as O

RINF = 0xFFFFFFFF


def bits_for(x: int) -> int:
    return max(1, int(x).bit_length())


def vertices(cidx: int, k: int, n: int):
    """Eq 5.6 decode (test helper): k vertices, decreasing."""
    out, hi = [], n
    for p in range(k):
        kk = k - p
        v = kk - 1
        while v + 1 < hi and math.comb(v + 1, kk) <= cidx:
            v += 1
        out.append(v)
        cidx -= math.comb(v, kk)
        hi = v
    return out


class ModelBackend:
    def __init__(self, lt, n, max_dim, rank_id, world):
        self.n, self.D, self.rank_id, self.world = n, max_dim, rank_id, world
        self.lt = np.ascontiguousarray(lt, np.float32)
        self.t = O.enclosing_radius(self.lt, n)
        srt = np.sort(self.lt)
        self.m = int(np.searchsorted(srt, np.float32(self.t), side="right"))
        self.maxr = self.m - 1
        self.values = srt[: self.m].astype(np.float32)
        sq = G.square_from_lower_tri(self.lt, n)
        R = np.searchsorted(srt, sq, side="left").astype(np.uint32)
        R[sq > np.float32(self.t)] = RINF
        np.fill_diagonal(R, 0)
        self.R = R
        self.device = torch.device("cpu")
        self.ref = O.barcode(self.lt, n, max_dim, self.t)
        # dimension 0 (replicated): deaths = the merging edges
        p0 = self.ref.dims[0]
        self.pairs = {0: [(float(b), float(d)) for b, d in zip(p0.birth, p0.death)]}
        deaths0 = [int(c) for c, d in zip(p0.death_cidx, p0.death) if np.isfinite(d)]
        self.bitmaps = {}
        for d in range(1, max_dim + 1):
            words = (math.comb(n, d + 1) + 31) // 32
            self.bitmaps[d] = np.zeros(max(words, 1), np.uint32)
        self._set_bits(1, deaths0)
        self.local = {}
        self.counters_ = {}

    def _set_bits(self, d, cids):
        if d in self.bitmaps:
            for c in cids:
                self.bitmaps[d][c >> 5] |= np.uint32(1 << (c & 31))

    def _bit(self, d, c):
        return bool((int(self.bitmaps[d][c >> 5]) >> (c & 31)) & 1)

    def dim_local(self, d):
        n = self.n
        cidx, app, partner = O.apparent(self.lt, n, d, self.t)
        rows_total = math.comb(n, d)
        cb = bits_for(math.comb(n, d + 1) - 1)
        keys, surv, napp, ncl = [], 0, 0, 0
        for c, a, pt in zip(cidx.tolist(), app.tolist(), partner.tolist()):
            vs = vertices(c, d + 1, n)
            row = sum(math.comb(vs[i], d - i) for i in range(d))  # colex rank of the top d vertices
            if (rows_total - 1 - row) % self.world != self.rank_id:
                continue
            surv += 1
            if self._bit(d, c):
                ncl += 1
                continue
            if a:
                napp += 1
                self._set_bits(d + 1, [pt])
                continue
            rs = max(int(self.R[x, y]) for x, y in itertools.combinations(vs, 2))
            keys.append(((self.maxr - rs) << cb) | c)
        self.local[d] = np.sort(np.array(keys, np.uint64))
        self.counters_[d] = [surv, napp, ncl, 0, 0, len(keys)]
        words = len(self.bitmaps[d + 1]) if d < self.D else 0
        return len(keys), words

    def local_keys(self, d, nkeys):
        return torch.from_numpy(self.local[d].view(np.int64).copy())

    def bitmap_out(self, d, words):
        return torch.from_numpy(self.bitmaps[d].view(np.int32).copy())

    def bitmap_in(self, d, t):
        self.bitmaps[d] = t.numpy().view(np.uint32).copy()

    def counters(self, d):
        return list(self.counters_[d])

    def dim_finish(self, d, merged):
        cb = bits_for(math.comb(self.n, d + 1) - 1)
        b, de, bc, dc, _ = vr.host_residual(self.R.reshape(-1), self.values, self.n, d, self.maxr, cb, merged)
        self.pairs[d] = list(zip(b.tolist(), de.tolist()))
        deaths = [int(x) for x, y in zip(dc.tolist(), de.tolist()) if math.isfinite(y)]
        self._set_bits(d + 1, deaths)

    def end(self):
        bc = vr.Barcode(self.D, float(self.t))
        for d in range(self.D + 1):
            ps = sorted((b, e) for b, e in self.pairs.get(d, []) if b < e)
            bc.pairs.append(np.array(ps, np.float32).reshape(-1, 2))
            s = {k: 0 for k in ("survivors", "apparent", "cleared", "queued", "scanned")}
            s["pairs_all"] = sum(1 for b, e in self.pairs.get(d, []) if math.isfinite(e))
            if d >= 1:
                s["apparent"] = self.counters_[d][1]
                s["pairs_all"] += s["apparent"]
            bc.stats.append(s)
        return bc


# ------------------------------------------------------------------ the protocol (model)
def merge_sorted_keys(parts: list) -> np.ndarray:
    """k-way merge of per-rank ascending uint64 key arrays (keys are distinct simplices)."""
    parts = [np.asarray(p, dtype=np.uint64) for p in parts if len(p)]
    if not parts:
        return np.zeros(0, np.uint64)
    out = np.concatenate(parts)
    out.sort(kind="stable")
    return out



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


def globalize_stats(bc, totals: dict, local: dict):
    """Hot-path counters of the returned barcode are local to the rank: replace them by
    the sums over the ranks (pairs_all counts the apparent pairs, zero-length)."""
    for d, t in totals.items():
        bc.stats[d]["pairs_all"] += t["apparent"] - local[d]["apparent"]
        for k in ("survivors", "apparent", "cleared", "queued", "scanned"):
            bc.stats[d][k] = t[k]
    return bc


