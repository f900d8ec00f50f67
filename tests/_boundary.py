"""Test-only builders of explicit Z/2 boundary matrices in CSC (col_ptr, rows, dims) for the
HYPHA row (PAPER.md Ch.4).  Pure input generation: simplices are listed, sorted into a
filtration order and their facets looked up — no reduction arithmetic lives here.

A filtration order only needs every face before its cofaces; the Rips one
sorts by (diameter, dimension, vertices), the sphere one by (dimension, vertices).
"""
from __future__ import annotations

import itertools

import numpy as np


def _csc(simplices):
    index = {s: i for i, s in enumerate(simplices)}
    ptr = np.zeros(len(simplices) + 1, np.int64)
    rows, dims = [], np.zeros(len(simplices), np.int32)
    for j, s in enumerate(simplices):
        dims[j] = len(s) - 1
        col = sorted(index[f] for f in itertools.combinations(s, len(s) - 1)) if len(s) > 1 else []
        rows.extend(col)
        ptr[j + 1] = ptr[j] + len(col)
    return ptr, np.array(rows, np.int32), dims


def rips(lt: np.ndarray, n: int, max_dim: int, threshold: float = float("inf")):
    """Boundary matrix of the Rips filtration up to dimension max_dim (+1 so that the top
    dimension's classes can die), ordered by (diameter, dimension, colex)."""
    sq = np.zeros((n, n), np.float32)
    iu = np.tril_indices(n, -1)
    sq[iu] = lt
    sq = np.maximum(sq, sq.T)
    simp = []
    for k in range(1, max_dim + 3):
        for s in itertools.combinations(range(n), k):
            dia = max((sq[a, b] for a, b in itertools.combinations(s, 2)), default=np.float32(0))
            if dia <= threshold:
                simp.append((float(dia), k, s[::-1], s))  # ties: colex (= cidx order, Eq 5.6)
    simp.sort()
    return _csc([s for _, _, _, s in simp])


def rips_fast(lt: np.ndarray, n: int, max_dim: int):
    """rips() without a threshold, vectorised (simplices named by Eq 5.6 cidx per dimension):
    the (max_dim+1)-skeleton of the full Rips filtration — e.g. n = 50, max_dim = 3 gives
    the 4-skeleton of the mumford-shaped matrix of Table 4.1 (2.37e6 columns)."""
    from math import comb
    sq = np.zeros((n, n), np.float32)
    sq[np.tril_indices(n, -1)] = lt
    sq = np.maximum(sq, sq.T)
    C = np.array([[comb(v, k) for k in range(max_dim + 3)] for v in range(n + 1)], np.int64)
    per_dim = []
    for k in range(1, max_dim + 3):  # k vertices
        vs = np.array(list(itertools.combinations(range(n), k)), np.int64).reshape(-1, k)[:, ::-1]  # decreasing
        cidx = sum(C[vs[:, i], k - i] for i in range(k))
        srt = np.argsort(cidx)  # generation index = cidx
        vs, cidx = vs[srt], cidx[srt]
        dia = np.zeros(len(vs), np.float32)
        for a in range(k):
            for b in range(a + 1, k):
                dia = np.maximum(dia, sq[vs[:, a], vs[:, b]])
        per_dim.append((vs, cidx, dia))
    dia_all = np.concatenate([p[2] for p in per_dim])
    dim_all = np.concatenate([np.full(len(p[0]), k, np.int64) for k, p in enumerate(per_dim)])
    cid_all = np.concatenate([p[1] for p in per_dim])
    order = np.lexsort((cid_all, dim_all, dia_all))
    pos = np.empty(order.size, np.int64)
    pos[order] = np.arange(order.size)
    base = np.cumsum([0] + [len(p[0]) for p in per_dim])
    # position of (dim k, cidx c): simplices of one dim are generated in cidx order
    ptr = np.zeros(order.size + 1, np.int64)
    cnt = np.concatenate([np.full(len(p[0]), k, np.int64) for k, p in enumerate(per_dim)])  # k+1 facets for k>=1
    cnt[dim_all == 0] = 0
    cnt[dim_all > 0] += 1
    ptr[1:] = np.cumsum(cnt[order])
    rows = np.empty(int(ptr[-1]), np.int64)
    for k, (vs, cidx, dia) in enumerate(per_dim):
        if k == 0:
            continue
        gidx = base[k] + np.arange(len(vs))
        start = ptr[pos[gidx]]
        assert np.array_equal(cidx, np.arange(len(vs)))
        for drop in range(k + 1):
            keep = [i for i in range(k + 1) if i != drop]
            f = vs[:, keep]
            fc = sum(C[f[:, i], k - i] for i in range(k))
            rows[start + drop] = pos[base[k - 1] + fc]
    rows = rows.astype(np.int32)
    # sort rows within each column
    colid = np.repeat(np.arange(order.size), cnt[order])
    o = np.lexsort((rows, colid))
    return ptr, rows[o], (dim_all[order]).astype(np.int32)


def sphere(k: int):
    """All proper faces of the k-simplex on k+1 vertices: a (k-1)-sphere, 2^(k+1)-2 cells."""
    simp = [s for d in range(1, k + 1) for s in itertools.combinations(range(k + 1), d)]
    return _csc(simp)


def sphere_fast(k: int):
    """sphere(k) for large k, vectorised: subsets as bitmasks, ordered by (popcount, colex).
    Facets of the subset mask s are s with one bit cleared."""
    N = 1 << (k + 1)
    masks = np.arange(1, N - 1, dtype=np.int64)
    pop = np.array([bin(int(x)).count("1") for x in range(1 << 12)], np.int64)
    pc = pop[masks & 4095] + pop[(masks >> 12) & 4095] + pop[(masks >> 24) & 4095]
    order = np.lexsort((masks, pc))
    masks = masks[order]
    pc = pc[order]
    pos = np.full(N, -1, np.int64)
    pos[masks] = np.arange(masks.size)
    ptr = np.zeros(masks.size + 1, np.int64)
    cnt = np.where(pc > 1, pc, 0)
    ptr[1:] = np.cumsum(cnt)
    rows = np.empty(int(ptr[-1]), np.int64)
    fill = ptr[:-1].copy()
    for b in range(k + 1):
        has = ((masks >> b) & 1).astype(bool) & (pc > 1)
        idx = np.nonzero(has)[0]
        rows[fill[idx]] = pos[masks[idx] ^ (1 << b)]
        fill[idx] += 1
    # sort rows within each column
    colid = np.repeat(np.arange(masks.size), cnt)
    o = np.lexsort((rows, colid))
    return ptr, rows[o].astype(np.int32), (pc - 1).astype(np.int32)


def random_upper(ncols: int, density: float, seed: int):
    """A random strictly upper-triangular Z/2 matrix (not a boundary matrix)."""
    rng = np.random.default_rng(seed)
    ptr = np.zeros(ncols + 1, np.int64)
    rows = []
    for j in range(ncols):
        if j:
            k = rng.binomial(j, min(1.0, density))
            col = np.sort(rng.choice(j, size=k, replace=False)) if k else np.zeros(0, np.int64)
        else:
            col = np.zeros(0, np.int64)
        rows.extend(col.tolist())
        ptr[j + 1] = ptr[j] + len(col)
    return ptr, np.array(rows, np.int32)


def columns(ptr, rows):
    return [rows[ptr[j]: ptr[j + 1]].tolist() for j in range(len(ptr) - 1)]
