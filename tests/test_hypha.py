"""HYPHA (PAPER.md Ch.4, Algs 3-10) against the oracle's Alg 2.

The low of every column of a reduced matrix is unique (the pairing does not
depend on the reduction order), so the GPU-scan + host path must reproduce the oracle's
low array exactly — with and without compression, in standard and twist order.
Clearing and compression are only valid on boundary matrices (they use ∂∂ = 0), so the
random non-boundary matrices run without them.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import _boundary as B
from datagen import clouds as G
from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------------ CPU: generators and oracle pins
def test_sphere_generators_agree():
    for k in (2, 3, 5):
        a, b = B.sphere(k), B.sphere_fast(k)
        # same cells in the same (dimension, vertex-set) classes: compare column sizes per dim
        assert a[0][-1] == b[0][-1]
        assert np.array_equal(np.sort(a[2]), np.sort(b[2]))


@pytest.mark.parametrize("k", [2, 4, 6])
def test_oracle_sphere_pair_count(k):
    # ∂Δ^k is a (k-1)-sphere: Betti 1 in dims 0 and k-1, so (#cells - 2)/2 pivots (closed form)
    ptr, rows, dims = B.sphere(k)
    low = O.reduce_columns(B.columns(ptr, rows))
    assert sum(1 for x in low if x >= 0) == (len(low) - 2) // 2
    assert O.reduce_csc(ptr, rows).tolist() == low


@pytest.mark.parametrize("seed", range(3))
def test_rips_generators_agree(seed):
    lt = G.random_tied(9, seed, levels=4) if seed == 1 else G.random_cloud(9, seed)
    for a, b in zip(B.rips(lt, 9, 2), B.rips_fast(lt, 9, 2)):
        assert np.array_equal(a, b)


def test_rips_boundary_is_a_boundary():
    ptr, rows, dims = B.rips(G.random_cloud(7, 0), 7, 2)
    cols = B.columns(ptr, rows)
    for j, c in enumerate(cols):  # ∂∂ = 0 over Z/2
        acc = {}
        for f in c:
            for g in cols[f]:
                acc[g] = acc.get(g, 0) ^ 1
        assert not any(acc.values()), j


# ------------------------------------------------------------------ GPU parity
def _check(ptr, rows, dims, compression, clearing=True):
    import paper_2502_05063_b200 as vr
    exp = O.reduce_csc(ptr, rows).tolist()
    low, st = vr.hypha_pivots(ptr, rows, dims, compression=compression, clearing=clearing)
    assert low.tolist() == exp
    assert st["stable"] + st["unstable"] == len(exp)
    return st


@pytest.mark.gpu
@pytest.mark.parametrize("compression", [False, True])
@pytest.mark.parametrize("twist", [False, True])
def test_fig41(compression, twist):
    cols = []
    for line in open(os.path.join(GOLDEN, "fig4_1_boundary.txt")):
        f = line.split()
        if f and f[0] == "col":
            cols.append([int(x) for x in f[2:]])
    ptr = np.cumsum([0] + [len(c) for c in cols]).astype(np.int64)
    rows = np.array([r for c in cols for r in c], np.int32)
    dims = np.array([0, 0, 0, 1, 1, 1, 2], np.int32) if twist else None
    import paper_2502_05063_b200 as vr
    low, st = vr.hypha_pivots(ptr, rows, dims, compression=compression)
    assert {(int(lo), j) for j, lo in enumerate(low) if lo >= 0} == {(2, 3), (1, 4), (5, 6)}
    # Fig 4.2 narration: (2,3) and (1,4) are 0-addition pivots found by the scan; column 6's
    # low 5 is the leftmost 1 of row 5 too, so the whole matrix is stable but column 5
    assert st["stable"] >= 6


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("compression", [False, True])
@pytest.mark.parametrize("twist", [False, True])
def test_rips_boundary(seed, compression, twist):
    n = 9 + seed % 3
    lt = G.random_tied(n, seed, levels=5) if seed % 2 else G.random_cloud(n, seed)
    t = O.enclosing_radius(lt, n) if seed % 3 == 0 else float("inf")
    ptr, rows, dims = B.rips(lt, n, 2, t)
    _check(ptr, rows, dims if twist else None, compression)
    if not twist and not compression:
        _check(ptr, rows, None, False, clearing=False)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(5))
def test_random_upper(seed):
    ptr, rows = B.random_upper(300 + 50 * seed, 0.02 * (seed + 1), seed)
    _check(ptr, rows, None, False, clearing=False)


@pytest.mark.gpu
@pytest.mark.parametrize("k", [3, 8, 11])
def test_sphere(k):
    ptr, rows, dims = B.sphere_fast(k)
    for comp in (False, True):
        _check(ptr, rows, dims, comp)


@pytest.mark.gpu
def test_empty_and_degenerate():
    import paper_2502_05063_b200 as vr
    low, st = vr.hypha_pivots(np.zeros(1, np.int64), np.zeros(0, np.int32))
    assert low.size == 0
    ptr = np.zeros(6, np.int64)  # five zero columns
    low, st = vr.hypha_pivots(ptr, np.zeros(0, np.int32))
    assert low.tolist() == [-1] * 5 and st["stable"] == 5
    with pytest.raises(Exception):  # a row below the diagonal is not a filtration matrix
        vr.hypha_pivots(np.array([0, 1], np.int64), np.array([0], np.int32))
    with pytest.raises(Exception):  # rows must ascend
        vr.hypha_pivots(np.array([0, 0, 0, 2], np.int64), np.array([1, 0], np.int32))


@pytest.mark.gpu
def test_sphere18_closed_form():
    # The 18-sphere of Fig 4.4 / Table 4.1 (∂Δ^19, 2^20 - 2 cells): (cells - 2)/2 pivots,
    # every pivot row distinct and every pivot row a zero column (a creator).
    import paper_2502_05063_b200 as vr
    ptr, rows, dims = B.sphere_fast(19)
    low, st = vr.hypha_pivots(ptr, rows, dims, compression=True)
    assert np.array_equal(low, O.reduce_csc(ptr, rows))
    piv = low[low >= 0]
    assert piv.size == (low.size - 2) // 2
    assert np.unique(piv).size == piv.size
    assert np.all(low[piv] == -1)


@pytest.mark.gpu
def test_mumford_shaped_4_skeleton():
    # Table 4.1's mumford: the 4-skeleton of the Rips filtration of 50 points (2.37e6 columns)
    import paper_2502_05063_b200 as vr
    ptr, rows, dims = B.rips_fast(G.random_cloud(50, 1), 50, 3)
    exp = O.reduce_csc(ptr, rows)
    for comp in (False, True):
        low, st = vr.hypha_pivots(ptr, rows, dims, compression=comp)
        assert np.array_equal(low, exp)
