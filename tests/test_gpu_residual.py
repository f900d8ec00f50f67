"""The host residual reduction's inputs from the device and its parallel schedule.

* residual hints (csrc/residual_prep.cu): per residual column, the first equal-diameter
  cofacet and whether it is apparent-claimed, which the host's emergent test (§5.2.11,
  P:4874-4888) uses instead of its own scan.  VR_CHECK_HINTS=1 makes the library recompute
  them with the host's scans (host.cpp, an independent implementation) and fail on any
  difference; VR_NO_RESIDUAL_HINTS=1 runs the host test itself — the barcode, the pairing
  and the counters must not change.
* the in-order-commit parallel reduction: any block size and thread count gives the
  sequential algorithm's pivots (the pairing is unique), checked against the
  oracle where it is feasible and against one thread elsewhere.
* the output-sensitive host graph (bitmap rows + packed neighbour ranks, no n x n copy).
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2502_05063_b200 as vr
from datagen import clouds as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _quant(n, seed, levels=16):
    lt = G.random_cloud(n, seed)
    return (np.round(lt * levels / lt.max()) / levels).astype(np.float32)


def _same(a, b, D):
    for d in range(D + 1):
        assert np.array_equal(a.pairs[d].view(np.uint32), b.pairs[d].view(np.uint32)), d
        assert {tuple(x) for x in a.index_pairs[d].tolist()} == {tuple(x) for x in b.index_pairs[d].tolist()}, d
        for k in ("survivors", "apparent", "cleared", "residual_columns", "emergent", "pairs_all", "essential"):
            assert a.stats[d][k] == b.stats[d][k], (d, k)


CASES = [  # (name, n, D, threshold quantile or None = enclosing radius, sparse_mode)
    ("cloud", 150, 3, 0.08, 2), ("quant", 150, 3, 0.10, 2), ("cloud", 300, 2, 0.05, 2),
    ("cloud", 60, 3, None, 1), ("quant", 90, 3, None, 1), ("tied", 70, 2, None, 1),
]


def _input(kind, n, seed):
    if kind == "cloud":
        return G.random_cloud(n, seed)
    if kind == "quant":
        return _quant(n, seed)
    return G.random_tied(n, seed, levels=4)


def _t(lt, n, q):
    return O.enclosing_radius(lt, n) if q is None else float(np.quantile(lt, q))


@pytest.mark.parametrize("kind,n,D,q,mode", CASES)
def test_hints_match_host_scans(kind, n, D, q, mode, monkeypatch):
    lt = _input(kind, n, 900 + n + D)
    t = _t(lt, n, q)
    ref = vr.barcodes(lt, n, D, t, index_pairs=True, sparse_mode=mode)
    monkeypatch.setenv("VR_CHECK_HINTS", "1")  # raises inside the library on a mismatch
    got = vr.barcodes(lt, n, D, t, index_pairs=True, sparse_mode=mode)
    _same(ref, got, D)
    monkeypatch.delenv("VR_CHECK_HINTS")
    monkeypatch.setenv("VR_NO_RESIDUAL_HINTS", "1")
    _same(ref, vr.barcodes(lt, n, D, t, index_pairs=True, sparse_mode=mode), D)


@pytest.mark.parametrize("block,threads", [(1, 16), (3, 4), (32, 16), (1000, 2)])
def test_block_commit_schedules_vs_oracle(block, threads, monkeypatch):
    n, D = 14, 3
    lt = G.random_tied(n, 77, levels=3)  # ties: many emergent and residual columns
    t = O.enclosing_radius(lt, n)
    monkeypatch.setenv("VR_RESIDUAL_BLOCK", str(block))
    monkeypatch.setenv("VR_RESIDUAL_THREADS", str(threads))
    got = vr.barcodes(lt, n, D, t, index_pairs=True)
    ref = O.barcode(lt, n, D, got.threshold)
    for d in range(D + 1):
        assert np.array_equal(got.pairs[d].view(np.uint32), ref.positive(d).view(np.uint32)), d
        assert {(int(a), int(b)) for a, b in got.index_pairs[d]} == ref.index_pairs(d), d


@pytest.mark.parametrize("block,threads", [(1, 16), (5, 8), (64, 16)])
def test_block_commit_schedules_equal_one_thread(block, threads, monkeypatch):
    # config 5's shape at a size with thousands of residual columns per dimension
    cfg = G.CONFIGS["c5_o3_4096"]
    lt = cfg.patch(1200)  # the full cloud's density (a first-n subsample is nearly empty at t)
    monkeypatch.setenv("VR_RESIDUAL_THREADS", "1")
    a = vr.barcodes(lt, 1200, 3, cfg.threshold, index_pairs=True)
    assert a.stats[3]["residual_columns"] > 1000
    monkeypatch.setenv("VR_RESIDUAL_BLOCK", str(block))
    monkeypatch.setenv("VR_RESIDUAL_THREADS", str(threads))
    _same(a, vr.barcodes(lt, 1200, 3, cfg.threshold, index_pairs=True), 3)
