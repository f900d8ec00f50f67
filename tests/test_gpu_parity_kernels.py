"""GPU parity of each enumeration kernel against the CPU oracle, element by element.

The dense path has two kernels (hotpath.cu): the row kernel `k_enumerate` and the
flattened-chunk kernel `k_enumerate_flat` (dimensions >= 2 at 32 <= n <= 544, and dimension
1 from n = 128 on), both with the scan window in shared memory; the output-sensitive path
has `k_enum_sparse` (threshold-graph bitmap rows).  `vr_stats.kernels` says which ran, so
every case below first asserts that the kernel it means to test is the one that ran, then
compares with the oracle (explicit boundary matrix + Alg 2): the fp32 bars per dimension,
the full index-level pairing (every apparent, residual and dimension-0 pair; unique for the
§5.1.4 refinement, Thm 3.2.20) and the counts.  Inputs: random clouds and
heavily tied integer metrics (ties exercise the `== diam` branches of Lemma 5.3.6's
condition 2), thresholds R and distance quantiles.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2502_05063_b200 as vr
from datagen import clouds as G
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _input(kind, n, seed):
    if kind == "cloud":
        return G.random_cloud(n, seed)
    if kind.startswith("quant"):  # a cloud with its distances on a grid of `levels` values:
        # heavy ties, yet geometric (short residual reductions at any n)
        lt = G.random_cloud(n, seed)
        levels = int(kind[5:])
        return (np.round(lt * levels / lt.max()) / levels).astype(np.float32)
    return G.random_tied(n, seed, levels={"tied3": 3, "tied5": 5, "tied8": 8}[kind])


def _threshold(lt, n, thr):
    if thr == "R":
        return O.enclosing_radius(lt, n)
    return float(np.quantile(lt, float(thr[1:]) / 100.0))


def _check(lt, n, D, t, want_kernel, dims, **opts):
    got = vr.barcodes(lt, n, D, t, index_pairs=True, **opts)
    for d in dims:
        assert got.stats[d]["kernels"] & want_kernel, (d, got.stats[d]["kernels"])
    ref = O.barcode(lt, n, D, got.threshold)
    for d in range(D + 1):
        exp = ref.positive(d)
        assert np.array_equal(got.pairs[d].view(np.uint32), exp.view(np.uint32)), d
        g = {(int(a), int(b)) for a, b in got.index_pairs[d]}
        assert len(g) == len(got.index_pairs[d])
        assert g == ref.index_pairs(d), d
        s = got.stats[d]
        assert s["pairs_all"] == ref.num_pairs_all(d), d
        assert s["essential"] == ref.num_essential(d), d
        if d >= 1:
            assert s["survivors"] == ref.n_simplices[d], d
    return got


# k_enumerate_flat<3> (and <2>): n = 33..40 at max_dim 3, oracle-feasible
FLAT3 = [(n, kind, thr, seed) for seed, (n, kind, thr) in enumerate(
    [(n, kind, thr) for n in (33, 36, 40) for kind in ("cloud", "tied3", "tied8", "quant16") for thr in ("R", "q55")])]


@pytest.mark.parametrize("n,kind,thr,seed", FLAT3)
def test_flat_dim3_vs_oracle(n, kind, thr, seed):
    lt = _input(kind, n, 100 + seed)
    _check(lt, n, 3, _threshold(lt, n, thr), vr.KERNEL_FLAT, dims=(2, 3), sparse_mode=1)


# k_enumerate_flat<1>: n = 128..140 at max_dim 1, thresholded
FLAT1 = [(n, kind, thr, seed) for seed, (n, kind, thr) in enumerate(
    [(n, kind, thr) for n in (128, 133, 140) for kind in ("cloud", "tied3", "quant16") for thr in ("R", "q30", "q50")])]


@pytest.mark.parametrize("n,kind,thr,seed", FLAT1)
def test_flat_dim1_vs_oracle(n, kind, thr, seed):
    lt = _input(kind, n, 200 + seed)
    _check(lt, n, 1, _threshold(lt, n, thr), vr.KERNEL_FLAT, dims=(1,), sparse_mode=1)


# k_enumerate_flat<2> at sizes spanning several chunks and a ragged tail, tied
@pytest.mark.parametrize("n,kind", [(64, "tied3"), (70, "tied8"), (90, "cloud")])
def test_flat_dim2_vs_oracle(n, kind):
    lt = _input(kind, n, 300 + n)
    _check(lt, n, 2, _threshold(lt, n, "q40"), vr.KERNEL_FLAT, dims=(2,), sparse_mode=1)


# the row kernel with the shared-memory window (n in [32, 128) at dimension 1)
@pytest.mark.parametrize("n,kind,thr", [(32, "tied3", "R"), (57, "cloud", "q60"), (100, "tied8", "R")])
def test_row_kernel_window_dim1_vs_oracle(n, kind, thr):
    lt = _input(kind, n, 400 + n)
    _check(lt, n, 1, _threshold(lt, n, thr), vr.KERNEL_ROW | vr.KERNEL_SMEM_WINDOW, dims=(1,), sparse_mode=1)


# k_enum_sparse / k_enum_sparse2: the bitmap rows over several words (n > 32, ragged n % 32)
# at every dimension, tied and untied, with and without the clearing set (hash + Bloom)
@pytest.mark.parametrize("n,D,kind,thr", [(45, 3, "tied3", "q50"), (45, 3, "cloud", "q60"), (70, 2, "tied5", "q35"),
                                          (70, 2, "cloud", "R"), (150, 1, "tied8", "q20"), (97, 2, "tied3", "q25")])
@pytest.mark.parametrize("hashset", [False, True])
@pytest.mark.parametrize("levels", [1, 2])
def test_sparse_kernel_vs_oracle(n, D, kind, thr, hashset, levels, monkeypatch):
    # levels = 2: dimensions >= 2 on k_enum_sparse2 (rows = survivors of d-2, two vertices
    # added); 1: every dimension on k_enum_sparse (rows = survivors of d-1)
    if hashset:
        monkeypatch.setenv("VR_FORCE_CLEAR_HASH", "1")
    if levels == 1:
        monkeypatch.setenv("VR_SPARSE_1LEVEL", "1")
    lt = _input(kind, n, 500 + n + D)
    _check(lt, n, D, _threshold(lt, n, thr), vr.KERNEL_SPARSE, dims=range(1, D + 1), sparse_mode=2)


# the output-sensitive kernels on rows whose C(σ) lists pass SP_LCAP = 256 entries (the
# segmented path, dense graphs) against the dense kernels (pinned to the oracle above) —
# the oracle itself is not feasible at these sizes
@pytest.mark.parametrize("n,D,kind,thr", [(300, 1, "cloud", "R"), (300, 2, "quant16", "q95"), (400, 3, "cloud", "q12")])
@pytest.mark.parametrize("levels", [1, 2])
def test_sparse_long_lists_equal_dense(n, D, kind, thr, levels, monkeypatch):
    lt = _input(kind, n, 700 + n + D)
    t = _threshold(lt, n, thr)
    a = vr.barcodes(lt, n, D, t, index_pairs=True, sparse_mode=1)
    if levels == 1:
        monkeypatch.setenv("VR_SPARSE_1LEVEL", "1")
    b = vr.barcodes(lt, n, D, t, index_pairs=True, sparse_mode=2)
    for d in range(1, D + 1):
        assert b.stats[d]["kernels"] & vr.KERNEL_SPARSE, d
    for d in range(D + 1):
        assert np.array_equal(a.pairs[d], b.pairs[d])
        assert {tuple(x) for x in a.index_pairs[d].tolist()} == {tuple(x) for x in b.index_pairs[d].tolist()}
        for k in ("survivors", "apparent", "cleared", "residual_columns", "pairs_all", "essential"):
            assert a.stats[d][k] == b.stats[d][k], (d, k)


# ADVICE (round 1): ties through the window kernels at the sizes where they run, flat
# against the row kernel (VR_NO_FLAT) at index level — the oracle is not feasible there.
# Quantized clouds: 16-32 distinct distances (random integer metrics this large make the
# host residual reduction take minutes)
@pytest.mark.parametrize("n,D", [(128, 1), (128, 2), (128, 3), (300, 1), (300, 2), (544, 1), (544, 2)])
@pytest.mark.parametrize("kind,thr", [("quant16", "R"), ("quant32", "q45")])
def test_flat_equals_row_kernel_tied(n, D, kind, thr, monkeypatch):
    lt = _input(kind, n, 600 + n + D)
    t = _threshold(lt, n, thr)
    a = vr.barcodes(lt, n, D, t, index_pairs=True, sparse_mode=1)
    for d in range(1, D + 1):
        assert a.stats[d]["kernels"] & vr.KERNEL_FLAT, d
    monkeypatch.setenv("VR_NO_FLAT", "1")
    b = vr.barcodes(lt, n, D, t, index_pairs=True, sparse_mode=1)
    for d in range(1, D + 1):
        assert b.stats[d]["kernels"] & vr.KERNEL_ROW, d
    for d in range(D + 1):
        assert np.array_equal(a.pairs[d], b.pairs[d])
        assert {tuple(x) for x in a.index_pairs[d].tolist()} == {tuple(x) for x in b.index_pairs[d].tolist()}
        for k in ("survivors", "apparent", "cleared", "residual_columns"):
            assert a.stats[d][k] == b.stats[d][k], (d, k)


# Thm 5.4.2 at sizes where the flat kernels run: in the all-equal metric the
# dimension-d apparent count is C(n-1, d+1)
@pytest.mark.parametrize("n", [128, 200])
def test_thm542_all_equal_flat(n):
    got = vr.barcodes(G.all_equal(n), n, 2, 1.0, sparse_mode=1)
    for d in (1, 2):
        assert got.stats[d]["kernels"] & vr.KERNEL_FLAT
        assert got.stats[d]["apparent"] == math.comb(n - 1, d + 1)
