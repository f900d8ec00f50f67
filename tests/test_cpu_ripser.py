"""The single-threaded Ripser-style CPU run (cpu_ripser/, BASELINE.json north_star's
"single-threaded Ripser-style CPU run") — a timed baseline, checked here so its timings
are of a correct program.

* CPU: bit-exact positive bars against the oracle (explicit boundary matrix + Alg 2) on
  random clouds, integer-valued matrices with heavy ties, and thresholds below R;
* GPU: bit-exact bars against the library on config 4a (max_dim 2) and config 1.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import cpu_ripser as RS
from datagen import clouds as G
from oracle import oracle as O


def _case(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 17))
    D = int(rng.integers(1, 4))
    if seed % 3 == 0:
        lt = rng.integers(1, 6, n * (n - 1) // 2).astype(np.float32)  # heavy ties
    else:
        lt = G.random_cloud(n, seed)
    thr = math.inf if seed % 2 else float(np.quantile(lt, 0.7))
    return lt, n, D, thr


@pytest.mark.parametrize("seed", range(48))
def test_equals_oracle(seed):
    lt, n, D, thr = _case(seed)
    ob = O.barcode(lt, n, D, thr)
    got, st = RS.barcode(lt, n, D, thr)
    for d in range(D + 1):
        np.testing.assert_array_equal(got[d], ob.positive(d))
    # every d-simplex under the threshold is counted (n_d of the oracle)
    for d in range(1, D + 1):
        assert st[d]["simplices"] == ob.n_simplices[d]


def test_circle_and_sierpinski_sample_equal_oracle():
    for name, m, D in (("c1_circle64", 64, 1), ("c4a_sierpinski512", 40, 2)):
        cfg = G.CONFIGS[name]
        lt = cfg.lower_tri(m)
        R = O.enclosing_radius(lt, m)
        ob = O.barcode(lt, m, D, R)
        got, _ = RS.barcode(lt, m, D, R)
        for d in range(D + 1):
            np.testing.assert_array_equal(got[d], ob.positive(d))


def test_emergent_shortcut_taken_and_counts_add_up():
    cfg = G.CONFIGS["c2_s3_192"]
    lt = cfg.lower_tri(60)
    R = O.enclosing_radius(lt, 60)
    _, st = RS.barcode(lt, 60, 2, R)
    for d in (1, 2):
        assert st[d]["emergent"] + st[d]["reduced"] == st[d]["columns"]
        assert st[d]["emergent"] > 0.9 * st[d]["columns"]  # the §5.2.7 shortcut does the bulk


def _sorted(a):
    a = np.asarray(a, np.float32).reshape(-1, 2)
    return a[np.lexsort((a[:, 1], a[:, 0]))] if len(a) else a


@pytest.mark.gpu
@pytest.mark.parametrize("name,D", [("c1_circle64", 1), ("c4a_sierpinski512", 2)])
def test_equals_library(name, D):
    import paper_2502_05063_b200 as vr
    cfg = G.CONFIGS[name]
    lt = cfg.lower_tri()
    bc = vr.barcodes(lt, cfg.n, D, cfg.threshold)
    got, _ = RS.barcode(lt, cfg.n, D, bc.threshold)
    for d in range(D + 1):
        np.testing.assert_array_equal(_sorted(got[d]), _sorted(bc.pairs[d]))


@pytest.mark.parametrize("seed", range(6))
def test_sparse_mode_equals_oracle(seed):
    # thresholds keeping <= 1/4 of the edges at n > 64 switch cpu_ripser to neighbour lists
    n, D = 72 + seed, 1 + seed % 3
    lt = G.random_cloud(n, 40 + seed) if seed % 2 else (np.round(G.random_cloud(n, 40 + seed) * 8) / 8).astype(np.float32)
    thr = float(np.quantile(lt, 0.12 if D == 3 else 0.2))
    ob = O.barcode(lt, n, D, thr)
    got, st = RS.barcode(lt, n, D, thr)
    for d in range(D + 1):
        np.testing.assert_array_equal(got[d], ob.positive(d))
    for d in range(1, D + 1):
        assert st[d]["simplices"] == ob.n_simplices[d]
