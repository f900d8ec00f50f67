"""PDoptFlow (PAPER.md Ch.6, Alg 22) against the W1 oracle.

* exact mode (complete network) = Eq 6.36 by assignment, to 1e-9;
* the library's network simplex on the network the library builds = the LP optimum of
  the same network (HiGHS), to 1e-9 — at every s;
* approximate mode inside the guaranteed band bound_lo·W1 <= w1 <= bound_hi·W1
  (Prop 6.3.2 × Thm 6.3.6);
* the spanner: every pair of network points joined by a path of length <= t·||p - q||,
  t = (s+4)/(s-4);
* RWMD (Alg 20) = the oracle's; supplies = the 0-condensed multiplicities; δ-snapping
  moves no point farther than √2·δ/2 (proof of Prop 6.3.2).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from datagen import diagrams as PD
from oracle import w1 as W

pytestmark = pytest.mark.gpu


def _vr():
    import paper_2502_05063_b200 as vr
    return vr


def _pairs(seed):
    kinds = [(PD.gaussian, PD.gaussian), (PD.clustered, PD.clustered), (PD.gaussian, PD.clustered), (PD.uniform, PD.uniform)]
    fa, fb = kinds[seed % len(kinds)]
    rng = np.random.default_rng(seed)
    na, nb = int(rng.integers(1, 160)), int(rng.integers(1, 160))
    return fa(na, seed), fb(nb, seed + 1000)


@pytest.mark.parametrize("seed", range(12))
def test_exact_mode_equals_oracle(seed):
    A, B = _pairs(seed)
    got, st = _vr().w1(A, B, exact=True)
    assert st["optimal"] == 1
    assert got == pytest.approx(W.w1_exact(A, B), rel=1e-9, abs=1e-12)


def test_exact_mode_edge_cases():
    vr = _vr()
    e = np.zeros((0, 2), np.float32)
    p = np.array([[1.0, 3.0]], np.float32)
    assert vr.w1(e, e, exact=True)[0] == 0.0
    assert vr.w1(p, e, exact=True)[0] == pytest.approx(2.0 / math.sqrt(2.0))
    assert vr.w1(e, p, exact=True)[0] == pytest.approx(2.0 / math.sqrt(2.0))
    A = PD.gaussian(50, 3)
    assert vr.w1(A, A, exact=True)[0] == pytest.approx(0.0, abs=1e-12)
    assert vr.w1(A, A, s=18)[0] == pytest.approx(0.0, abs=1e-12)
    with pytest.raises(Exception):
        vr.w1(np.array([[0.0, np.inf]], np.float32), p)


@pytest.mark.parametrize("s", [0.0, 1.0, 6.0, 18.0])
@pytest.mark.parametrize("seed", range(4))
def test_simplex_equals_lp_on_the_built_network(s, seed):
    vr = _vr()
    A, B = _pairs(seed + 20)
    net = vr.w1_network(A, B, s=s, seed=seed, exact=(s == 0.0))
    assert net["supply"].sum() == 0
    assert net["supply"][-2] == -len(A) and net["supply"][-1] == len(B)
    lp = W.min_cost_flow(net["supply"], net["tail"], net["head"], net["cost"])
    ns, st = vr.min_cost_flow(net["supply"], net["tail"], net["head"], net["cost"])
    assert st["optimal"] == 1
    assert ns == pytest.approx(lp, rel=1e-9, abs=1e-12)
    got, _ = vr.w1(A, B, s=s, seed=seed, exact=(s == 0.0))
    assert got == pytest.approx(lp, rel=1e-9, abs=1e-12)


@pytest.mark.parametrize("s", [12.0, 18.0, 40.0])
@pytest.mark.parametrize("seed", range(4))
def test_approximation_band(s, seed):
    A = PD.gaussian(300 + 50 * seed, seed) if seed % 2 == 0 else PD.clustered(400, seed)
    B = PD.gaussian(280 + 40 * seed, seed + 7) if seed % 2 == 0 else PD.clustered(380, seed + 7)
    exact = W.w1_exact(A, B)
    got, st = _vr().w1(A, B, s=s, seed=seed)
    assert st["optimal"] == 1
    assert st["bound_lo"] * exact - 1e-9 <= got <= st["bound_hi"] * exact + 1e-9, (got, exact, st)
    assert st["rwmd"] <= exact + 1e-9
    # without δ-condensation only the spanner factor remains (Thm 6.3.6)
    got2, st2 = _vr().w1(A, B, s=s, seed=seed, condense=False)
    assert exact - 1e-9 <= got2 <= (1 + st2["eps_spanner"]) * exact + 1e-9


@pytest.mark.parametrize("s", [5.0, 8.0, 18.0])
def test_spanner_stretch(s):
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import shortest_path
    A, B = PD.gaussian(120, 11), PD.gaussian(100, 12)
    net = _vr().w1_network(A, B, s=s, condense=False)
    xy = net["xy"][:-2]
    N = len(xy)
    real = (net["tail"] < N) & (net["head"] < N)
    t, h, c = net["tail"][real], net["head"][real], net["cost"][real]
    G = coo_matrix((c, (t, h)), shape=(N, N)).tocsr()
    sp = shortest_path(G, directed=False)
    direct = np.sqrt(((xy[:, None, :] - xy[None, :, :]) ** 2).sum(-1))
    iu = np.triu_indices(N, 1)
    stretch = (sp[iu] / direct[iu]).max()
    assert stretch <= (s + 4) / (s - 4) + 1e-9
    assert np.allclose(c, np.hypot(*(xy[t] - xy[h]).T))  # arc costs are l2 lengths


@pytest.mark.parametrize("seed", range(4))
def test_rwmd_supplies_and_snapping(seed):
    vr = _vr()
    A, B = PD.clustered(300, seed, levels=32), PD.gaussian(250, seed + 5)
    _, st = vr.w1(A, B, s=18, seed=seed)
    assert st["rwmd"] == pytest.approx(W.rwmd(A, B), rel=1e-9)
    # exact-mode nodes: the 0-condensed points, supply = #A - #B at each location
    net = vr.w1_network(A, B, exact=True)
    Au, ca = W.condense0(A)
    Bu, cb = W.condense0(B)
    want = {}
    for p, k in zip(map(tuple, Au), ca):
        want[p] = want.get(p, 0) + int(k)
    for p, k in zip(map(tuple, Bu), cb):
        want[p] = want.get(p, 0) - int(k)
    got = {tuple(p): int(k) for p, k in zip(net["xy"][:-2], net["supply"][:-2])}
    assert got == want
    # δ-condensed nodes: every input point within √2·δ/2 of some node of its cell
    net = vr.w1_network(A, B, s=18, seed=seed)
    d = net["stats"]["delta"]
    assert d > 0 and net["stats"]["condensed"] == 1
    xy = net["xy"][:-2]
    P = np.concatenate([A, B]).astype(np.float64)
    dist = np.sqrt(((P[:, None, :] - xy[None, :, :]) ** 2).sum(-1)).min(1)
    assert dist.max() <= math.sqrt(2) * d / 2 + 1e-12
    assert net["supply"][:-2].sum() == len(A) - len(B)


@pytest.mark.parametrize("seed", range(3))
def test_warm_diagonal_start(seed):
    A, B = _pairs(seed + 40)
    a, st = _vr().w1(A, B, s=6, seed=seed, warm=True)
    b, _ = _vr().w1(A, B, s=6, seed=seed)
    assert st["warm_start"] == 1
    assert a == pytest.approx(b, rel=1e-9, abs=1e-12)


def test_determinism_and_seeds():
    vr = _vr()
    A, B = PD.gaussian(400, 1), PD.gaussian(350, 2)
    a1, _ = vr.w1(A, B, s=18, seed=5)
    a2, _ = vr.w1(A, B, s=18, seed=5)
    assert a1 == a2
    exact = W.w1_exact(A, B)
    for sd in (1, 2, 3):
        v, st = vr.w1(A, B, s=18, seed=sd)
        assert st["bound_lo"] * exact - 1e-9 <= v <= st["bound_hi"] * exact + 1e-9


def test_w1_between_vr_barcodes():
    # W1 between the diagrams the library produces — the H1
    # diagrams of two noisy circles (config-1-shaped) — exact and approximate, vs the oracle
    from datagen import clouds as G
    vr = _vr()
    rng = np.random.default_rng(4)
    diags = []
    for k in range(2):
        th = rng.random(80) * 2 * np.pi
        pts = np.stack([np.cos(th), np.sin(th)], 1) + rng.normal(0, 0.08 + 0.04 * k, (80, 2))
        lt = G.lower_tri_from_points(pts)
        bc = vr.barcodes(lt, 80, 1)
        diags.append(np.concatenate([bc.pairs[0][np.isfinite(bc.pairs[0][:, 1])], bc.pairs[1]]))
    A, B = diags
    exact = W.w1_exact(A, B)
    got, _ = vr.w1(A, B, exact=True)
    assert got == pytest.approx(exact, rel=1e-9, abs=1e-12)
    v, st = vr.w1(A, B, s=18)
    assert st["bound_lo"] * exact - 1e-9 <= v <= st["bound_hi"] * exact + 1e-9
