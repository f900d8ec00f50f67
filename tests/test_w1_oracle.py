"""Pins for the W1 oracle (oracle/w1.py) against things other than itself (PAPER.md Ch.6).

A plausible mistake in the oracle — a missing diagonal term, the l∞ or l1 norm instead of
l2 (P:6438 insists on l2), a wrong projection distance, a matching that forbids leaving
points unmatched, a transposed cost block — fails at least one of:
closed forms, brute-force enumeration of partial matchings (Eq 6.36), metric axioms,
homogeneity / diagonal-translation invariance, Prop 6.2.3 (the transshipment LP of
Def 6.2.2 has the same optimum as the matching), and RWMD <= W1.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from datagen import diagrams as PD
from oracle import w1 as W

R2 = math.sqrt(2.0)


def test_closed_forms():
    p = np.array([[1.0, 3.0]])
    q = np.array([[1.5, 3.2]])
    far = np.array([[0.0, 10.0]])
    empty = np.zeros((0, 2))
    assert W.w1_exact(p, empty) == pytest.approx(2.0 / R2)         # one point to Δ
    assert W.w1_exact(empty, p) == pytest.approx(2.0 / R2)
    assert W.w1_exact(empty, empty) == 0.0
    assert W.w1_exact(p, p) == pytest.approx(0.0, abs=1e-12)
    # two points: matched (||p-q||) or both to the diagonal
    assert W.w1_exact(p, q) == pytest.approx(min(math.hypot(0.5, 0.2), 2.0 / R2 + 1.7 / R2))
    assert W.w1_exact(p, far) == pytest.approx(min(math.hypot(1.0, 7.0), 2.0 / R2 + 10.0 / R2))
    # near-diagonal points are cheaper to project than to match across the plane
    a = np.array([[0.0, 0.1]])
    b = np.array([[5.0, 5.1]])
    assert W.w1_exact(a, b) == pytest.approx(0.2 / R2)


@pytest.mark.parametrize("seed", range(12))
def test_brute_force(seed):
    rng = np.random.default_rng(seed)
    A = PD.uniform(int(rng.integers(0, 5)), seed)
    B = PD.uniform(int(rng.integers(0, 5)), seed + 100)
    assert W.w1_exact(A, B) == pytest.approx(W.w1_brute(A, B), rel=1e-9, abs=1e-12)


@pytest.mark.parametrize("seed", range(5))
def test_metric_axioms_and_invariances(seed):
    A, B, C = PD.gaussian(30, seed), PD.gaussian(25, seed + 50), PD.gaussian(20, seed + 99)
    ab, ba = W.w1_exact(A, B), W.w1_exact(B, A)
    assert ab == pytest.approx(ba, rel=1e-9)
    assert W.w1_exact(A, C) <= ab + W.w1_exact(B, C) + 1e-9
    assert W.w1_exact(3.0 * A.astype(np.float64), 3.0 * B.astype(np.float64)) == pytest.approx(3.0 * ab, rel=1e-9)
    t = np.array([0.7, 0.7])
    assert W.w1_exact(A + t, B + t) == pytest.approx(ab, rel=1e-9)


def _complete_network(A, B):
    """G(A, B) of Def 6.2.2 / P:6480-6484 without any sparsification (test helper)."""
    Au, sa = W.condense0(A)
    Bu, sb = W.condense0(B)
    na, nb = len(Au), len(Bu)
    # nodes: 0..na-1 = Â, na = b̄, na+1 .. na+nb = B̂, na+nb+1 = ā
    bbar, abar = na, na + nb + 1
    supply = np.concatenate([sa, [len(B)], -sb, [-len(A)]]).astype(np.float64)
    tail, head, cost = [], [], []
    for i in range(na):
        for j in range(nb):
            tail.append(i); head.append(na + 1 + j); cost.append(float(np.hypot(*(Au[i] - Bu[j]))))
        tail.append(i); head.append(abar); cost.append(float(W.d_diag(Au[i:i + 1])[0]))
    for j in range(nb):
        tail.append(bbar); head.append(na + 1 + j); cost.append(float(W.d_diag(Bu[j:j + 1])[0]))
    tail.append(bbar); head.append(abar); cost.append(0.0)
    return supply, np.array(tail), np.array(head), np.array(cost)


@pytest.mark.parametrize("seed", range(6))
def test_prop_6_2_3_flow_equals_matching(seed):
    A = PD.clustered(40, seed, levels=8) if seed % 2 else PD.gaussian(40, seed)
    B = PD.clustered(35, seed + 7, levels=8) if seed % 2 else PD.gaussian(35, seed + 7)
    s, t, h, c = _complete_network(A, B)
    assert W.min_cost_flow(s, t, h, c) == pytest.approx(W.w1_exact(A, B), rel=1e-9, abs=1e-9)


@pytest.mark.parametrize("seed", range(6))
def test_rwmd_is_a_lower_bound(seed):
    A, B = PD.gaussian(50, seed), PD.clustered(40, seed, levels=16)
    assert W.rwmd(A, B) <= W.w1_exact(A, B) + 1e-9
    p = np.array([[0.0, 1.0]])
    assert W.rwmd(p, np.zeros((0, 2))) == pytest.approx(W.w1_exact(p, np.zeros((0, 2))))


def test_generators_above_the_diagonal():
    for P in (PD.gaussian(1000, 1), PD.clustered(1000, 2), PD.uniform(100, 3)):
        assert P.dtype == np.float32 and np.all(P[:, 1] > P[:, 0])
    assert len(np.unique(PD.clustered(2000, 4), axis=0)) < 2000  # coinciding points exist


def test_rwmd_exact_values():
    """Alg 20 by hand: L_A = Σ_{u∈Â} σ(u)·min(min_v ||u−v||, d_Δ(u)), L_B
    likewise, RWMD = max(L_A, L_B).  Dropping the multiplicity σ, taking min(L_A, L_B)
    instead of the max, using d_Δ = |d−b| (no √2) or skipping the diagonal option each
    changes one of these values."""
    # multiplicities: three copies of (0, 4) against one (0, 3).  Â = {(0,4)} with σ = 3:
    # nearest is (0,3) at 1 < d_Δ = 4/√2, so L_A = 3·1 = 3; L_B = min(1, 3/√2) = 1
    A = np.array([[0.0, 4.0]] * 3)
    B = np.array([[0.0, 3.0]])
    assert W.rwmd(A, B) == pytest.approx(3.0, rel=1e-12)
    assert W.rwmd(B, A) == pytest.approx(3.0, rel=1e-12)
    # asymmetric: L_A = d_Δ((0,1)) = 1/√2 (the diagonal beats both B points);
    # L_B = min(9, 10/√2) + min(√386, 15/√2) = 10/√2 + 15/√2 = 25/√2 > L_A
    A = np.array([[0.0, 1.0]])
    B = np.array([[0.0, 10.0], [5.0, 20.0]])
    assert W.rwmd(A, B) == pytest.approx(25.0 / R2, rel=1e-12)
    # nearest neighbour beats the diagonal on both sides: L_A = L_B = 0.5
    assert W.rwmd(np.array([[1.0, 5.0]]), np.array([[1.5, 5.0]])) == pytest.approx(0.5, rel=1e-12)
    # σ(v) on the B side: two copies of (2, 2.5) (d_Δ = 0.5/√2) against (2, 9):
    # L_A = 2·0.5/√2 (diagonal), L_B = min(6.5, 7/√2) = 7/√2 = 4.95 > L_A
    A = np.array([[2.0, 2.5], [2.0, 2.5]])
    B = np.array([[2.0, 9.0]])
    assert W.rwmd(A, B) == pytest.approx(7.0 / R2, rel=1e-12)
    assert W.rwmd(B, A) == pytest.approx(7.0 / R2, rel=1e-12)
    # σ decides: four copies of (0, 2) against one (0.5, 2): L_A = 4·0.5 = 2 > L_B = 0.5
    A = np.array([[0.0, 2.0]] * 4)
    B = np.array([[0.5, 2.0]])
    assert W.rwmd(A, B) == pytest.approx(2.0, rel=1e-12)
