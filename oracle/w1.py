"""The CPU ORACLE for the PDoptFlow row — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and the cpu_baseline / reference legs of the bench
scripts may import this module.  The product (paper_2502_05063_b200, libvr.so) never does.

What it computes, each step citing PAPER.md:

* `w1_exact(A, B)` — the 1-Wasserstein distance between persistence diagrams with the
  l2 ground metric, Eq 6.36: the minimum over partial matchings M of
  Σ_{(x,y)∈M} ||x-y||_2 + Σ_{unmatched x} d_Δ(x), d_Δ(x) = the l2 distance of x to the
  diagonal = (d - b)/√2.  Written as the perfect matching on Bi(A, B) of Eq 6.37
  (P:6444-6448): rows Ã ∪ B̃_proj, columns B̃ ∪ Ã_proj, weights ||p-q|| (Ã×B̃),
  d_Δ(p) on (p, p_proj), d_Δ(q) on (q_proj, q), 0 on Ã_proj × B̃_proj, and no edge
  elsewhere.  The assignment itself is a library primitive
  (scipy.optimize.linear_sum_assignment), as the task allows.  fp64 throughout.
* `w1_brute(A, B)` — Eq 6.36 by enumerating every partial matching (tiny inputs only):
  an independent check of the construction above.
* `min_cost_flow(supply, tail, head, cost)` — Eq 6.38, the uncapacitated
  min-cost flow of a transshipment network (Def 6.2.2), as a linear program solved by a
  library LP solver (scipy.optimize.linprog, HiGHS): minimise Σ c_a f_a subject to
  Σ_out f - Σ_in f = σ(v) for every node v, f >= 0.
* `rwmd(A, B)` — Alg 20 on the 0-condensed diagrams by brute-force
  nearest neighbours: L_A = Σ_{u∈Â} σ(u) min(min_{v∈B̂} ||u-v||, d_Δ(u)), L_B likewise,
  return max(L_A, L_B).

Pins: tests/test_w1_oracle.py (closed forms, brute force, metric axioms, LP ≡ assignment).
"""
from __future__ import annotations

import itertools
import math

import numpy as np

SQRT2 = math.sqrt(2.0)


def d_diag(P: np.ndarray) -> np.ndarray:
    """l2 distance of each point (b, d) to the diagonal Δ: |d - b| / √2."""
    P = np.asarray(P, np.float64).reshape(-1, 2)
    return np.abs(P[:, 1] - P[:, 0]) / SQRT2


def _pairwise(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    A = np.asarray(A, np.float64).reshape(-1, 2)
    B = np.asarray(B, np.float64).reshape(-1, 2)
    return np.sqrt(((A[:, None, :] - B[None, :, :]) ** 2).sum(-1))


def w1_exact(A, B) -> float:
    """Eq 6.36 via the perfect matching on Bi(A, B) (Eq 6.37)."""
    from scipy.optimize import linear_sum_assignment
    A = np.asarray(A, np.float64).reshape(-1, 2)
    B = np.asarray(B, np.float64).reshape(-1, 2)
    n1, n2 = len(A), len(B)
    if n1 + n2 == 0:
        return 0.0
    dA, dB = d_diag(A), d_diag(B)
    big = 1e6 * (1.0 + max(dA.max(initial=0), dB.max(initial=0)) + (_pairwise(A, B).max(initial=0)))
    N = n1 + n2
    C = np.full((N, N), big)
    # rows 0..n1-1 = Ã, rows n1.. = B̃_proj ; columns 0..n2-1 = B̃, columns n2.. = Ã_proj
    if n1 and n2:
        C[:n1, :n2] = _pairwise(A, B)                     # (i) Ã × B̃: ||p - q||
    for i in range(n1):
        C[i, n2 + i] = dA[i]                              # (iii) (p, p_proj): d_Δ(p)
    for j in range(n2):
        C[n1 + j, j] = dB[j]                              # (iv) (q_proj, q): d_Δ(q)
    C[n1:, n2:] = 0.0                                     # (ii) Ã_proj × B̃_proj: 0
    r, c = linear_sum_assignment(C)
    total = float(C[r, c].sum())
    assert total < big, "infeasible assignment"
    return total


def w1_brute(A, B) -> float:
    """Eq 6.36 by enumerating all partial matchings (len(A), len(B) <= 5)."""
    A = np.asarray(A, np.float64).reshape(-1, 2)
    B = np.asarray(B, np.float64).reshape(-1, 2)
    dA, dB = d_diag(A), d_diag(B)
    D = _pairwise(A, B) if len(A) and len(B) else np.zeros((len(A), len(B)))
    best = math.inf
    # a partial matching = an injective map from a subset of A into B
    for k in range(0, min(len(A), len(B)) + 1):
        for sa in itertools.combinations(range(len(A)), k):
            for sb in itertools.permutations(range(len(B)), k):
                cost = sum(D[i, j] for i, j in zip(sa, sb))
                cost += sum(dA[i] for i in range(len(A)) if i not in sa)
                cost += sum(dB[j] for j in range(len(B)) if j not in sb)
                best = min(best, cost)
    return float(best)


def min_cost_flow(supply, tail, head, cost) -> float:
    """Eq 6.38 as an LP (HiGHS): min Σ c f, out - in = σ, f >= 0 (uncapacitated)."""
    from scipy.optimize import linprog
    from scipy.sparse import coo_matrix
    supply = np.asarray(supply, np.float64)
    tail = np.asarray(tail, np.int64)
    head = np.asarray(head, np.int64)
    cost = np.asarray(cost, np.float64)
    n, m = len(supply), len(tail)
    rows = np.concatenate([tail, head])
    cols = np.concatenate([np.arange(m), np.arange(m)])
    vals = np.concatenate([np.ones(m), -np.ones(m)])
    Aeq = coo_matrix((vals, (rows, cols)), shape=(n, m)).tocsr()
    # HiGHS' default feasibility tolerances (1e-7) are coarser than the 1e-9 parity bar
    res = linprog(cost, A_eq=Aeq, b_eq=supply, bounds=(0, None), method="highs",
                  options={"primal_feasibility_tolerance": 1e-10, "dual_feasibility_tolerance": 1e-10})
    if res.status != 0:
        raise ValueError(f"min-cost flow LP failed: {res.message}")
    return float(res.fun)


def condense0(P):
    """0-condensation: identical points become one node with their count."""
    P = np.asarray(P, np.float64).reshape(-1, 2)
    if len(P) == 0:
        return P, np.zeros(0, np.int64)
    u, cnt = np.unique(P, axis=0, return_counts=True)
    return u, cnt


def rwmd(A, B) -> float:
    """Alg 20 on the 0-condensed diagrams, nearest neighbours by brute force."""
    Au, sa = condense0(A)
    Bu, sb = condense0(B)

    def side(U, su, V):
        if len(U) == 0:
            return 0.0
        best = d_diag(U)
        if len(V):
            best = np.minimum(best, _pairwise(U, V).min(1))
        return float((su * best).sum())

    return max(side(Au, sa, Bu), side(Bu, sb, Au))
