"""Pins for the CPU oracle (oracle/vr_oracle.c) against things other than itself.

Each pin is chosen so that a plausible mistake in the oracle (a dropped term, a wrong
sign or index, a transposed operand, a wrong tie-break, a wrong threshold comparison)
fails at least one of them:

* worked examples the paper prints (tests/golden/, each with its PAPER.md citation);
* closed forms (unit square, cross-polytopes, regular n-gons, full-Rips pair counts);
* the persistent Betti numbers rank(H_p(K_r) -> H_p(K_s)) computed by an independent
  Gaussian elimination over Z/2 (no reduction algorithm, no pairing) — they determine
  the barcode uniquely, so they pin every bar of every tiny input;
* invariants: the birth/death count identity n_p = P_p + E_p + P_{p-1}, Prop 5.2.13
  (threshold R), Obs 5.6.8 (monotone re-map), apparent pairs are persistence pairs.
"""
from __future__ import annotations

import itertools
import math
import os

import numpy as np
import pytest

from datagen import clouds as G
from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
F32_SQRT2 = np.float32(math.sqrt(2.0))


# ------------------------------------------------------------------ worked examples
def test_fig41_standard_reduction_pivots():
    cols, piv = [], set()
    for line in open(os.path.join(GOLDEN, "fig4_1_boundary.txt")):
        f = line.split()
        if not f or f[0].startswith("#"):
            continue
        if f[0] == "col":
            cols.append([int(x) for x in f[2:]])
        elif f[0] == "pivot":
            piv.add((int(f[1]), int(f[2])))
    low = O.reduce_columns(cols)
    got = {(lo, j) for j, lo in enumerate(low) if lo >= 0}
    assert got == piv  # P:4187 "the pivots are (2,3), (1,4), and (5,6)"
    # Fig 4.2(a): column 5 is zeroed by the reduction (P:4185 narration)
    assert low[5] == -1


def test_fig51_unit_square():
    pts, bars = [], {0: [], 1: []}
    for line in open(os.path.join(GOLDEN, "fig5_1_unit_square.txt")):
        f = line.split()
        if not f or f[0].startswith("#"):
            continue
        if f[0] == "point":
            pts.append([float(f[1]), float(f[2])])
        else:
            bars[int(f[1])].append((np.float32(f[2]), np.float32(float(f[3]))))
    lt = G.lower_tri_from_points(np.array(pts))
    b = O.barcode(lt, 4, 1)
    for d in (0, 1):
        assert [tuple(x) for x in b.positive(d).tolist()] == sorted(bars[d])
    assert b.positive(1)[0, 1] == F32_SQRT2


def test_fig55_all_equal_apparent_set():
    exp = {}
    for line in open(os.path.join(GOLDEN, "fig5_5_apparent.txt")):
        f = line.split()
        if not f or f[0].startswith("#"):
            continue
        v1, v0, app = int(f[1]), int(f[2]), int(f[3])
        cidx = math.comb(v1, 2) + v0
        partner = None
        if app:
            a, b, c = (int(x) for x in f[4:7])
            partner = math.comb(a, 3) + math.comb(b, 2) + c
        exp[cidx] = (bool(app), partner)
    c, flag, partner = O.apparent(G.all_equal(5), 5, 1)
    got = {int(ci): (bool(fl), int(p) if fl else None) for ci, fl, p in zip(c, flag, partner)}
    assert got == exp


@pytest.mark.parametrize("n", [5, 6, 7])
def test_fig56_distinct_diameters_keep_apparent_set(n):
    # §5.4.3: assigning decreasing distances along the increasing lex order
    # keeps exactly the all-equal apparent set (d = 1)
    c1, f1, _ = O.apparent(G.all_equal(n), n, 1)
    c2, f2, _ = O.apparent(G.fig56_lex_decreasing(n), n, 1)
    assert (c1 == c2).all() and (f1 == f2).all()
    assert f2.sum() == math.comb(n - 1, 2)


@pytest.mark.parametrize("n,d", [(n, d) for n in range(4, 13) for d in (1, 2)] + [(8, 3), (9, 3)])
def test_thm542_all_equal_apparent_count(n, d):
    # Thm 5.4.2 tightness: all diameters equal -> C(n-1, d+1) apparent
    _, f, _ = O.apparent(G.all_equal(n), n, d)
    assert f.sum() == math.comb(n - 1, d + 1)


def test_table51_closed_forms():
    # The full-Rips pair-count identity reproduces the paper's printed Table 5.1/5.5
    # numbers; the same identity is then checked on the oracle below.
    for line in open(os.path.join(GOLDEN, "table5_1_all_pairs.txt")):
        f = line.split()
        if not f or f[0].startswith("#"):
            continue
        name, n, d, allp, poss, tored, rem, clr = f[0], *map(int, f[1:])
        assert sum(math.comb(n - 1, p + 1) for p in range(1, d + 1)) == allp
        possible = sum(math.comb(n, p + 1) for p in range(1, d + 1))
        assert tored + rem + clr == possible
        if name != "sphere_3_192":  # printed typo, reading A13
            assert poss == possible


# ------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("k", [2, 3, 4])
def test_cross_polytope(k):
    b = O.barcode(G.cross_polytope(k), 2 * k, k - 1)
    h0 = b.positive(0)
    assert len(h0) == 2 * k and (h0[:-1, 1] == F32_SQRT2).all() and np.isinf(h0[-1, 1])
    for p in range(1, k - 1):
        assert len(b.positive(p)) == 0
    top = b.positive(k - 1)
    assert top.tolist() == [[F32_SQRT2, 2.0]]


@pytest.mark.parametrize("n", range(6, 13))
def test_regular_ngon_one_long_bar(n):
    b = O.barcode(G.regular_ngon(n), n, 1)
    h1 = b.positive(1)
    long = h1[(h1[:, 1] - h1[:, 0]) > 1e-3]
    assert len(long) == 1
    birth, death = float(long[0, 0]), float(long[0, 1])
    assert birth == pytest.approx(2 * math.sin(math.pi / n), rel=1e-6)
    assert death == pytest.approx(2 * math.sin(math.pi * math.ceil(n / 3) / n), rel=1e-6)


@pytest.mark.parametrize("seed", range(6))
def test_full_rips_pair_counts(seed):
    n, D = 7 + seed % 3, 2
    lt = G.random_cloud(n, seed) if seed % 2 else G.random_tied(n, seed)
    b = O.barcode(lt, n, D)
    assert b.num_pairs_all(0) == n - 1 and b.num_essential(0) == 1
    for p in range(1, D + 1):
        assert b.num_pairs_all(p) == math.comb(n - 1, p + 1)
        assert b.num_essential(p) == 0


@pytest.mark.parametrize("seed", range(12))
def test_count_identity_and_euler(seed):
    # n_p = P_p + E_p + P_{p-1} (birth/death partition), hence the Euler form
    n, D = 6 + seed % 4, 1 + seed % 3
    lt = G.random_tied(n, seed, levels=5) if seed % 2 else G.random_cloud(n, seed)
    t = float(np.quantile(lt, [0.3, 0.6, 1.0][seed % 3]))
    b = O.barcode(lt, n, D, t)
    P = [b.num_pairs_all(p) for p in range(D + 1)]
    E = [b.num_essential(p) for p in range(D + 1)]
    for p in range(D + 1):
        assert b.n_simplices[p] == P[p] + E[p] + (P[p - 1] if p else 0)
    lhs = sum((-1) ** p * b.n_simplices[p] for p in range(D + 1))
    rhs = sum((-1) ** p * E[p] for p in range(D + 1)) + (-1) ** D * P[D]
    assert lhs == rhs


# ------------------------------------------------------------------ persistent Betti numbers
def _gf2_rank(vecs):
    basis = {}
    r = 0
    for v in vecs:
        while v:
            h = v.bit_length() - 1
            if h in basis:
                v ^= basis[h]
            else:
                basis[h] = v
                r += 1
                break
    return r


def _gf2_kernel(cols):
    """Basis of the kernel of the linear map given by `cols` (ints), as subsets of
    column indices (ints)."""
    basis = {}   # pivot bit -> (vector, combination)
    ker = []
    for j, v in enumerate(cols):
        comb = 1 << j
        while v:
            h = v.bit_length() - 1
            if h in basis:
                bv, bc = basis[h]
                v ^= bv
                comb ^= bc
            else:
                basis[h] = (v, comb)
                break
        if not v:
            ker.append(comb)
    return ker


def _persistent_betti_barcode(lt, n, D):
    """Barcode (as a sorted list of (dim, birth, death)) from the persistent Betti numbers
    beta_p^{i,j} = dim Z_p(K_i) - dim(Z_p(K_i) ∩ B_p(K_j)), each a rank over Z/2.
    Bars with birth < death only; essential bars have death = inf."""
    dist = G.square_from_lower_tri(lt, n)
    simp = {k: [] for k in range(D + 2)}
    for k in range(D + 2):
        for vs in itertools.combinations(range(n), k + 1):
            dm = max((dist[a, b] for a, b in itertools.combinations(vs, 2)), default=np.float32(0))
            simp[k].append((vs, np.float32(dm)))
    vals = sorted({float(d) for k in simp for _, d in simp[k]})
    m = len(vals)
    index = {k: {vs: i for i, (vs, _) in enumerate(simp[k])} for k in simp}

    def bd(k, vs):  # boundary of a k-simplex as a bitmask over (k-1)-simplices
        out = 0
        for f in itertools.combinations(vs, k):
            out ^= 1 << index[k - 1][f]
        return out

    bars = []
    for p in range(D + 1):
        def cycles(i):
            ids = [a for a, (vs, dm) in enumerate(simp[p]) if dm <= vals[i]]
            if p == 0:
                return [1 << a for a in ids]
            cols = [bd(p, simp[p][a][0]) for a in ids]
            out = []
            for comb in _gf2_kernel(cols):
                v, q = 0, 0
                while comb:
                    if comb & 1:
                        v ^= 1 << ids[q]
                    comb >>= 1
                    q += 1
                out.append(v)
            return out

        def bounds(j):
            return [bd(p + 1, vs) for vs, dm in simp[p + 1] if dm <= vals[j]]

        Z = [cycles(i) for i in range(m)]
        B = [bounds(j) for j in range(m)]
        rB = [_gf2_rank(b) for b in B]

        def beta(i, j):
            if i < 0:
                return 0
            z = Z[i]
            dim_sum = _gf2_rank(z + B[j])
            inter = len(z) + rB[j] - dim_sum
            return len(z) - inter

        for i in range(m):
            for j in range(i + 1, m):
                mu = beta(i, j - 1) - beta(i, j) - beta(i - 1, j - 1) + beta(i - 1, j)
                bars += [(p, vals[i], vals[j])] * mu
            mu_inf = beta(i, m - 1) - beta(i - 1, m - 1)
            bars += [(p, vals[i], math.inf)] * mu_inf
    return sorted(bars)


def _oracle_bars(b, D):
    out = []
    for p in range(D + 1):
        for x, y in b.positive(p).tolist():
            out.append((p, x, y))
    return sorted(out)


@pytest.mark.parametrize("seed", range(10))
def test_persistent_betti_numbers_brute_force(seed):
    n, D = (6, 2) if seed % 2 == 0 else (8, 1)
    if seed % 3 == 0:
        lt = G.random_tied(n, seed, levels=3)
    elif seed % 3 == 1:
        lt = G.random_cloud(n, seed, dim=2)
    else:
        lt = G.regular_ngon(n)
    b = O.barcode(lt, n, D)
    assert _oracle_bars(b, D) == _persistent_betti_barcode(lt, n, D)


# ------------------------------------------------------------------ invariants
def test_enclosing_radius_examples():
    assert O.enclosing_radius(G.unit_square(), 4) == F32_SQRT2
    assert O.enclosing_radius(G.lower_tri_from_points(np.array([[0.0], [1.0], [3.0]])), 3) == 2.0
    assert O.enclosing_radius(np.zeros(0, np.float32), 1) == 0.0


@pytest.mark.parametrize("seed", range(6))
def test_prop5213_threshold_R_keeps_positive_bars(seed):
    n, D = 8, 2
    lt = G.random_cloud(n, seed) if seed % 2 else G.random_tied(n, seed)
    R = O.enclosing_radius(lt, n)
    full, cut = O.barcode(lt, n, D), O.barcode(lt, n, D, R)
    for p in range(D + 1):
        assert np.array_equal(full.positive(p), cut.positive(p))


@pytest.mark.parametrize("seed", range(4))
def test_obs568_monotone_remap(seed):
    # Obs 5.6.8: a strictly monotone re-map of the distances keeps the
    # index-level pairing and maps the endpoints.
    n, D = 7, 2
    lt = G.random_tied(n, seed, levels=6)
    remap = (lt.astype(np.float64) ** 2 * 3 + 1).astype(np.float32)
    a, b = O.barcode(lt, n, D), O.barcode(remap, n, D)
    for p in range(D + 1):
        assert a.index_pairs(p) == b.index_pairs(p)


@pytest.mark.parametrize("seed", range(8))
def test_apparent_pairs_are_persistence_pairs(seed):
    # Def 5.3.4 pairs are zero-persistence persistence pairs: the apparent set
    # computed on explicit sets must be contained in the reduction's index pairing.
    n = 7
    lt = G.random_tied(n, seed, levels=3) if seed % 2 else G.random_cloud(n, seed)
    t = [math.inf, float(np.quantile(lt, 0.6))][seed % 2]
    b = O.barcode(lt, n, 3, t)
    for d in (1, 2):
        c, f, partner = O.apparent(lt, n, d, t)
        pairs = b.index_pairs(d)
        for ci, pi in zip(c[f], partner[f]):
            assert (int(ci), int(pi)) in pairs


def test_circle_config1_one_long_h1_bar():
    cfg = G.CONFIGS["c1_circle64"]
    b = O.barcode(cfg.lower_tri(), cfg.n, cfg.max_dim)
    h1 = b.positive(1)
    pers = h1[:, 1] - h1[:, 0]
    assert (pers > 1.0).sum() == 1 and (pers[pers <= 1.0] < 0.2).all()
    assert b.n_simplices[:3] == [64, 2016, 41664]


def test_sphere_s2_betti():
    # beta_2(S^2) = 1: a 50-point sample has exactly one H2 bar, a long one, and at the
    # enclosing radius no essential classes above dimension 0 (Prop 5.2.13 proof)
    pts = G.sphere(50, 2, seed=3)
    lt = G.lower_tri_from_points(pts)
    R = O.enclosing_radius(lt, 50)
    b = O.barcode(lt, 50, 2, R)
    h2 = b.positive(2)
    assert len(h2) == 1 and h2[0, 1] - h2[0, 0] > 0.5
    assert b.num_essential(1) == 0 and b.num_essential(2) == 0 and b.num_essential(0) == 1


@pytest.mark.parametrize("seed", range(4))
def test_apparent_one_matches_set_definition(seed):
    # the per-simplex brute force (used on sampled full-size outputs) agrees with the
    # pinned set-based Def 5.3.4 on every simplex of small inputs
    n = 8
    lt = G.random_tied(n, seed, levels=3) if seed % 2 else G.random_cloud(n, seed)
    t = [math.inf, float(np.quantile(lt, 0.7))][seed % 2]
    for d in (1, 2):
        c, f, p = O.apparent(lt, n, d, t)
        for ci, fl, pi in zip(c.tolist(), f.tolist(), p.tolist()):
            vs, x, hi = [], ci, n
            for q in range(d + 1):
                kk = d + 1 - q
                v = kk - 1
                while v + 1 < hi and math.comb(v + 1, kk) <= x:
                    v += 1
                vs.append(v)
                x -= math.comb(v, kk)
                hi = v
            assert O.apparent_one(lt, n, vs, t) == (fl, pi if fl else None)
