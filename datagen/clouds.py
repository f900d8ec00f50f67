"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module holds NONE of the method's arithmetic (no simplices, no diameters, no
filtration, no reduction).  It only draws point clouds with numpy's PCG64 and turns
them into the fp32 distance matrix that every consumer reads, exactly as the survey's
input recipe states (SURVEY.md §8(d) "Inputs"):

    D_ij = float32( sqrt( sum_k (x_ik - x_jk)^2 ) )   computed in float64, rounded once

The output layout is Ripser's lower-distance order (SPEC.md "lower-distance format",
S:159 / A25): entry (i, j), i > j, sits at index i*(i-1)/2 + j of a flat float32
vector of length n*(n-1)/2.

Point-cloud shapes follow BASELINE.json `configs` and SURVEY.md §8(d):
  1  circle        n=64    theta ~ U[0, 2pi)                               seed 1
  2  S^3           n=192   g ~ N(0, I_4), g/|g|                            seed 2
  3  trefoil tube  n=1000  radius-0.3 tube around the trefoil + N(0,.02^2)  seed 3
  4a Sierpinski    n=512   tetrahedron chaos game, 100 burn-in + N(0,.003^2) seed 4
  4b Clifford torus n=2000 (cos a, sin a, cos b, sin b)                    seed 5
  5  O(3)          n=4096  Haar O(3) via QR with sign fix, flattened to R^9 seed 6
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


# --------------------------------------------------------------------------------------
# point clouds
# --------------------------------------------------------------------------------------

def circle(n: int, seed: int = 1) -> np.ndarray:
    rng = np.random.default_rng(seed)
    th = rng.uniform(0.0, 2.0 * math.pi, n)
    return np.stack([np.cos(th), np.sin(th)], axis=1)


def sphere(n: int, dim: int, seed: int) -> np.ndarray:
    """Uniform sample of S^dim in R^(dim+1) (normalised Gaussians)."""
    rng = np.random.default_rng(seed)
    g = rng.standard_normal((n, dim + 1))
    return g / np.linalg.norm(g, axis=1, keepdims=True)


def trefoil_tube(n: int, seed: int = 3, radius: float = 0.3, noise: float = 0.02) -> np.ndarray:
    """Tube of radius `radius` around the trefoil knot (a genus-1 surface) plus noise."""
    rng = np.random.default_rng(seed)
    s = rng.uniform(0.0, 2.0 * math.pi, n)
    phi = rng.uniform(0.0, 2.0 * math.pi, n)
    c = np.stack([np.sin(s) + 2 * np.sin(2 * s), np.cos(s) - 2 * np.cos(2 * s), -np.sin(3 * s)], 1)
    dc = np.stack([np.cos(s) + 4 * np.cos(2 * s), -np.sin(s) + 4 * np.sin(2 * s), -3 * np.cos(3 * s)], 1)
    tang = dc / np.linalg.norm(dc, axis=1, keepdims=True)
    # a normal frame: Gram-Schmidt of a fixed helper vector against the tangent
    helper = np.where(np.abs(tang[:, 2:3]) < 0.9, np.array([[0.0, 0.0, 1.0]]), np.array([[1.0, 0.0, 0.0]]))
    n1 = helper - (helper * tang).sum(1, keepdims=True) * tang
    n1 /= np.linalg.norm(n1, axis=1, keepdims=True)
    n2 = np.cross(tang, n1)
    pts = c + radius * (np.cos(phi)[:, None] * n1 + np.sin(phi)[:, None] * n2)
    return pts + rng.normal(0.0, noise, pts.shape)


def sierpinski(n: int, seed: int = 4, burn_in: int = 100, noise: float = 0.003) -> np.ndarray:
    """Chaos game on the regular tetrahedron (Sierpinski tetrahedron) plus noise."""
    rng = np.random.default_rng(seed)
    verts = np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], dtype=np.float64)
    x = rng.uniform(-1, 1, 3)
    out = np.empty((n, 3))
    for i in range(burn_in + n):
        x = 0.5 * (x + verts[rng.integers(0, 4)])
        if i >= burn_in:
            out[i - burn_in] = x
    return out + rng.normal(0.0, noise, out.shape)


def clifford_torus(n: int, seed: int = 5) -> np.ndarray:
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.0, 2.0 * math.pi, n)
    b = rng.uniform(0.0, 2.0 * math.pi, n)
    return np.stack([np.cos(a), np.sin(a), np.cos(b), np.sin(b)], 1)


def haar_o3(n: int, seed: int = 6) -> np.ndarray:
    """Haar-random O(3) matrices (QR of Gaussian with the sign fix), flattened to R^9."""
    rng = np.random.default_rng(seed)
    out = np.empty((n, 9))
    for i in range(n):
        q, r = np.linalg.qr(rng.standard_normal((3, 3)))
        q = q * np.sign(np.diag(r))[None, :]
        out[i] = q.reshape(-1)
    return out


# --------------------------------------------------------------------------------------
# distances
# --------------------------------------------------------------------------------------

def lower_tri_from_points(x: np.ndarray) -> np.ndarray:
    """fp32 lower-distance vector (Ripser order) of the Euclidean metric of `x`.

    Computed in float64 and rounded to float32 once (round-to-nearest-even).
    """
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0]
    out = np.empty(n * (n - 1) // 2, dtype=np.float32)
    for i in range(1, n):
        d = np.sqrt(((x[:i] - x[i]) ** 2).sum(axis=1))
        out[i * (i - 1) // 2: i * (i + 1) // 2] = d.astype(np.float32)
    return out


def square_from_lower_tri(lt: np.ndarray, n: int) -> np.ndarray:
    """Symmetric n x n float32 matrix with zero diagonal (a pure re-layout of `lt`)."""
    m = np.zeros((n, n), dtype=np.float32)
    if n > 1:
        i, j = np.tril_indices(n, -1)
        # np.tril_indices enumerates row-major (i asc, j asc) == Ripser lower order
        m[i, j] = lt
        m[j, i] = lt
    return m


def lower_tri_from_square(m: np.ndarray) -> np.ndarray:
    n = m.shape[0]
    i, j = np.tril_indices(n, -1)
    return np.ascontiguousarray(m[i, j], dtype=np.float32)


# --------------------------------------------------------------------------------------
# closed-form and fixture inputs (SURVEY.md §4, §8(c) pins table)
# --------------------------------------------------------------------------------------

def unit_square() -> np.ndarray:
    """Fig 5.1: four corners of the unit square."""
    return lower_tri_from_points(np.array([[0, 0], [1, 0], [1, 1], [0, 1]], dtype=np.float64))


def cross_polytope(k: int) -> np.ndarray:
    """+-e_i in R^k (2k points)."""
    pts = np.concatenate([np.eye(k), -np.eye(k)], axis=0)
    return lower_tri_from_points(pts)


def regular_ngon(n: int) -> np.ndarray:
    th = 2.0 * math.pi * np.arange(n) / n
    return lower_tri_from_points(np.stack([np.cos(th), np.sin(th)], 1))


def all_equal(n: int, value: float = 1.0) -> np.ndarray:
    """Thm 5.4.2 tightness case: every pairwise distance equal."""
    return np.full(n * (n - 1) // 2, value, dtype=np.float32)


def fig56_lex_decreasing(n: int) -> np.ndarray:
    """§5.4.3 / Fig 5.6: distinct distances assigned DEcreasing along the
    increasing lexicographic order of edges (v1 > v0), i.e. edge number k (0-based, in
    the order (1,0),(2,0),(2,1),(3,0),...) gets distance m - k with m = n(n-1)/2.
    The lower-distance order enumerates exactly that edge order."""
    m = n * (n - 1) // 2
    return (m - np.arange(m)).astype(np.float32)


def random_tied(n: int, seed: int, levels: int = 4) -> np.ndarray:
    """Random symmetric metric-like input with heavy ties (integer levels 1..levels)."""
    rng = np.random.default_rng(seed)
    return rng.integers(1, levels + 1, n * (n - 1) // 2).astype(np.float32)


def random_cloud(n: int, seed: int, dim: int = 3) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return lower_tri_from_points(rng.uniform(0, 1, (n, dim)))


# --------------------------------------------------------------------------------------
# the BASELINE.json configs
# --------------------------------------------------------------------------------------

@dataclass(frozen=True)
class Config:
    name: str
    n: int
    max_dim: int
    threshold: float      # +inf means "no threshold" (library cuts at the enclosing radius)
    seed: int
    shape: str

    def points(self, n: int | None = None) -> np.ndarray:
        m = self.n if n is None else n
        f = {
            "circle": lambda: circle(m, self.seed),
            "s3": lambda: sphere(m, 3, self.seed),
            "trefoil": lambda: trefoil_tube(m, self.seed),
            "sierpinski": lambda: sierpinski(m, self.seed),
            "torus": lambda: clifford_torus(m, self.seed),
            "o3": lambda: haar_o3(m, self.seed),
        }[self.shape]
        return f()

    def lower_tri(self, n: int | None = None) -> np.ndarray:
        """fp32 lower-distance vector; `n` < self.n draws the first n points of the same
        generator stream (a subsample usable by the oracle)."""
        return lower_tri_from_points(self.points(n))

    def patch(self, m: int, center: int = 0) -> np.ndarray:
        """fp32 lower-distance vector of the m points of the full cloud nearest to point
        `center` (itself included; ties by index), in index order: a local patch with the
        full cloud's density — for thresholded configs (config 5) the first-m subsample is
        nearly empty at the config's threshold, a patch is not."""
        x = self.points()
        d = np.sqrt(((x - x[center]) ** 2).sum(1))
        idx = np.sort(np.argsort(d, kind="stable")[:m])
        return lower_tri_from_points(x[idx])


INF = float("inf")

CONFIGS = {
    "c1_circle64": Config("c1_circle64", 64, 1, INF, 1, "circle"),
    "c2_s3_192": Config("c2_s3_192", 192, 3, INF, 2, "s3"),
    "c3_trefoil1000": Config("c3_trefoil1000", 1000, 2, INF, 3, "trefoil"),
    "c4a_sierpinski512": Config("c4a_sierpinski512", 512, 2, INF, 4, "sierpinski"),
    "c4b_torus2000": Config("c4b_torus2000", 2000, 2, INF, 5, "torus"),
    "c5_o3_4096": Config("c5_o3_4096", 4096, 3, 1.4, 6, "o3"),
}
