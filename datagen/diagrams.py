"""Seeded synthetic persistence diagrams for the PDoptFlow row.

Input generation only — no W1 arithmetic lives here.  A diagram is an (n, 2) float32
array of (birth, death) points with death > birth (off the diagonal Δ).

  gaussian(n, seed)   PAPER.md §6.10.2 / Fig 6.1: "points randomly distributed
                      on the plane above the diagonal ... follow a Gaussian distribution".
                      Recipe: (b, d) = (mu_b, mu_d) + N(0, Sigma) with mu = (1.0, 2.0),
                      Sigma = [[0.25, 0.1], [0.1, 0.25]]; points with d <= b are reflected
                      across Δ (swap b and d); exact ties with Δ are redrawn.
  clustered(n, seed)  filtration values on a 2^8 lattice (the voxel case of (6.42),
                      §6.3.3): b, d drawn from 256 levels, so many points coincide —
                      the shape where 0-condensation and δ-condensation collapse nodes.
"""
from __future__ import annotations

import numpy as np


def _above(b: np.ndarray, d: np.ndarray) -> np.ndarray:
    lo, hi = np.minimum(b, d), np.maximum(b, d)
    return np.stack([lo, hi], 1).astype(np.float32)


def gaussian(n: int, seed: int, mu=(1.0, 2.0), cov=((0.25, 0.1), (0.1, 0.25))) -> np.ndarray:
    rng = np.random.default_rng(seed)
    out = np.zeros((0, 2), np.float32)
    while out.shape[0] < n:
        x = rng.multivariate_normal(mu, cov, size=n - out.shape[0])
        p = _above(x[:, 0], x[:, 1])
        p = p[p[:, 1] > p[:, 0]]
        out = np.concatenate([out, p])
    return out[:n]


def clustered(n: int, seed: int, levels: int = 256) -> np.ndarray:
    rng = np.random.default_rng(seed)
    out = np.zeros((0, 2), np.float32)
    while out.shape[0] < n:
        b = rng.integers(0, levels, n - out.shape[0])
        life = np.maximum(1, np.round(rng.exponential(levels / 8, n - out.shape[0]))).astype(np.int64)
        d = np.minimum(b + life, levels)
        p = np.stack([b, d], 1).astype(np.float32) / np.float32(levels)
        p = p[p[:, 1] > p[:, 0]]
        out = np.concatenate([out, p])
    return out[:n]


def uniform(n: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """Small random diagrams for brute-force pins: b ~ U[0, s), d = b + U(0, s]."""
    rng = np.random.default_rng(seed)
    b = rng.random(n) * scale
    d = b + (1.0 - rng.random(n)) * scale
    return np.stack([b, d], 1).astype(np.float32)
