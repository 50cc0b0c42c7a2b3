"""Seeded synthetic velocity media (BASELINE.json configs 2 and 4).

Readings (listed again in DESIGN.md):
  * the depth axis is the slowest grid index (y in 2D, z in 3D), depth 0 at
    the surface, layers are horizontal;
  * cfg2: numpy default_rng(0); draws, in order, c = U[1500,4500]^8 (layer 0..7
    top to bottom), m = integers(1,4,7), phi = U[0,2pi)^7; interface j (1..7)
    at depth j/8 + 0.05 sin(2 pi m_j x + phi_j); c(x,y) = c[#{j: y >= y_j(x)}];
  * cfg4: default_rng(0); c = U[1500,4500]^10, centres = U[0.1,0.9]^(8x3),
    a = U[-0.2,0.2]^8; layer = min(floor(10 z), 9);
    c = c[layer] * clip(1 + sum_m a_m exp(-|x-x_m|^2 / (2*0.1^2)), 0.8, 1.2).

The paper's own media (wedge, Marmousi, BP, ... PAPER.md section 6) are not
available; these stand in for them with the same grid sizes.  Only velocity
values are produced here; the wavenumber k = omega / c is formed in
configs.py.  No solver arithmetic lives in this module.
"""
from __future__ import annotations

import numpy as np


def element_centroids(n: int, dim: int):
    """Centroid coordinates of the n^dim cells of the unit square/cube, each
    returned as an array of shape (n,)*dim indexed [z][y][x] (x fastest)."""
    c = (np.arange(n, dtype=np.float64) + 0.5) / n
    grids = np.meshgrid(*([c] * dim), indexing="ij")  # grids[0] slowest
    # meshgrid 'ij' with axes ordered (slow..fast): return x, y(, z)
    return tuple(reversed(grids))


def _layered_2d_params(seed: int = 0):
    rng = np.random.default_rng(seed)
    c = rng.uniform(1500.0, 4500.0, 8)
    m = rng.integers(1, 4, 7)
    phi = rng.uniform(0.0, 2.0 * np.pi, 7)
    return c, m, phi


def layered_2d_velocity(x: np.ndarray, y: np.ndarray, seed: int = 0) -> np.ndarray:
    """c(x, y) of the cfg2 medium (8 layers, sinusoidal interfaces, amp 0.05)."""
    c, m, phi = _layered_2d_params(seed)
    count = np.zeros(np.broadcast(x, y).shape, dtype=np.int64)
    for j in range(1, 8):
        yj = j / 8.0 + 0.05 * np.sin(2.0 * np.pi * m[j - 1] * x + phi[j - 1])
        count += (y >= yj).astype(np.int64)
    return c[count]


def _inclusion_3d_params(seed: int = 0):
    rng = np.random.default_rng(seed)
    c = rng.uniform(1500.0, 4500.0, 10)
    centres = rng.uniform(0.1, 0.9, (8, 3))
    a = rng.uniform(-0.2, 0.2, 8)
    return c, centres, a


def inclusion_3d_velocity(x: np.ndarray, y: np.ndarray, z: np.ndarray,
                          seed: int = 0) -> np.ndarray:
    """c(x, y, z) of the cfg4 medium (10 layers + 8 Gaussian inclusions)."""
    c, centres, a = _inclusion_3d_params(seed)
    layer = np.minimum(np.floor(10.0 * z).astype(np.int64), 9)
    pert = np.ones(np.broadcast(x, y, z).shape)
    for mm in range(8):
        r2 = (x - centres[mm, 0]) ** 2 + (y - centres[mm, 1]) ** 2 + (z - centres[mm, 2]) ** 2
        pert = pert + a[mm] * np.exp(-r2 / (2.0 * 0.1 ** 2))
    return c[layer] * np.clip(pert, 0.8, 1.2)
