"""Seeded test vectors and sampled node sets shared by the golden generator
(`scripts/make_goldens.py`, oracle side) and the GPU parity tests.

Only random numbers and index sets live here: no element matrices, no
operators, no solver steps (the rule of workloads/__init__.py).
"""
from __future__ import annotations

import numpy as np


def random_complex(n: int, seed: int) -> np.ndarray:
    """x_i = a_i + i b_i with a, b ~ N(0, 1), numpy default_rng(seed)."""
    r = np.random.default_rng(seed)
    return r.standard_normal(n) + 1j * r.standard_normal(n)


def sampled_nodes(n_cells: int, dim: int, count: int, seed: int, extra=()) -> np.ndarray:
    """`count` seeded node indices of the (n_cells+1)^dim grid, plus every
    grid corner, the centre node and `extra`, sorted and unique."""
    N1 = n_cells + 1
    total = N1 ** dim
    r = np.random.default_rng(seed)
    rows = [int(v) for v in r.integers(0, total, count)]
    for c in range(2 ** dim):                          # grid corners
        rows.append(sum(((c >> d) & 1) * n_cells * N1 ** d for d in range(dim)))
    rows.append(sum((n_cells // 2) * N1 ** d for d in range(dim)))
    rows += [int(v) for v in extra]
    return np.array(sorted(set(rows)), dtype=np.int64)
