"""BASELINE.json configs 0-4 as concrete, seeded problem specifications.

Readings (repeated in DESIGN.md "Readings"):
  C7  unit point source = the exact FE load of a Dirac delta, F_i = phi_i(s);
  C9  cfg1: n = smallest even integer >= k / kh_target (actual kh <= target);
  C10 max_iters = 500 everywhere;
  C14 restart/rtol: cfg0/1/2 -> restart 100, rtol 1e-6; cfg3/4 -> restart 50;
  C15 omega = 0.6, nu = 2 + 2 everywhere;
  C16 cfg4 source at the centre node;
  C17 media in media.py, omega_ang = 0.5 * min_e c_e / h (max k_e h = 0.5).
Per-element wavenumbers are sampled at element centroids (C1); coarse
elements use their own centroids (C4).  No solver arithmetic lives here.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .media import element_centroids, layered_2d_velocity, inclusion_3d_velocity

CONFIG_NAMES = ("cfg0", "cfg1", "cfg2", "cfg3", "cfg4")


@dataclass
class ProblemSpec:
    name: str
    dim: int
    n: int                       # fine cells per side (even); h = 1/n
    k_const: Optional[float]     # constant wavenumber, or None if heterogeneous
    k_fine: Optional[np.ndarray] = None    # (n^dim,) per-element k, x fastest
    k_coarse: Optional[np.ndarray] = None  # ((n/2)^dim,) per coarse element
    beta: float = 1.0            # eps_e = beta * k_e^sigma
    sigma: float = 1.5
    nu_pre: int = 2
    nu_post: int = 2
    omega: float = 0.6
    restart: int = 100
    rtol: float = 1e-6
    max_iters: int = 500
    source: tuple = (0.5, 0.5)
    meta: dict = field(default_factory=dict)
    shift_map: int = 0           # > 0: sigma = sigma_p(k_e, log2 n) of Table 1 row p

    @property
    def h(self) -> float:
        return 1.0 / self.n

    @property
    def n_nodes(self) -> int:
        return (self.n + 1) ** self.dim

    @property
    def n_coarse_nodes(self) -> int:
        return (self.n // 2 + 1) ** self.dim

    def rhs(self) -> np.ndarray:
        """Point-source load vector (complex128, x-fastest)."""
        b = np.zeros(self.n_nodes, dtype=np.complex128)
        idx, w = point_source_weights(self.n, self.dim, self.source)
        b[idx] = w
        return b


def point_source_weights(n: int, dim: int, s):
    """Nodes and weights of F_i = phi_i(s) for the Q1 nodal basis on the
    uniform n^dim grid (reading C7).  Returns (flat node indices, weights)."""
    per_dim = []
    for d in range(dim):
        t = s[d] * n
        i = min(int(math.floor(t)), n - 1)
        f = t - i
        per_dim.append([(i, 1.0 - f), (i + 1, f)])
    idx, wts = [], []
    stride = [(n + 1) ** d for d in range(dim)]
    import itertools
    for combo in itertools.product(*per_dim):
        w = 1.0
        flat = 0
        for d, (i, wd) in enumerate(combo):
            w *= wd
            flat += i * stride[d]
        if w != 0.0:
            idx.append(flat)
            wts.append(w)
    return np.asarray(idx, dtype=np.int64), np.asarray(wts, dtype=np.float64)


def _het_k(dim: int, n: int, seed: int = 0):
    """Fine and coarse per-element k = omega_ang / c for the cfg2/cfg4 media."""
    vel = layered_2d_velocity if dim == 2 else inclusion_3d_velocity
    cf = vel(*element_centroids(n, dim), seed=seed).reshape(-1)
    cc = vel(*element_centroids(n // 2, dim), seed=seed).reshape(-1)
    omega_ang = 0.5 * cf.min() * n          # max_e k_e h = 0.5 exactly
    return omega_ang / cf, omega_ang / cc, omega_ang


def config_spec(name: str, n: Optional[int] = None) -> ProblemSpec:
    """BASELINE.json config `name`; `n` overrides the grid for smaller
    analogues of the same recipe (used by parity tests)."""
    if name == "cfg0":
        return ProblemSpec("cfg0", 2, n or 64, 20.0, beta=1.0, sigma=1.5,
                           restart=100, source=(0.5, 0.5))
    if name == "cfg2":
        nn = n or 1024
        kf, kc, om = _het_k(2, nn)
        return ProblemSpec("cfg2", 2, nn, None, kf, kc, beta=0.5, sigma=1.5,
                           restart=100, source=(0.5, 0.1),
                           meta={"omega_ang": om, "k_min": float(kf.min()),
                                 "k_max": float(kf.max())})
    if name == "cfg3":
        return ProblemSpec("cfg3", 3, n or 128, 40.0, beta=0.5, sigma=1.5,
                           restart=50, source=(0.5, 0.5, 0.5))
    if name == "cfg4":
        nn = n or 256
        kf, kc, om = _het_k(3, nn)
        return ProblemSpec("cfg4", 3, nn, None, kf, kc, beta=0.5, sigma=1.5,
                           restart=50, source=(0.5, 0.5, 0.5),
                           meta={"omega_ang": om, "k_min": float(kf.min()),
                                 "k_max": float(kf.max())})
    raise ValueError(f"unknown config {name!r} (cfg1 is a sweep: use sweep_samples)")


SWEEP_K = tuple(float(10 * i) for i in range(1, 17))          # 10..160
SWEEP_KH = (0.3, 0.6)
SWEEP_SIGMA = tuple((10 + i) / 10.0 for i in range(11))       # 1.0..2.0
SWEEP_BETA = tuple(i / 10.0 for i in range(1, 11))            # 0.1..1.0


def sweep_grid_n(k: float, kh_target: float) -> int:
    """Reading C9: smallest even n with k/n <= kh_target."""
    n = math.ceil(k / kh_target - 1e-12)
    if n % 2:
        n += 1
    return max(n, 4)


def sweep_samples():
    """The 3,520 cfg1 samples (k outer, then kh, sigma, beta innermost)."""
    out = []
    sid = 0
    for k in SWEEP_K:
        for kh in SWEEP_KH:
            n = sweep_grid_n(k, kh)
            for s in SWEEP_SIGMA:
                for b in SWEEP_BETA:
                    out.append({"id": sid, "dim": 2, "n": n, "k": k, "kh_target": kh,
                                "sigma": s, "beta": b})
                    sid += 1
    return out


def sweep_sample_spec(sample: dict) -> ProblemSpec:
    """ProblemSpec of one cfg1 sample (cfg0's solver settings, C14)."""
    return ProblemSpec(f"cfg1#{sample['id']}", 2, sample["n"], sample["k"],
                       beta=sample["beta"], sigma=sample["sigma"], restart=100,
                       source=(0.5, 0.5), meta=dict(sample))


# ------------------------------------------------------------------ shift-search recipe
def search_samples(count: int, seed: int = 0, levels=(4, 5, 6, 7, 8, 9, 10), p: int = 1):
    """Sec. 5 steps 1-3 for Q1 (p = 1): l uniform in `levels`,
    h = 2^-l (n = 2^l), k uniform in [3p/(16h), 3p/(4h)]; shift eps = k^sigma
    (beta = 1).  Seeded; returns dicts with id, n, k, l."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        l = int(rng.choice(levels))
        n = 2 ** l
        k = float(rng.uniform(3 * p * n / 16, 3 * p * n / 4))
        out.append({"id": i, "dim": 2, "n": n, "l": l, "k": k, "beta": 1.0})
    return out


def search_rhs(sample: dict, seed: int = 0) -> np.ndarray:
    """Step 4: right-hand side with components uniform in [-1, 1]
    (real), drawn once per sample (seed, id) and reused for every sigma."""
    rng = np.random.default_rng([seed, int(sample["id"])])
    n1 = (sample["n"] + 1) ** 2
    return rng.uniform(-1.0, 1.0, n1).astype(np.complex128)


def search_sample_spec(sample: dict) -> ProblemSpec:
    """ProblemSpec of one search sample at sigma = 1.5 (sigma is the search variable);
    BASELINE's V-cycle settings (2 + 2, omega 0.6), no restart within the 50-iteration
    budget (the paper uses none)."""
    return ProblemSpec(f"search#{sample['id']}", 2, sample["n"], sample["k"], beta=1.0, sigma=1.5,
                       restart=50, rtol=1e-8, max_iters=50, meta=dict(sample))
