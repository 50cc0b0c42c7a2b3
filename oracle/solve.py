"""Oracle end-to-end driver: ProblemSpec -> FGMRES solve with the two-grid
preconditioner (section 4) and its per-sample record
(PAPER.md:416-420).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import time

import numpy as np

from . import fem
from .fgmres import fgmres
from .twogrid import TwoGrid
from .shiftmap import map_shifts


def coefficients(spec):
    """Per-element k and eps on the fine and coarse meshes (readings C1, C2, C4;
    with spec.shift_map = p the fitted map sigma_p of PAPER.md:437-443, C20)."""
    ne_f = spec.n ** spec.dim
    ne_c = (spec.n // 2) ** spec.dim
    if spec.k_const is not None:
        kf = np.full(ne_f, spec.k_const)
        kc = np.full(ne_c, spec.k_const)
    else:
        kf, kc = spec.k_fine, spec.k_coarse
    p = getattr(spec, "shift_map", 0)
    if p:
        l = np.log2(spec.n)
        return kf, map_shifts(kf, spec.beta, p, l), kc, map_shifts(kc, spec.beta, p, l)
    return kf, fem.shifts(kf, spec.beta, spec.sigma), kc, fem.shifts(kc, spec.beta, spec.sigma)


class OracleProblem:
    """Everything the oracle needs for one spec: A_0, the two-grid on A_eps."""

    def __init__(self, spec):
        t0 = time.perf_counter()
        self.spec = spec
        kf, ef, kc, ec = coefficients(spec)
        self.A0 = fem.system_matrix(spec.dim, spec.n, kf, 0.0)
        self.tg = TwoGrid(spec.dim, spec.n, kf, ef, kc, ec, spec.nu_pre, spec.nu_post,
                          spec.omega)
        self.setup_s = time.perf_counter() - t0

    def apply(self, op: int, x):
        """op 0: A_0 x; op 1: A_eps x; op 2: A_eps^{(1)} x (coarse)."""
        return (self.A0, self.tg.A, self.tg.Ac)[op] @ x

    def vcycle(self, f):
        return self.tg.vcycle(f)

    def solve(self, b=None, fixed_iters=0, reorth=True):
        spec = self.spec
        if b is None:
            b = spec.rhs()
        t0 = time.perf_counter()
        x, rep = fgmres(lambda v: self.A0 @ v, self.tg.vcycle, b, restart=spec.restart,
                        rtol=spec.rtol, max_iters=spec.max_iters, fixed_iters=fixed_iters,
                        reorth=reorth)
        rep.solve_s = time.perf_counter() - t0
        rep.setup_s = self.setup_s
        return x, rep


def solve_spec(spec, **kw):
    return OracleProblem(spec).solve(**kw)
