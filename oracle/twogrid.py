"""Oracle: two-grid V(nu,nu) cycle on the shifted operator A_eps.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:369-386 (section 4, Alg. 1, L = 2):
    nu x   u <- u + S^{-1}(F - A_eps u)          presmoothing
           r <- I^T (F - A_eps u)                 restrict residual
           u_c <- A_eps^{(1)}^{-1} r              direct coarse solve
           u <- u + I u_c                          coarse-grid correction
    nu x   u <- u + S^{-T}(F - A_eps u)          postsmoothing
Damped Jacobi S^{-1} = omega D^{-1}, D = diag(A_eps);
for a diagonal D the post-smoother S^{-T} equals S^{-1}.  Readings: D
includes the -i k B boundary diagonal (C6); the coarse operator is the
rediscretisation on the 2h mesh (C4); the paper's "A_e" in the
postsmoothing line is A_eps (G7).  The coarse matrix is factored once and
reused, here by SuperLU with partial pivoting (or dense
LAPACK LU for tiny grids).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse.linalg as spla

from . import fem


class CoarseSolver:
    """Direct solve with A_eps^{(1)} (Alg. 1 line 3)."""

    def __init__(self, Ac, dense_below: int = 2000):
        self.N = Ac.shape[0]
        if self.N < dense_below:
            self.kind = "dense-lu"
            self.lu = sla.lu_factor(Ac.toarray())
        else:
            self.kind = "superlu"
            self.lu = spla.splu(Ac.tocsc(), permc_spec="COLAMD")

    def solve(self, r):
        if self.kind == "dense-lu":
            return sla.lu_solve(self.lu, r)
        return self.lu.solve(r)


class TwoGrid:
    """Holds A_eps (fine), A_eps^{(1)} (coarse, factored) and I for one problem."""

    def __init__(self, dim, n, k_fine, eps_fine, k_coarse, eps_coarse,
                 nu_pre=2, nu_post=2, omega=0.6, coarse_dense_below=2000):
        self.dim, self.n = dim, n
        self.A = fem.system_matrix(dim, n, k_fine, eps_fine)
        self.Ac = fem.system_matrix(dim, n // 2, k_coarse, eps_coarse)
        self.P = fem.prolongation(dim, n)
        self.D = self.A.diagonal()
        if np.any(self.D == 0):
            raise ZeroDivisionError("zero Jacobi diagonal")
        self.coarse = CoarseSolver(self.Ac, coarse_dense_below)
        self.nu_pre, self.nu_post, self.omega = nu_pre, nu_post, omega

    def jacobi(self, u, f):
        """One damped Jacobi step u + omega D^{-1} (f - A_eps u)."""
        return u + self.omega * (f - self.A @ u) / self.D

    def restrict_residual(self, u, f):
        """r_c = I^T (f - A_eps u)   (Alg. 1 'Restrict residual'; I^T not conjugated)."""
        return self.P.T @ (f - self.A @ u)

    def vcycle(self, f, u0=None):
        """z = V-cycle(u0 (default 0), f) exactly in Alg. 1 order."""
        u = np.zeros_like(f) if u0 is None else u0.copy()
        for _ in range(self.nu_pre):
            u = self.jacobi(u, f)
        r = self.restrict_residual(u, f)
        uc = self.coarse.solve(r)
        u = u + self.P @ uc
        for _ in range(self.nu_post):
            u = self.jacobi(u, f)
        return u
