"""Pins of oracle/twogrid.py (and the transfers in oracle/fem.py).  -m "not gpu"."""
import numpy as np
import pytest
import scipy.linalg as sla

from oracle import fem, lfa
from oracle.twogrid import TwoGrid, CoarseSolver


@pytest.mark.parametrize("dim,n", [(2, 8), (2, 12), (3, 4)])
def test_prolongation_reproduces_linears(dim, n):
    """Nested Q1 spaces: I maps the coarse nodal values of a linear function to
    its exact fine nodal values ('canonical interpolation')."""
    P = fem.prolongation(dim, n)
    cf = fem.node_coords(dim, n)
    cc = fem.node_coords(dim, n // 2)
    coef = [0.3, -1.7, 2.2][:dim]
    lin_f = 0.5 + sum(a * c for a, c in zip(coef, cf))
    lin_c = 0.5 + sum(a * c for a, c in zip(coef, cc))
    np.testing.assert_allclose((P @ lin_c).real, lin_f, atol=1e-14)


@pytest.mark.parametrize("dim,n,s", [(2, 8, 4.0), (3, 6, 8.0)])
def test_restriction_weights(dim, n, s):
    """I^T 1 = 4 (2D) / 8 (3D) at interior coarse nodes (PAPER.md:169-177
    stencil (1/4)[1 2 1; 2 4 2; 1 2 1] times the factor 4 of reading C5)."""
    P = fem.prolongation(dim, n)
    r = (P.T @ np.ones(P.shape[0])).real
    cc = fem.node_coords(dim, n // 2)
    inner = np.ones(P.shape[1], bool)
    for c in cc:
        inner &= (c > 1e-9) & (c < 1 - 1e-9)
    np.testing.assert_allclose(r[inner], s)
    # unit vector at a coarse-coincident fine node: weights 1, 1/2, 1/4 (2D)
    if dim == 2:
        e = np.zeros(P.shape[0]); N1 = n + 1
        e[4 + 4 * N1 + 1] = 1.0          # fine (5,4): edge midpoint between coarse (2,2),(3,2)
        rc = (P.T @ e).real
        assert sorted(rc[rc != 0]) == [0.5, 0.5]


@pytest.mark.parametrize("dim,n", [(2, 8), (2, 16), (3, 4), (3, 8)])
def test_galerkin_identity_constant_k(dim, n):
    """Rediscretised coarse operator equals I^T A_h I for constant k, boundary
    term included (nested spaces + exact integration)."""
    k, eps = 7.0, 0.5 * 7.0 ** 1.5
    A = fem.system_matrix(dim, n, k, eps)
    Ac = fem.system_matrix(dim, n // 2, k, eps)
    P = fem.prolongation(dim, n)
    G = (P.T @ A @ P).toarray()
    assert np.abs(G - Ac.toarray()).max() <= 1e-13 * np.abs(Ac.toarray()).max()


def test_coarse_solver_dense_and_sparse_agree():
    """Coarse direct solve: SuperLU and dense LAPACK LU give the same solution,
    and the residual is at round-off (BASELINE north_star: 'exact agreement of
    a brute-force dense LU solve on tiny grids')."""
    rng = np.random.default_rng(3)
    n = 24
    k = rng.uniform(5, 12, n * n)
    Ac = fem.system_matrix(2, n, k, 0.5 * k ** 1.5)
    r = rng.standard_normal(Ac.shape[0]) + 1j * rng.standard_normal(Ac.shape[0])
    x1 = CoarseSolver(Ac, dense_below=10 ** 9).solve(r)
    x2 = CoarseSolver(Ac, dense_below=0).solve(r)
    x3 = np.linalg.solve(Ac.toarray(), r)
    assert np.linalg.norm(x1 - x3) <= 1e-12 * np.linalg.norm(x3)
    assert np.linalg.norm(x2 - x3) <= 1e-12 * np.linalg.norm(x3)
    assert np.linalg.norm(Ac @ x2 - r) <= 1e-12 * np.linalg.norm(r)


def _tg(n, k, eps, dim=2, **kw):
    ne, nc = n ** dim, (n // 2) ** dim
    return TwoGrid(dim, n, np.full(ne, k), np.full(ne, eps), np.full(nc, k), np.full(nc, eps), **kw)


def test_vcycle_equals_dense_two_grid_operator():
    """On a 9x9 node grid: zero-start V-cycle output z = (I - T) A_eps^{-1} f
    with T = S^nu (I - I A_c^{-1} I^T A_eps) S^nu, S = I - omega D^{-1} A_eps
    (PAPER.md:145-149 two-grid error propagator), built from dense inverses."""
    tg = _tg(8, 5.0, 5.0 ** 1.5)
    A = tg.A.toarray(); Ac = tg.Ac.toarray(); P = tg.P.toarray()
    Nf = A.shape[0]
    S = np.eye(Nf) - 0.6 * np.diag(1 / np.diag(A)) @ A
    T = np.linalg.matrix_power(S, 2) @ (np.eye(Nf) - P @ np.linalg.inv(Ac) @ P.T @ A) @ \
        np.linalg.matrix_power(S, 2)
    rng = np.random.default_rng(0)
    for _ in range(5):
        f = rng.standard_normal(Nf) + 1j * rng.standard_normal(Nf)
        z = tg.vcycle(f)
        want = (np.eye(Nf) - T) @ np.linalg.solve(A, f)
        assert np.linalg.norm(z - want) <= 1e-12 * np.linalg.norm(want)


def test_vcycle_linear_and_fixed_point():
    """V(f) is linear in f; the exact solution is a fixed point."""
    tg = _tg(16, 9.0, 9.0 ** 1.5)
    rng = np.random.default_rng(1)
    N = tg.A.shape[0]
    f1 = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    f2 = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    a, b = 0.3 - 1.2j, 2.0 + 0.5j
    lhs = tg.vcycle(a * f1 + b * f2)
    rhs = a * tg.vcycle(f1) + b * tg.vcycle(f2)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)
    u = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    f = tg.A @ u
    assert np.linalg.norm(tg.vcycle(f, u0=u) - u) <= 1e-12 * np.linalg.norm(u)


def _measured_contraction(n, k, eps, iters=60):
    tg = _tg(n, k, eps)
    e = np.random.default_rng(0).standard_normal(tg.A.shape[0]) + 0j
    r = 0.0
    for _ in range(iters):
        e2 = e - tg.vcycle(tg.A @ e)
        r = np.linalg.norm(e2) / np.linalg.norm(e)
        e = e2 / np.linalg.norm(e2)
    return r


@pytest.mark.parametrize("kh,sigma", [(0.25, 2.0), (0.5, 2.0)])
def test_vcycle_contraction_matches_lfa_strong_shift(kh, sigma):
    """Two-grid contraction on A_eps vs the paper's LFA rho_loc
    for nu=2, omega=0.6, h=2^-5 and a strong shift eps = k^sigma: within 0.02.
    A wrong restriction scale, smoother diagonal or coarse operator breaks this."""
    h = 1 / 32
    k = kh / h
    eps = k ** sigma
    rl = lfa.rho_loc(k * k + 1j * eps, h, 0.6, 2, 2, m=48)
    meas = _measured_contraction(32, k, eps)
    assert abs(meas - rl) <= 0.02, (meas, rl)


def test_vcycle_contraction_weak_shift_bounded_by_lfa():
    """Weak shift (kh=0.5, sigma=1): the bounded-domain two-grid contracts no
    worse than the LFA rho_loc (LFA ignores the absorbing boundary)."""
    h = 1 / 32
    k = 0.5 / h
    rl = lfa.rho_loc(k * k + 1j * k, h, 0.6, 2, 2, m=48)
    meas = _measured_contraction(32, k, k)
    assert meas <= rl and meas < 1.0, (meas, rl)


def test_jacobi_symbol_matches_paper():
    """One Jacobi step on an interior Fourier mode multiplies it by the paper's
    smoother symbol S~_h, with D = diag(A_eps)."""
    n, k = 32, 8.0
    eps = k ** 1.5
    tg = _tg(n, k, eps)
    h = 1 / n
    x, y = fem.node_coords(2, n)
    th = (0.7, -0.4)
    u = np.exp(1j * (th[0] * x + th[1] * y) / h)
    Su = tg.jacobi(u, np.zeros_like(u))      # error propagation S u
    inner = (x > 1e-9) & (x < 1 - 1e-9) & (y > 1e-9) & (y < 1 - 1e-9)
    sym = lfa.S_h(th[0], th[1], k * k + 1j * eps, h, 0.6)
    np.testing.assert_allclose(Su[inner], sym * u[inner], rtol=1e-12)
