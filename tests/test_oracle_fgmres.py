"""Pins of oracle/fgmres.py and the end-to-end oracle solve.  -m "not gpu"."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import fem
from oracle.fgmres import fgmres, average_rate, givens
from oracle.solve import OracleProblem
from workloads import config_spec


def test_average_rate_examples():
    """rho = (r_end/r_0)^(1/end): 1e-8 over 8 its -> 0.1;
    r0=4, r_end=1, end=2 -> 0.5; stagnation -> 1."""
    assert abs(average_rate(1.0, 1e-8, 8) - 0.1) < 1e-15
    assert abs(average_rate(4.0, 1.0, 2) - 0.5) < 1e-15
    assert average_rate(3.0, 3.0, 5) == 1.0
    with pytest.raises(ValueError):
        average_rate(1.0, 0.5, 0)


def test_givens_zeroes_second_component():
    rng = np.random.default_rng(0)
    for _ in range(20):
        a, b = rng.standard_normal(2) + 1j * rng.standard_normal(2)
        c, s = givens(a, b)
        G = np.array([[c, s], [-np.conj(s), c]])
        r = G @ np.array([a, b])
        assert abs(r[1]) < 1e-15 * abs(r[0])
        assert np.allclose(G.conj().T @ G, np.eye(2), atol=1e-15)


def _rand_system(N, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N)) + 3 * np.sqrt(N) * np.eye(N)
    b = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    return A, b


def test_exact_preconditioner_one_iteration():
    """P^{-1} = A^{-1} (dense): converges in one iteration to round-off."""
    A, b = _rand_system(40, 1)
    Ainv = np.linalg.inv(A)
    x, rep = fgmres(lambda v: A @ v, lambda v: Ainv @ v, b, rtol=1e-12)
    assert rep.iterations == 1
    assert rep.rel_res_true < 1e-12


def test_unpreconditioned_finite_termination():
    """Identity preconditioner on N <= 25: GMRES finishes in <= N steps at the
    dense solution."""
    A, b = _rand_system(25, 2)
    x, rep = fgmres(lambda v: A @ v, lambda v: v, b, rtol=1e-13, restart=100)
    assert rep.iterations <= 25
    xs = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xs) <= 1e-11 * np.linalg.norm(xs)


def test_flexible_preconditioner_and_monotone_residual():
    """Iteration-varying preconditioner (alternating identity / Jacobi) still
    reaches the dense solution; |g_{j+1}| is non-increasing within a cycle."""
    A, b = _rand_system(50, 3)
    d = np.diag(A)
    state = {"i": 0}

    def pinv(v):
        state["i"] += 1
        return v if state["i"] % 2 else v / d

    x, rep = fgmres(lambda v: A @ v, pinv, b, rtol=1e-12, restart=100)
    xs = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xs) <= 1e-10 * np.linalg.norm(xs)
    h = rep.history
    assert all(h[i + 1] <= h[i] * (1 + 1e-14) for i in range(len(h) - 1))
    assert rep.max_orth_loss <= 1e-12


def test_restarted_reaches_solution():
    A, b = _rand_system(60, 4)
    x, rep = fgmres(lambda v: A @ v, lambda v: v, b, rtol=1e-10, restart=5, max_iters=500)
    assert rep.restarts >= 1 and rep.converged
    assert rep.rel_res_true <= 1.01e-10


def test_cfg0_oracle_solve():
    """cfg0 (BASELINE.json configs[0]): the preconditioned solve converges, the
    true residual is at the tolerance and x matches the direct solution u* =
    A_0^{-1} F within rtol * cond-level slack."""
    spec = config_spec("cfg0")
    op = OracleProblem(spec)
    x, rep = op.solve()
    assert rep.converged and 5 <= rep.iterations <= 20
    assert rep.rel_res_true <= 1.01 * spec.rtol
    b = spec.rhs()
    us = spla.spsolve(op.A0.tocsc(), b)
    assert np.linalg.norm(x - us) <= 1e-3 * np.linalg.norm(us)
    assert rep.max_orth_loss <= 1e-12
    h = rep.history
    assert all(h[i + 1] <= h[i] * (1 + 1e-14) for i in range(len(h) - 1))


def test_fixed_iters_runs_exactly():
    spec = config_spec("cfg0", n=16)
    op = OracleProblem(spec)
    x, rep = op.solve(fixed_iters=3)
    assert rep.iterations == 3
