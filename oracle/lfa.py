"""Oracle: Local Fourier Analysis symbols of the 2D Q1 two-grid method,
transcribed from PAPER.md section 3.  Used ONLY as an independent pin of the
assembled operator (Fourier-mode test) and of the V-cycle (measured
contraction vs rho_loc); it is not on the product path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:205-217  harmonics theta^(a) and T^low = (-pi/2, pi/2]^2
PAPER.md:245-249  rho_loc = sup_{theta in T^low} rho(T_hat(theta))
PAPER.md:252-258  T_hat = S^nu2 K_hat S^nu1,  K_hat = I - I_2h^h L_2h^{-1} I_h^2h L_h
PAPER.md:273-277  symbol of L_h
PAPER.md:283-289  symbol of L_2h (evaluated at 2 theta)
PAPER.md:292-306  prolongation / restriction symbols, I_h^2h = (1/4) (I_2h^h)^T
PAPER.md:343-346  sigma_c = argmin_{sigma in [1,2]} {rho_loc(sigma) < 1} (I_conv = [sigma_c, 2],
                  reading G2), found by bisection (sigma_c below)
PAPER.md:327-334  symbol of the damped Jacobi smoother S_h (the symbol is
                  right; the printed S_h *stencil* corners at PAPER.md:157-160
                  are garbled, reading G1 in DESIGN.md)
lambda = k^2 + i eps (the paper's eps = k^sigma; BASELINE adds a factor beta).
"""
from __future__ import annotations

import numpy as np


def L_h(t1, t2, lam, h):
    """Fourier symbol of L_h."""
    c1, c2 = np.cos(t1), np.cos(t2)
    return (8 - 2 * c1 - 2 * c2 - 4 * c1 * c2) / 3.0 - lam * h * h / 36.0 * (
        16 + 8 * c1 + 8 * c2 + 4 * c1 * c2)


def L_2h(t1, t2, lam, h):
    """Fourier symbol of L_2h at frequency theta (uses cos 2 theta)."""
    c1, c2 = np.cos(2 * t1), np.cos(2 * t2)
    return (8 - 2 * c1 - 2 * c2 - 4 * c1 * c2) / 3.0 - lam * h * h / 9.0 * (
        16 + 8 * c1 + 8 * c2 + 4 * c1 * c2)


def S_h(t1, t2, lam, h, omega):
    """Damped Jacobi symbol."""
    c1, c2 = np.cos(t1), np.cos(t2)
    den = 8.0 / 3.0 - lam * h * h * 16.0 / 36.0
    a = (2.0 / 3.0 + lam * h * h * 8.0 / 36.0) / den
    b = (4.0 / 3.0 + lam * h * h * 4.0 / 36.0) / den
    return (1 - omega) + omega * a * c1 + omega * a * c2 + omega * b * c1 * c2


def harmonics(t1, t2):
    """theta^(0,0), theta^(1,1), theta^(1,0), theta^(0,1)."""
    b1 = t1 + np.pi if t1 < 0 else t1 - np.pi
    b2 = t2 + np.pi if t2 < 0 else t2 - np.pi
    return [(t1, t2), (b1, b2), (b1, t2), (t1, b2)]


def prolongation_symbol(t1, t2):
    """Column I_hat_2h^h(theta)."""
    c1, c2 = np.cos(t1), np.cos(t2)
    return np.array([(1 + c1) * (1 + c2), (1 - c1) * (1 - c2),
                     (1 - c1) * (1 + c2), (1 + c1) * (1 - c2)], dtype=np.complex128)


def two_grid_symbol(t1, t2, lam, h, omega, nu1, nu2):
    """T_hat(theta) = S^nu2 (I - P L_2h^{-1} R L_h) S^nu1."""
    H = harmonics(t1, t2)
    Lh = np.diag([L_h(a, b, lam, h) for a, b in H])
    Sh = np.diag([S_h(a, b, lam, h, omega) for a, b in H])
    P = prolongation_symbol(t1, t2).reshape(4, 1)
    R = 0.25 * P.T
    L2 = L_2h(t1, t2, lam, h)
    K = np.eye(4) - (P @ R @ Lh) / L2
    return np.linalg.matrix_power(Sh, nu2) @ K @ np.linalg.matrix_power(Sh, nu1)


def rho_loc(lam, h, omega, nu1, nu2, m=128):
    """sup over an m x m grid of T^low = (-pi/2, pi/2]^2 of rho(T_hat)
    (PAPER.md:247), skipping theta = 0 where L_2h may be singular."""
    ts = -np.pi / 2 + np.pi * (np.arange(m) + 1) / m
    best = 0.0
    for t1 in ts:
        for t2 in ts:
            if abs(t1) < 1e-12 and abs(t2) < 1e-12:
                continue
            T = two_grid_symbol(t1, t2, lam, h, omega, nu1, nu2)
            best = max(best, float(np.max(np.abs(np.linalg.eigvals(T)))))
    return best


def lam_of(k, beta, sigma):
    """lambda = k^2 + i beta k^sigma (reading C2)."""
    return k * k + 1j * beta * k ** sigma


def sigma_c(k, h, beta=1.0, omega=0.6, nu1=2, nu2=2, m=64, lo=1.0, hi=2.0, tol=1e-3):
    """Smallest sigma in [lo, hi] with rho_loc(sigma) < 1, by
    bisection assuming rho_loc decreases with sigma: lo if rho_loc(lo) < 1, NaN if
    rho_loc(hi) >= 1, else the upper end of the final bracket (width <= tol)."""
    r = lambda s: rho_loc(lam_of(k, beta, s), h, omega, nu1, nu2, m)
    if r(lo) < 1.0:
        return lo
    if not r(hi) < 1.0:
        return float("nan")
    while hi - lo > tol:
        mid = 0.5 * (lo + hi)
        if r(mid) < 1.0:
            hi = mid
        else:
            lo = mid
    return hi
