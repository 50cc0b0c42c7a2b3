"""Oracle: right-preconditioned flexible GMRES(m) (Saad 1993).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md:357-360 (section 4): solve A_0 P_eps^{-1} (P_eps u) = F with
A_0 = A(k, 0) and P_eps^{-1} one V-cycle on A_eps; the flexible variant keeps
the preconditioned vectors z_j = P^{-1} v_j.  PAPER.md:416-420: the average
convergence rate rho = (r_end / r_0)^(1/end) uses TRUE residuals.

Readings: modified Gram-Schmidt with selective
re-orthogonalisation (DGKS, threshold 1/sqrt 2) and inner product
<v, w> = sum conj(v_i) w_i (C11, C19); complex Givens rotations
c = |a|/t, s = (a/|a|) conj(b)/t, t = sqrt(|a|^2+|b|^2); stopping test
|g_{j+1}| <= rtol ||b|| (C13); x0 = 0; restarts recompute r = b - A_0 x and
keep the threshold relative to ||b|| (C14); iterations = number of
preconditioner applications.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class FgmresReport:
    iterations: int = 0
    restarts: int = 0
    converged: bool = False
    rel_res_lsq: float = float("nan")
    rel_res_true: float = float("nan")
    rho: float = float("nan")
    history: list = field(default_factory=list)   # |g_{j+1}| / ||b|| per iteration
    max_orth_loss: float = 0.0                     # max_cycle ||V^H V - I||


def givens(a: complex, b: complex):
    """Complex Givens rotation zeroing b in (a, b): returns (c, s) with
    [c, s; -conj(s), c] (a, b)^T = (r, 0)^T."""
    if b == 0:
        return 1.0, 0.0
    if a == 0:
        return 0.0, 1.0 + 0j
    t = np.sqrt(abs(a) ** 2 + abs(b) ** 2)
    c = abs(a) / t
    s = (a / abs(a)) * np.conj(b) / t
    return c, s


def average_rate(r0: float, r_end: float, end: int) -> float:
    """rho = (r_end / r_0)^(1/end)."""
    if end < 1 or r0 <= 0:
        raise ValueError("rho undefined for end < 1 or r0 <= 0")
    return (r_end / r0) ** (1.0 / end)


def fgmres(apply_A, apply_Pinv, b, restart=100, rtol=1e-6, max_iters=500,
           fixed_iters=0, reorth=True, x0=None):
    """Flexible GMRES(restart).  Returns (x, FgmresReport)."""
    N = b.shape[0]
    x = np.zeros(N, dtype=np.complex128) if x0 is None else x0.astype(np.complex128).copy()
    bnorm = np.linalg.norm(b)
    rep = FgmresReport()
    if bnorm == 0:
        rep.converged, rep.rel_res_lsq, rep.rel_res_true = True, 0.0, 0.0
        return x, rep
    target = rtol * bnorm
    r = b - apply_A(x) if x0 is not None else b.astype(np.complex128).copy()
    beta = np.linalg.norm(r)
    total = 0
    m = restart
    done = False
    while not done:
        V = np.zeros((m + 1, N), dtype=np.complex128)
        Z = np.zeros((m, N), dtype=np.complex128)
        H = np.zeros((m + 1, m), dtype=np.complex128)
        cs = np.zeros(m)
        sn = np.zeros(m, dtype=np.complex128)
        g = np.zeros(m + 1, dtype=np.complex128)
        V[0] = r / beta
        g[0] = beta
        j_end = 0
        for j in range(m):
            Z[j] = apply_Pinv(V[j])
            w = apply_A(Z[j])
            # modified Gram-Schmidt
            wnorm0 = np.linalg.norm(w)
            for i in range(j + 1):
                H[i, j] = np.vdot(V[i], w)
                w = w - H[i, j] * V[i]
            wnorm = np.linalg.norm(w)
            if reorth and wnorm < wnorm0 / np.sqrt(2.0):
                for i in range(j + 1):
                    c_ = np.vdot(V[i], w)
                    H[i, j] += c_
                    w = w - c_ * V[i]
                wnorm = np.linalg.norm(w)
            H[j + 1, j] = wnorm
            # apply previous rotations to the new column
            for i in range(j):
                hi, hi1 = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * hi + sn[i] * hi1
                H[i + 1, j] = -np.conj(sn[i]) * hi + cs[i] * hi1
            cs[j], sn[j] = givens(H[j, j], H[j + 1, j])
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            total += 1
            j_end = j + 1
            rep.history.append(abs(g[j + 1]) / bnorm)
            breakdown = wnorm == 0.0
            if not breakdown:
                V[j + 1] = w / wnorm
            if fixed_iters:
                if total >= fixed_iters:
                    done = True
                    break
            elif abs(g[j + 1]) <= target or total >= max_iters:
                done = True
                break
            if breakdown:
                done = True
                break
        # orthogonality diagnostic for this cycle
        Vc = V[: j_end + 1] if np.any(V[j_end] != 0) else V[:j_end]
        G = Vc.conj() @ Vc.T
        rep.max_orth_loss = max(rep.max_orth_loss, float(np.abs(G - np.eye(G.shape[0])).max()))
        # y = H^{-1} g (upper triangular j_end x j_end), x <- x + Z y
        y = np.zeros(j_end, dtype=np.complex128)
        for i in range(j_end - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:j_end] @ y[i + 1:j_end]) / H[i, i]
        x = x + Z[:j_end].T @ y
        rep.rel_res_lsq = abs(g[j_end]) / bnorm
        if not done:
            rep.restarts += 1
            r = b - apply_A(x)
            beta = np.linalg.norm(r)
            if (not fixed_iters) and beta <= target:
                done = True
    rep.iterations = total
    rtrue = np.linalg.norm(b - apply_A(x))
    rep.rel_res_true = rtrue / bnorm
    rep.converged = bool(rep.rel_res_lsq <= rtol) if not fixed_iters else bool(rep.rel_res_true <= rtol)
    rep.rho = average_rate(bnorm, rtrue, total) if total > 0 else float("nan")
    return x, rep
