"""Oracle of the near-optimal shift search (Sec. 5, steps 1-6).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Step 5: "Find the optimal exponent sigma_hat in [1,2] of the
complex shift k^sigma using the gradient free golden-section search [Kiefer
1953] with a tolerance of 1e-2", where the objective is the
average convergence rate rho = (r_end / r_0)^(1/end) of the FGMRES solve of the
UNSHIFTED system with the true residual norms, solved "until either a relative
residual reduction of 1e-8 is obtained or a maximum of 50 iterations".

golden_section follows Kiefer's two-interior-point reduction literally: the
bracket [a, b] keeps the interior points c = b - (b - a)/phi, d = a + (b - a)/phi;
if f(c) < f(d) the minimum is kept in [a, d], else (including ties) in [c, b];
one new evaluation per reduction; stop when b - a <= tol; return (a + b) / 2.
A failed solve scores rho = 1 (reading S1 in DESIGN.md).
"""
from __future__ import annotations

import math
from dataclasses import replace

import numpy as np

from .solve import OracleProblem

INVPHI = (math.sqrt(5.0) - 1.0) / 2.0


def golden_section(f, a: float, b: float, tol: float):
    """Minimise f on [a, b]; returns (midpoint of the final bracket, evaluations list)."""
    if not a < b or not tol > 0:
        raise ValueError("need a < b and tol > 0")
    evals = []

    def F(x):
        v = f(x)
        evals.append((x, v))
        return v

    c = b - INVPHI * (b - a)
    d = a + INVPHI * (b - a)
    fc, fd = F(c), F(d)
    while b - a > tol:
        if fc < fd:            # minimum in [a, d]
            b, d, fd = d, c, fc
            c = b - INVPHI * (b - a)
            fc = F(c)
        else:                  # minimum in [c, b]
            a, c, fc = c, d, fd
            d = a + INVPHI * (b - a)
            fd = F(d)
    return 0.5 * (a + b), evals


def rho_of(spec, sigma: float, rhs, rtol=1e-8, max_iters=50):
    """rho(sigma): FGMRES on A_0 u = rhs, V-cycle on A(k, beta k^sigma)."""
    s = replace(spec, sigma=sigma, rtol=rtol, max_iters=max_iters)
    try:
        _, rep = OracleProblem(s).solve(rhs)
    except Exception:          # breakdown: worst score
        return 1.0, 0
    r = rep.rho if np.isfinite(rep.rho) else 1.0
    return float(r), rep.iterations


def search_sample(spec, rhs, lo=1.0, hi=2.0, tol=1e-2, rtol=1e-8, max_iters=50, iters=None):
    """(sigma_hat, evaluations [(sigma, rho)]) for one (k, l) sample; `iters`, if a
    list, receives the FGMRES iteration count of every evaluation."""
    def f(s):
        r, its = rho_of(spec, s, rhs, rtol, max_iters)
        if iters is not None:
            iters.append(its)
        return r
    return golden_section(f, lo, hi, tol)
