"""Oracle of the fitted shift-exponent map sigma_p (Table 1).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

  k_c(l)      = k_c1 * exp(k_c0 * l)
  alpha(l)    = alpha_1 * exp(alpha_0 * l)
  beta(k, l)  = 2 - exp(-alpha(l) * (k - k_c(l)))
  sigma_p     = min(max(beta, 1), 2)
with the weights (k_c0, k_c1, alpha_0, alpha_1) of Table 1.
The shift of a heterogeneous solve is eps_e = k_e^{sigma_p(k_e, l)}
(PAPER.md:532-533); l = log2(n) of the fine mesh on both levels (reading C20).
"""
from __future__ import annotations

import numpy as np

TABLE1 = {
    1: (0.4592788619853418, 2.5790032999702346, -0.6261637288068426, 1.7580549857142198),
    2: (0.5736926870738827, 2.5729974893966001, -0.6615199737374460, 1.5966386518185063),
    3: (0.6305770719029798, 2.4284320222555804, -0.4465407372367102, 0.1287828338493968),
}


def sigma_p(k, l, coeffs):
    kc0, kc1, a0, a1 = coeffs
    kc = kc1 * np.exp(kc0 * l)
    alpha = a1 * np.exp(a0 * l)
    beta = 2.0 - np.exp(-alpha * (np.asarray(k, dtype=np.float64) - kc))
    return np.minimum(np.maximum(beta, 1.0), 2.0)


def map_shifts(k_elem, beta, p, l):
    """eps_e = beta * k_e^{sigma_p(k_e, l)}."""
    k = np.asarray(k_elem, dtype=np.float64)
    return beta * k ** sigma_p(k, l, TABLE1[p])


def loss(coeffs, k, l, sigma_hat):
    """loss_p = sum_i w_{l_i}^-2 (sigma_hat_i - sigma_p(k_i, l_i))^2, w_l = N_l / |D|."""
    l = np.asarray(l)
    w = np.array([np.mean(l == li) for li in l])
    return float(np.sum(w ** -2 * (np.asarray(sigma_hat) - sigma_p(k, l, coeffs)) ** 2))
